# usage: bash scripts/gpu_prof.sh <config> <tag> [kernel-regex] [launch-skip] [count]
cd $GRAFT_REPO_ROOT
C=${1:-2}; TAG=${2:-x}; KR=${3:-main_kernel}; S=${4:-2}; CNT=${5:-2}
CMD="python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:$KR -s $S -c $CNT -o /tmp/prof_$TAG $CMD > /tmp/ncu_$TAG.log 2>&1; echo "ncu exit $?"
tail -2 /tmp/ncu_$TAG.log
ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page details --csv > gpurun_out/prof_${TAG}_details.csv 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src.csv 2>&1; gzip -c /tmp/src.csv > gpurun_out/prof_${TAG}_source.csv.gz
sz=$(stat -c %s /tmp/prof_$TAG.ncu-rep); if [ "$sz" -lt 25000000 ]; then cp /tmp/prof_$TAG.ncu-rep gpurun_out/; fi
ls -la gpurun_out | tail -5
