cd $GRAFT_REPO_ROOT
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench exit $?"
for c in 3 4 5 1; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "bench c$c exit $?"
done
CMD="python bench.py --steps 2 --warmup 3 --cpu-budget 1"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
CMD2="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD2 > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:main_kernel -s 2 -c 2 -o /tmp/prof_c2 $CMD2 > /tmp/ncu_full.log 2>&1; echo "ncu full exit $?"
tail -3 /tmp/ncu_full.log
ncu -i /tmp/prof_c2.ncu-rep --page raw --csv > gpurun_out/prof_c2_raw.csv 2>&1
ncu -i /tmp/prof_c2.ncu-rep --page details --csv > gpurun_out/prof_c2_details.csv 2>&1
ncu -i /tmp/prof_c2.ncu-rep --page source --csv --print-source sass > /tmp/src.csv 2>&1; gzip -c /tmp/src.csv > gpurun_out/prof_c2_source.csv.gz
ls -la /tmp/prof_c2.ncu-rep gpurun_out/
sz=$(stat -c %s /tmp/prof_c2.ncu-rep); if [ "$sz" -lt 30000000 ]; then cp /tmp/prof_c2.ncu-rep gpurun_out/; fi
for f in gpurun_out/bench_c*.json; do echo $f; cut -c1-300 $f; done
