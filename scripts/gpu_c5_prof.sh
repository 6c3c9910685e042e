cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 exit $?"
cat gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5.err
timeout 300 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2>&1; echo "bench c2 exit $?"; cat gpurun_out/bench_c2.json
# launch list of the default bench command
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
# full capture of the two persistent kernels
timeout 900 bash scripts/gpu_prof.sh 2 c2r1 main_kernel 2 2
