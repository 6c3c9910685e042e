# round bench: every config with default settings (+ oracle baseline, cuFFT line), launch list and
# one full ncu capture of config 2's two persistent kernels
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
for c in 2 1 3 4 5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "bench c$c exit $?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_c$c.json')); r=d['roofline']
print('c$c img/s %.1f step %.4f ms | fwd %.4f inv %.4f | dom %s frac %.3f | e2e %.1f | cpu %s | cufft %s | clocks %s'%(d['value'],d['ms_per_step'],r['kernel_ms']['fwd_main'],r['kernel_ms']['inv_main'],r['kernel'],r['frac'],d['e2e']['value'] if d['e2e'] else 0, (d['cpu_baseline'] or {}).get('value'), (d['cufft_line'] or {}).get('value'), d['clocks']))" || tail -3 gpurun_out/bench_c$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cufft > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
timeout 600 bash scripts/gpu_prof.sh 2 c2final main_kernel 2 2 > /dev/null 2>&1; echo "ncu full exit $?"
