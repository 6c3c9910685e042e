cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -4 gpurun_out/pytest_gpu.log
for c in 1 2; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-cufft > gpurun_out/bench_c$c.json 2>gpurun_out/bench_c$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_c$c.json')); r=d['roofline']; print($c, round(d['value'],1), round(d['ms_per_step'],4), {k: round(v,4) for k,v in r['kernel_ms'].items()})" || tail -3 gpurun_out/bench_c$c.err
done
