# smooth-variant parity + classic perf check (one gpurun call)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "smooth" > gpurun_out/pytest_smooth.log 2>&1; echo "pytest smooth exit $?"; tail -15 gpurun_out/pytest_smooth.log
for c in 2 3; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-cufft > gpurun_out/bench_c$c.json 2>gpurun_out/bench_c$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_c$c.json')); print($c, d['value'], d['ms_per_step'], d.get('compact_line',{}).get('value'))"
done
