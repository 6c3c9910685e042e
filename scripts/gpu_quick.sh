# usage: bash scripts/gpu_quick.sh "<pytest -k expr or empty>" "<configs>"
cd $GRAFT_REPO_ROOT
K="$1"; CFGS="${2:-2 3}"
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "$K" > gpurun_out/pytest_quick.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_quick.log
fi
for c in $CFGS; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "bench c$c exit $?"
  python - <<PY
import json
d=json.load(open('gpurun_out/bench_c$c.json')); r=d['roofline']
print('c$c img/s %.1f ms/step %.3f hbmfrac %.3f | fwd %.3f inv %.3f ms | dom %s frac %.3f | rt %.1e'%(d['value'],d['ms_per_step'],d['hbm_frac_step'],r['kernel_ms']['fwd_main'],r['kernel_ms']['inv_main'],r['kernel'],r['frac'],d['roundtrip_max_rel_err']))
PY
done
