# usage: bash scripts/gpu_iter.sh "<pytest -k expr | all | none>" "<configs>" [extra env for a comparison run, e.g. FFST_PATH=cta]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
K="$1"; CFGS="${2:-2 3}"; CMP="$3"
if [ "$K" = "all" ]; then
  timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/pytest_gpu.log
elif [ "$K" != "none" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "$K" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/pytest_gpu.log
fi
summ() {
python - "$1" <<'PY'
import json,sys
d=json.load(open(sys.argv[1])); r=d['roofline']
print('%s img/s %.1f ms/step %.4f hbmfrac %.3f | fwd %.4f inv %.4f ms | dom %s frac %.3f | rt %.1e | e2e %.1f'%(sys.argv[1].split('/')[-1],d['value'],d['ms_per_step'],d['hbm_frac_step'],r['kernel_ms']['fwd_main'],r['kernel_ms']['inv_main'],r['kernel'],r['frac'],d['roundtrip_max_rel_err'],d['e2e']['value'] if d['e2e'] else 0))
PY
}
for c in $CFGS; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "bench c$c exit $?"; tail -2 gpurun_out/bench_c$c.err
  summ gpurun_out/bench_c$c.json
  if [ -n "$CMP" ]; then
    env $CMP timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c${c}_cmp.json 2> gpurun_out/bench_c${c}_cmp.err; echo "bench c$c ($CMP) exit $?"
    summ gpurun_out/bench_c${c}_cmp.json
  fi
done
