# usage: ENVS="A=1 B=2;A=2" CFGS="2 3" bash scripts/gpu_env.sh  — bench each ';'-separated env set
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
IFS=';' read -ra SETS <<< "${ENVS:-}"
[ ${#SETS[@]} -eq 0 ] && SETS=("")
for e in "${SETS[@]}"; do for c in ${CFGS:-2}; do
  env $e timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-cufft > gpurun_out/b.json 2>gpurun_out/b.err || tail -2 gpurun_out/b.err
  python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']
print('[$e] c$c | img/s %.0f step %.4f | fwd %.4f inv %.4f ms | frac %.3f rt %.1e'%(d['value'],d['ms_per_step'],r['kernel_ms']['fwd_main'],r['kernel_ms']['inv_main'],r['frac'],d['roundtrip_max_rel_err']))"
done; done
