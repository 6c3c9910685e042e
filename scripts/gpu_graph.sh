cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 1 2 3; do for g in "" "--no-graph"; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-cufft $g > gpurun_out/g.json 2>gpurun_out/g.err || tail -3 gpurun_out/g.err
  python -c "
import json; d=json.load(open('gpurun_out/g.json')); r=d['roofline']
print('c$c $g | img/s %.0f step %.4f | fwd %.4f inv %.4f | %s | launches %s'%(d['value'],d['ms_per_step'],r['kernel_ms']['fwd_main'],r['kernel_ms']['inv_main'],d['config']['launch'],d['gpu_launches']))"
done; done
