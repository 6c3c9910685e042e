cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for only in "" 1 2; do
  if [ -n "$only" ]; then export FFST_QUEUE_ONLY=$only; else unset FFST_QUEUE_ONLY; fi
  for c in ${CFGS:-2}; do
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err || tail -3 gpurun_out/b.err
    python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']
print('only=${only:-all} c$c | fwd %.4f inv %.4f ms'%(r['kernel_ms']['fwd_main'],r['kernel_ms']['inv_main']))"
  done
done
