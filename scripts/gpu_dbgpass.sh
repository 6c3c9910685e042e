cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export FFST_RING_MB=96
for only in 1 2; do for dbg in ${DBGS:-0 1 2 4 7}; do
  FFST_QUEUE_ONLY=$only FFST_DBG=$dbg timeout 300 python bench.py --config ${C:-2} --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err || tail -2 gpurun_out/b.err
  python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']
print('only=$only dbg=$dbg | fwd %.4f inv %.4f ms'%(r['kernel_ms']['fwd_main'],r['kernel_ms']['inv_main']))"
done; done
