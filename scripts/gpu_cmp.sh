cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export FFST_RING_MB=${RING:-96}
for v in ${VARIANTS:-default}; do
  if [ "$v" != "default" ]; then export FFST_LIB=$PWD/paper_1202_1773_b200/libffst_$v.so; else unset FFST_LIB; fi
  for c in ${CFGS:-2}; do for only in ${ONLY:-0}; do
    if [ "$only" != "0" ]; then export FFST_QUEUE_ONLY=$only; else unset FFST_QUEUE_ONLY; fi
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err || tail -2 gpurun_out/b.err
    python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']
print('$v c$c only=$only | img/s %.0f step %.4f | fwd %.4f inv %.4f ms | rt %.1e'%(d['value'],d['ms_per_step'],r['kernel_ms']['fwd_main'],r['kernel_ms']['inv_main'],d['roundtrip_max_rel_err']))"
  done; done
done
