cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in A B A B; do
  if [ $v = B ]; then export FFST_LIB=$PWD/_scratch/b/paper_1202_1773_b200/libffst.so; else unset FFST_LIB; fi
  timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-cufft > gpurun_out/g.json 2>gpurun_out/g.err || tail -3 gpurun_out/g.err
  python -c "
import json; d=json.load(open('gpurun_out/g.json')); r=d['roofline']
print('$v c5 | img/s %.2f step %.3f | fwd %.3f inv %.3f'%(d['value'],d['ms_per_step'],r['kernel_ms']['fwd_main'],r['kernel_ms']['inv_main']))"
done
