cd $GRAFT_REPO_ROOT
for cp in 2 4 8 16; do for ring in 48 96; do
  FFST_CHUNK_PLANES=$cp FFST_RING_MB=$ring timeout 300 python bench.py --config ${1:-2} --steps 5 --warmup 3 --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/b.json')); r=d['roofline']
print('chunk_planes $cp ring $ring: img/s %.0f ms %.3f fwd %.3f inv %.3f'%(d['value'],d['ms_per_step'],r['kernel_ms']['fwd_main'],r['kernel_ms']['inv_main']))"
done; done
