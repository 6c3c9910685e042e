cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for a in "2048 f64 classic" "2048 f32 classic" "4096 f32 classic" "2048 f32 smooth"; do echo "-- $a: $(timeout 120 python scripts/fwd_inv_check.py $a 2>&1 | tail -1)"; done
timeout 900 python -m pytest tests -q -m gpu -x -k "config5 or large or config_sampled or config2_full" 2>&1 | tail -2
for c in 5 4 2; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-cufft > gpurun_out/g.json 2>gpurun_out/g.err || tail -3 gpurun_out/g.err
  python -c "
import json; d=json.load(open('gpurun_out/g.json')); r=d['roofline']
print('c$c | img/s %.2f step %.3f | fwd %.3f inv %.3f | rt %.1e'%(d['value'],d['ms_per_step'],r['kernel_ms']['fwd_main'],r['kernel_ms']['inv_main'],d['roundtrip_after_timed_steps']))"
done
