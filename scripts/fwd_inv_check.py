# one forward + inverse of a plan: python scripts/fwd_inv_check.py N f32|f64 classic|smooth
import sys, torch
sys.path.insert(0, '.')
import paper_1202_1773_b200 as F
import synth
n = int(sys.argv[1]); dt = torch.float64 if sys.argv[2] == 'f64' else torch.float32; var = sys.argv[3]
x = torch.from_numpy(synth.make_batch(2, batch=3, n=n)).to(dt).cuda()
plan = F.Plan(n, 3, dt, variant=var)
c = plan.forward(x); torch.cuda.synchronize(); print('fwd ok', flush=True)
r = plan.inverse(c); torch.cuda.synchronize(); print('inv ok', float((r - x).abs().max()), flush=True)
