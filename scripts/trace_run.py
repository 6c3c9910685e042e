"""Per-item timeline of the persistent kernels (GPU box).  Usage:
   python scripts/trace_run.py <config> [out.npz]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1202_1773_b200 as F  # noqa: E402
import synth  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
out = sys.argv[2] if len(sys.argv) > 2 else f"gpurun_out/trace_c{cid}.npz"
cfg = synth.config(cid)
dtype = torch.float32 if cfg.dtype == "f32" else torch.float64
plan = F.Plan(cfg.n, cfg.batch, dtype)
x = torch.from_numpy(synth.make_batch(cid)).to(dtype).cuda()
c = plan.forward(x)
rec = plan.inverse(c)
torch.cuda.synchronize()
plan.set_trace(True)
plan.forward(x, out=c)
plan.inverse(c, out=rec)
torch.cuda.synchronize()
res = {}
for which, name in ((0, "fwd"), (1, "inv")):
    t = plan.trace(which)
    res[name] = t
    t0 = t[:, 3].min()
    span = (t[:, 5].max() - t0) / 1e3
    print(f"== {name}: items {len(t)} span {span:.1f} us")
    for ty in (0, 1):
        m = t[:, 0] == ty
        if not m.any():
            continue
        wait = (t[m, 4] - t[m, 3]) / 1e3
        work = (t[m, 5] - t[m, 4]) / 1e3
        print(f"  type {ty}: n={m.sum()} wait mean {wait.mean():.2f} p90 {np.percentile(wait, 90):.2f} max {wait.max():.1f} us"
              f" | work mean {work.mean():.2f} p10 {np.percentile(work, 10):.2f} p90 {np.percentile(work, 90):.2f} us"
              f" | total work {work.sum():.0f} us, total wait {wait.sum():.0f} us")
    # per-CTA busy fraction: sum of (t_end - t_start) per sm over the span
    sms = t[:, 2]
    busy = np.zeros(sms.max() + 1)
    for s in np.unique(sms):
        mm = sms == s
        busy[s] = ((t[mm, 5] - t[mm, 3]).sum()) / 1e3
    print(f"  per-SM item time (2 CTAs/SM => max 2x span): mean {busy[busy > 0].mean():.1f} us of span {span:.1f}")
    # gaps between consecutive items on the same SM (scheduling overhead)
np.savez_compressed(out, **res)
print("saved", out)
# intra-item probes (relative to t_ready)
for name in ("fwd", "inv"):
    t = res[name]
    for ty in (0, 1):
        m = (t[:, 0] == ty) & (t[:, 6] > 0)
        if not m.any():
            continue
        rel = [(t[m, 6 + i] - t[m, 4]) / 1e3 for i in range(4)]
        print(f"  {name} type {ty} probes (us after ready): " +
              " ".join(f"p{i}={np.median(r):.2f}" for i, r in enumerate(rel) if (t[m, 6 + i] > 0).any()) +
              f" end={np.median((t[m, 5] - t[m, 4]) / 1e3):.2f}")
