"""Debug: inverse (adjoint) of the GPU path vs the oracle for several n / batch / dtype."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
import synth
import paper_1202_1773_b200 as F

def perr(g, o):
    return float(np.max(np.abs(g - o)) / max(np.max(np.abs(o)), 1e-300))

for dtype in (torch.float64, torch.float32):
    for n in (8, 16, 32, 64, 128, 256):
        for batch in (1, 3):
            x = synth.make_batch(2, batch=batch, n=n)
            xt = torch.from_numpy(x).to(dtype)
            plan = F.Plan(n, batch, dtype)
            c = plan.forward(xt.cuda())
            rec = plan.inverse(c)
            torch.cuda.synchronize()
            cn = c.cpu().numpy(); rn = rec.cpu().numpy()
            psi = O.shearlet_spectra(n)
            fe, ie = [], []
            for b in range(batch):
                ref = O.forward(xt[b].double().numpy(), psi=psi)
                fe.append(perr(cn[b], ref))
                ie.append(perr(rn[b], O.inverse(cn[b].astype(np.complex128), psi=psi).real))
            # single-plane cubes: which planes break the inverse
            bad = []
            if max(ie) > (1e-3 if dtype == torch.float32 else 1e-8):
                for i in range(plan.eta):
                    z = torch.zeros_like(c)
                    z[0, i] = c[0, i]
                    r1 = plan.inverse(z)[0].cpu().numpy()
                    e = perr(r1, O.inverse(z[0].cpu().numpy().astype(np.complex128), psi=psi).real)
                    if e > (1e-3 if dtype == torch.float32 else 1e-8):
                        bad.append((i, F.index_to_params(plan.j0, i), round(e, 3)))
            print(f"{str(dtype)[6:]} n={n} B={batch} fwd {max(fe):.1e} inv {['%.1e' % v for v in ie]} bad planes {bad[:8]}", flush=True)
