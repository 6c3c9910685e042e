"""World-size-2 gloo test of the eta-sharded path's host logic (plane ownership,
broadcast in, reduce out) on CPU.  The per-rank transform is a stand-in built
from the oracle (test infrastructure); on GPUs the same ShardedTransform wraps
the CUDA Plan (covered by test_gpu_parity.py::test_shards_sum_to_full)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth


def _load_dist_module():
    # import paper_1202_1773_b200/dist.py without loading the CUDA library (CPU test of host logic)
    import importlib.util
    from pathlib import Path
    path = Path(__file__).resolve().parents[1] / "paper_1202_1773_b200" / "dist.py"
    spec = importlib.util.spec_from_file_location("ffst_dist_hostlogic", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


class OracleShard:
    """Per-rank stand-in: forward/inverse restricted to the owned planes (float64)."""

    def __init__(self, n, planes, variant="classic"):
        self.n = n
        self.local_planes = planes
        self.psi = O.shearlet_spectra(n, variant=variant)

    def forward(self, x):
        out = []
        for img in x.numpy():
            f_hat = O.dft2_centred(img)
            out.append(np.stack([O.idft2_centred(self.psi[i] * f_hat) for i in self.local_planes]))
        return torch.from_numpy(np.stack(out))

    def inverse(self, c):
        out = [O.inverse(cb.numpy(), psi=self.psi, planes=[i + 1 for i in self.local_planes]).real for cb in c]
        return torch.from_numpy(np.stack(out))


def _worker(rank, world, port, n, batch, result_q, variant="classic"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    D = _load_dist_module()
    eta = O.num_shearlets(O.scales_for_size(n))
    planes = D.owned_planes(eta, rank, world)
    st = D.ShardedTransform(OracleShard(n, planes, variant))
    if rank == 0:
        x = torch.from_numpy(synth.make_batch(2, batch=batch, n=n))
    else:
        x = torch.zeros(batch, n, n, dtype=torch.float64)
    c = st.forward(x)
    rec = st.inverse(c)
    if rank == 0:
        result_q.put(("rec", rec.numpy(), x.numpy()))
    result_q.put(("planes", rank, planes, c.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,variant", [(2, "classic"), (3, "classic"), (2, "smooth")])
def test_sharded_roundtrip_gloo(world, variant):
    n, batch = 32, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + world + (10 if variant == "smooth" else 0)
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, batch, q, variant)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world + 1)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rec = [r for r in results if r[0] == "rec"][0]
    assert np.max(np.abs(rec[1] - rec[2])) < 1e-12          # partials summed on the root = f
    shards = sorted([r for r in results if r[0] == "planes"], key=lambda r: r[1])
    eta = O.num_shearlets(O.scales_for_size(n))
    owned = sorted(i for s in shards for i in s[2])
    assert owned == list(range(eta))                          # every plane on exactly one rank
    full = np.stack([O.forward(img, variant=variant) for img in rec[2]])
    for _, rank, planes, c in shards:                         # each rank's cube = its planes of the full cube
        assert np.max(np.abs(c - full[:, planes])) < 1e-12
