"""gloo tests (world size 2-3, CPU) of the eta-sharded path's host logic: the library's plane
map (ffst_shard_planes, LPT and round robin), the image-group schedule of the exchange steps
(broadcast in, reduce out), and that the per-rank partial results sum to the full transform.
The per-rank transform is a stand-in built from the oracle (test infrastructure); on GPUs the
same ShardedTransform wraps the CUDA Plan with the library's own NCCL collectives
(test_gpu_parity.py::test_nccl_single_rank and ::test_shards_sum_to_full)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth


def _load_dist_module():
    # the package loads libffst.so without a GPU (host-only calls: the plane map)
    import paper_1202_1773_b200.dist as D
    return D


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


def _worker(rank, world, port, n, batch, result_q, variant="classic", policy="lpt"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    D = _load_dist_module()
    planes = D.owned_planes(n, rank, world, policy)
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


@pytest.mark.parametrize("world,variant,policy,batch", [(2, "classic", "lpt", 2), (3, "classic", "lpt", 5),
                                                       (2, "smooth", "lpt", 3), (3, "classic", "round_robin", 2)])
def test_sharded_roundtrip_gloo(world, variant, policy, batch):
    n = 32
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + 7 * world + 3 * batch + (50 if variant == "smooth" else 0) \
        + (20 if policy == "round_robin" else 0)
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, batch, q, variant, policy)) for r in range(world)]
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


def test_image_groups_cover_the_batch():
    D = _load_dist_module()
    for batch in (1, 2, 3, 4, 5, 16, 33):
        g = D.image_groups(batch)
        assert len(g) == min(batch, D.COMM_GROUPS)
        assert g[0][0] == 0 and g[-1][1] == batch
        assert all(a[1] == b[0] for a, b in zip(g, g[1:])) and all(b > a for a, b in g)


@pytest.mark.parametrize("n", [64, 256, 1024, 4096])
@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_shard_map_partition_and_balance(n, world):
    # ffst_shard_planes: every plane on exactly one rank (both policies); the LPT map's load (cost
    # n/2 + pruned column count per plane) differs between ranks by at most one plane
    D = _load_dist_module()
    import paper_1202_1773_b200 as F
    eta = O.num_shearlets(O.scales_for_size(n))
    cost = {i: n // 2 + (lambda lh: lh[1] - lh[0] + 1)(F.plane_support(n, i)) for i in range(eta)}
    for policy in ("lpt", "round_robin"):
        sets = [D.owned_planes(n, r, world, policy) for r in range(world)]
        assert sorted(i for s_ in sets for i in s_) == list(range(eta))
        assert all(s_ == sorted(s_) for s_ in sets)
        if policy == "round_robin":
            assert sets == [list(range(r, eta, world)) for r in range(world)]
        else:
            loads = [sum(cost[i] for i in s_) for s_ in sets]
            assert max(loads) - min(loads) <= max(cost.values())
