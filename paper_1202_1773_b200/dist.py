"""eta-sharded FFST across ranks.

Plane i (0-based flat index) is owned by rank i mod G.  forward: the root
broadcasts the images, each rank transforms its planes (the cube stays sharded).
inverse: each rank forms the partial image of its planes, the partials are
summed onto the root (the inverse is linear in the planes,
eq:inverseShearletTransform P:L1730-1764).  Collectives go through
torch.distributed (NCCL on GPUs; gloo in the CPU tests)."""
from __future__ import annotations

import torch
import torch.distributed as dist


def owned_planes(eta: int, rank: int, world: int):
    """Global flat indices owned by `rank` (round robin: every rank gets a mix of scales)."""
    return list(range(rank, eta, world))


class ShardedTransform:
    """Wraps a local per-rank transform (a ``Plan`` created with shard_rank = rank,
    shard_count = world, or any object with ``forward``/``inverse``/``local_planes``)."""

    def __init__(self, local, group=None, root: int = 0):
        self.local = local
        self.group = group
        self.root = root
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    @classmethod
    def create(cls, n: int, batch: int, dtype=torch.float32, device=None, group=None, root: int = 0,
               variant: str = "classic"):
        from .plan import Plan
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        return cls(Plan(n, batch, dtype, device=device, shard_rank=rank, shard_count=world,
                        variant=variant), group, root)

    def forward(self, x):
        """x: images (valid on the root; overwritten by the broadcast elsewhere)."""
        dist.broadcast(x, src=self.root, group=self.group)
        return self.local.forward(x)

    def inverse(self, c, out=None):
        """Partial inverse of the local planes, summed onto the root (valid there)."""
        part = self.local.inverse(c) if out is None else self.local.inverse(c, out=out)
        dist.reduce(part, dst=self.root, op=dist.ReduceOp.SUM, group=self.group)
        return part
