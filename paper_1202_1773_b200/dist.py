"""eta-sharded FFST across ranks.

The planes are dealt to the ranks by ``shard_planes`` (cost-balanced LPT by default, SURVEY 8(e):
cost n/2 + pruned column count).  The transform has one exchange step per direction:

* forward: the images are broadcast from rank 0; each rank transforms its planes and keeps its
  slice of the cube on its device;
* inverse: the inverse is linear in the planes (eq:inverseShearletTransform), so
  each rank forms the partial adjoint spectrum of its planes and the partials are summed onto
  the root, which alone runs the final synthesis.

On GPUs the exchange steps run inside the library (``Plan(nccl_comm=...)``): an NCCL
communicator created through the C ABI, collectives on a plan-owned stream, chunked by image
groups so that they overlap the kernels.  ``ShardedTransform`` sets that up from a
torch.distributed process group (used here only to hand the NCCL unique id to every rank).
With a non-NCCL group (the gloo CPU tests) it runs the same schedule with torch collectives
around a local stand-in transform.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .plan import NcclComm, Plan, shard_planes

COMM_GROUPS = 4   # image groups of the exchange steps (include/ffst.h; ffst_api.cu COMM_GROUPS)


def owned_planes(n: int, rank: int, world: int, policy: str = "lpt"):
    """Global flat indices (0-based) owned by `rank` (ffst_shard_planes)."""
    return shard_planes(n, world, rank, policy)


def image_groups(batch: int, groups: int = COMM_GROUPS):
    """[g0, g1) image ranges of the chunked exchange steps (the library's schedule)."""
    g = min(batch, groups)
    return [(batch * i // g, batch * (i + 1) // g) for i in range(g)]


def create_comm(group=None, device=None) -> NcclComm:
    """One NCCL communicator over the ranks of a torch.distributed group, created through the
    C ABI: rank 0 draws the unique id, the group broadcasts it."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [NcclComm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    dev = torch.cuda.current_device() if device is None else torch.device(device).index
    return NcclComm(world, rank, dev, obj[0])


class ShardedTransform:
    """The eta-sharded transform on the ranks of a process group.

    ``local`` is this rank's transform: a ``Plan`` created with shard_rank = rank, shard_count =
    world (and, on GPUs, nccl_comm: the library runs the exchange steps), or any object with
    ``forward``/``inverse`` (the CPU tests' stand-in; the exchange then uses torch collectives
    with the same image-group schedule)."""

    def __init__(self, local, group=None, root: int = 0):
        self.local = local
        self.group = group
        self.root = root
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.in_library = getattr(local, "comm", None) is not None

    @classmethod
    def create(cls, n: int, batch: int, dtype=torch.float32, device=None, group=None, root: int = 0,
               variant: str = "classic", shard_policy: str = "lpt"):
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        comm = create_comm(group, device) if dist.get_backend(group) == "nccl" else None
        plan = Plan(n, batch, dtype, device=device, shard_rank=rank, shard_count=world, variant=variant,
                    shard_policy=shard_policy, nccl_comm=comm)
        return cls(plan, group, root)

    def forward(self, x, out=None):
        """x: images on rank 0 (ignored elsewhere; may be None there in library mode)."""
        if self.in_library:
            return self.local.forward(x if self.rank == 0 else None, out=out,
                                      batch=None if x is None else x.shape[0])
        for g0, g1 in image_groups(x.shape[0]):
            dist.broadcast(x[g0:g1], src=0, group=self.group)
        return self.local.forward(x) if out is None else self.local.forward(x, out=out)

    def inverse(self, c, out=None):
        """The full inverse on `root` (partial images summed there)."""
        if self.in_library:
            return self.local.inverse(c, out=out, root=self.root)
        part = self.local.inverse(c) if out is None else self.local.inverse(c, out=out)
        for g0, g1 in image_groups(part.shape[0]):
            dist.reduce(part[g0:g1], dst=self.root, op=dist.ReduceOp.SUM, group=self.group)
        return part
