"""Multi-GPU plumbing: one process per GPU, H replicated on every rank,
candidates / search chains sharded by contiguous global index ranges.  The partition, the
argmin key and the combine are the C library's (include/hobo.h: hobo_shard, hobo_shard_owner,
hobo_best_key; C1 ncclAllReduce(MIN) and C2 ncclBroadcast run inside hobo_energy /
hobo_local_field / hobo_search once hobo_dist_init joined the library's communicator).  This
module only bootstraps that communicator through torch.distributed; it holds no arithmetic.
"""
from __future__ import annotations

from .hobo import shard, shard_owner  # noqa: F401  (re-exported: the library's partition)


def init_library_comm(device_index: int, group=None):
    """Join the C library's own NCCL communicator (hobo_dist_init) using an initialised
    torch.distributed group for the bootstrap: rank 0 creates the 128-byte unique id and
    broadcasts it.  Afterwards every `best` the library returns is already global (C1)
    and hobo_search shards its chains by rank (C1 + C2)."""
    import torch.distributed as dist

    from . import hobo
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [hobo.dist_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    hobo.dist_init(rank, world, obj[0], device_index)
    return rank, world
