"""Multi-GPU plumbing: H replicated on every rank, candidates / search
chains sharded by contiguous global index ranges, and the per-rank bests combined with
ONE all-reduce(MIN) of a packed 64-bit key plus a broadcast of the winner's x.

Backends: NCCL on GPUs (one process per GPU), gloo for the CPU tests.  Only the
8-byte key and the N-byte winner cross the fabric; H and the batch never do.
"""
from __future__ import annotations

import struct

import numpy as np


def shard(total: int, rank: int, world: int):
    """Contiguous shard [lo, hi) of `total` items for `rank` (first ranks get the remainder)."""
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def owner_of(index: int, total: int, world: int) -> int:
    for r in range(world):
        lo, hi = shard(total, r, world)
        if lo <= index < hi:
            return r
    raise ValueError("index outside [0, total)")


def pack_key(e: float, idx: int) -> int:
    """Signed-orderable (E, idx) key: lexicographic (E, idx) order == int64 order.
    ord(E) maps fp32 bits monotonically onto int32 (-0 canonicalised to +0)."""
    if e != e:
        raise ValueError("NaN energy")
    if e == 0.0:
        e = 0.0
    i = struct.unpack("<i", struct.pack("<f", e))[0]
    if i < 0:
        i ^= 0x7FFFFFFF
    if not 0 <= idx < (1 << 32):
        raise ValueError("index outside [0, 2^32)")
    return i * (1 << 32) + idx


def unpack_key(k: int):
    i, idx = k >> 32, k & 0xFFFFFFFF
    if i < 0:
        i ^= 0x7FFFFFFF
    return struct.unpack("<f", struct.pack("<i", i))[0], idx


def combine_best(e: float, idx: int, device=None, group=None):
    """Global lexicographic min of (E, idx) over the process group: one all-reduce(MIN)."""
    import torch
    import torch.distributed as dist
    key = torch.tensor([pack_key(e, idx)], dtype=torch.int64, device=device)
    dist.all_reduce(key, op=dist.ReduceOp.MIN, group=group)
    return unpack_key(int(key.item()))


def broadcast_x(x: np.ndarray | None, src: int, N: int, device=None, group=None) -> np.ndarray:
    """The winner's bit vector from its owner rank to every rank (N bytes)."""
    import torch
    import torch.distributed as dist
    buf = torch.zeros(N, dtype=torch.uint8, device=device)
    if dist.get_rank(group) == src:
        buf.copy_(torch.from_numpy(np.ascontiguousarray(x, np.uint8)))
    dist.broadcast(buf, src=src, group=group)
    return buf.cpu().numpy()


def search_sharded(t, seed: int, total_chains: int, iters: int, rank: int, world: int, device=None,
                   p0=0.5, p1=0.005):
    """hobo_search over `total_chains` chains sharded across ranks; identical result for any
    world size (each chain's RNG is keyed by its global id)."""
    lo, hi = shard(total_chains, rank, world)
    x, e, c = t.search(seed, total_chains, iters, chain0=lo, nchains=hi - lo, p0=p0, p1=p1)
    ge, gc = combine_best(e, c, device=device)
    xb = broadcast_x(x, owner_of(gc, total_chains, world), t.N, device=device)
    return xb, ge, gc


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
