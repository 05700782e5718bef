"""Multi-GPU host logic on CPU, through the LIBRARY's own functions (include/hobo.h:
hobo_shard, hobo_shard_owner, hobo_best_key, hobo_best_from_key -- the exact code hobo_search
and the best-combining calls run on every rank).  world_size 2..8 gloo process groups stand in
for the NCCL communicator: the library's C1 is ncclAllReduce(ncclUint64, ncclMin) of the key and
C2 an ncclBroadcast of the winner's bits from the owner rank; here the same two collectives run
over gloo (the unsigned key is biased by 2^63 so that gloo's signed int64 MIN orders it the
same way).  The per-rank results come from the oracle (test infrastructure), so the combined
answer must equal the single-process answer over all items, for every world size, including
ranks whose shard is empty."""
import os
import socket
import struct

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2407_19987_b200 import hobo as H

BIAS = 1 << 63
EMPTY = (1 << 64) - 1          # hobo_best_from_key: no candidate


def test_shard_covers_range_and_owner():
    for total in (0, 1, 5, 7, 64, 65536, 100003):
        for world in (1, 2, 3, 5, 8):
            parts = [H.shard(total, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in parts) - min(h - l for l, h in parts) <= 1
            assert all((h - l) >= (parts[-1][1] - parts[-1][0]) for l, h in parts)   # first ranks take the remainder
            for idx in sorted({0, total - 1, total // 2, total // 3}):
                if 0 <= idx < total:
                    lo, hi = parts[H.shard_owner(total, world, idx)]
                    assert lo <= idx < hi
    with pytest.raises(H.HoboError):
        H.shard_owner(10, 2, 10)
    with pytest.raises(H.HoboError):
        H.shard(10, 2, 2)


def test_key_orders_lexicographically():
    rng = np.random.default_rng(0)
    vals = np.concatenate([(rng.normal(size=4000) * 10.0 ** rng.integers(-30, 30, 4000)).astype(np.float32),
                           np.array([0.0, -0.0, 1e-45, -1e-45, 3.4e38, -3.4e38, 1.0, -1.0, np.inf, -np.inf],
                                    np.float32)])
    idx = rng.integers(0, 1 << 32, size=len(vals))
    keys = [H.best_key(float(e), int(i)) for e, i in zip(vals, idx)]
    order_k = sorted(range(len(vals)), key=lambda j: keys[j])          # unsigned order (ncclUint64 MIN)
    canon = [0.0 if v == 0 else float(v) for v in vals]
    order_l = sorted(range(len(vals)), key=lambda j: (canon[j], int(idx[j])))
    assert order_k == order_l
    for k, e, i in zip(keys, canon, idx):
        ee, ii = H.best_from_key(k)
        assert ii == i and struct.pack("<f", ee) == struct.pack("<f", e)
    assert H.best_from_key(EMPTY) == (float("inf"), -1)
    assert all(k < EMPTY for k in keys)
    with pytest.raises(H.HoboError):
        H.best_key(float("nan"), 0)
    with pytest.raises(H.HoboError):
        H.best_key(1.0, 1 << 32)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allreduce_min_key(key):
    """C1 over gloo: the library's ncclUint64 MIN, on a biased signed int64."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([key - BIAS], dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return int(t.item()) + BIAS


def _broadcast_x(x, src, N):
    """C2 over gloo: the winner's bits from the owner rank."""
    import torch
    import torch.distributed as dist
    buf = torch.zeros(N, dtype=torch.uint8)
    if dist.get_rank() == src:
        buf.copy_(torch.from_numpy(np.ascontiguousarray(x, np.uint8)))
    dist.broadcast(buf, src=src)
    return buf.numpy().copy()


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import Oracle
    from workloads import random_integer_problem, seating, x_bits
    out = {}
    # (1) energies: each rank evaluates its shard, packs its local best with the library key,
    # C1 combines; totals below the world size leave some ranks empty (key ~0)
    o = Oracle.from_problem(seating(4))
    for total in (1024, 5):
        lo, hi = H.shard(total, rank, world)
        key = EMPTY
        if hi > lo:
            E = o.energy(x_bits(1, hi - lo, 16, row0=lo))
            j = int(np.argmin(E))
            key = H.best_key(float(E[j]), lo + j)
        out[f"best{total}"] = H.best_from_key(_allreduce_min_key(key))
    # (2) the hobo_search combine: per-rank chain shards (oracle replay), C1 on (E_best, chain),
    # owner of the winning chain by the library, C2 of its bits
    p = random_integer_problem(3, 14, 5, nterms=120)
    op = Oracle.from_problem(p)
    for total in (97, 3):
        lo, hi = H.shard(total, rank, world)
        key, xs = EMPTY, None
        if hi > lo:
            r = op.search(7, lo, hi - lo, 6, nthreads=1)
            key = H.best_key(float(np.float32(r["e_best"])), r["best_chain"])
            xs = r["chain_xbest"]
        e, c = H.best_from_key(_allreduce_min_key(key))
        owner = H.shard_owner(total, world, c)
        x = _broadcast_x(xs[c - lo] if rank == owner else None, owner, p.N)
        out[f"search{total}"] = (x.tolist(), e, c, owner)
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_gloo_combine_through_library_functions(world):
    from oracle import Oracle
    from workloads import random_integer_problem, seating, x_bits
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process truth
    o = Oracle.from_problem(seating(4))
    op = Oracle.from_problem(random_integer_problem(3, 14, 5, nterms=120))
    for total in (1024, 5):
        E = o.energy(x_bits(1, total, 16))
        truth = (float(E.min()), int(np.argmin(E)))
        assert all(res[r][f"best{total}"] == truth for r in range(world)), total
    for total in (97, 3):
        r = op.search(7, 0, total, 6)
        for rank in range(world):
            x, e, c, owner = res[rank][f"search{total}"]
            assert (e, c) == (float(np.float32(r["e_best"])), r["best_chain"])
            assert x == r["chain_xbest"][c].tolist()
            lo, hi = H.shard(total, owner, world)
            assert lo <= c < hi


def test_bench_reference_arm_under_torchrun_world2():
    """The driver's launch of the reference arm at N=2 (torchrun, one process per rank):
    rank 0 alone times the oracle and stdout carries exactly one JSON line; the other rank
    exits 0 without work.  CPU only (the reference arm never touches a GPU)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, NCCL_DEBUG="WARN")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--impl",
                        "reference", "--gpus", "2", "--steps", "1", "--warmup", "0"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
