"""Host-side multi-GPU logic on CPU: world_size-2 gloo process groups exercise the batch
sharding, the packed (E, idx) key, the all-reduce(MIN) combine and the winner broadcast
(paper_2407_19987_b200/dist.py).  The per-rank search results come from the oracle's
replay, so the combined answer must equal the single-process search over all chains."""
import os
import socket
import struct

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2407_19987_b200 import dist as D


def test_shard_covers_range():
    for total in (1, 7, 64, 65536, 100003):
        for world in (1, 2, 3, 8):
            parts = [D.shard(total, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in parts) - min(h - l for l, h in parts) <= 1
            for idx in (0, total - 1, total // 2):
                lo, hi = parts[D.owner_of(idx, total, world)]
                assert lo <= idx < hi


def test_key_orders_lexicographically():
    rng = np.random.default_rng(0)
    vals = np.concatenate([(rng.normal(size=4000) * 10.0 ** rng.integers(-30, 30, 4000)).astype(np.float32),
                           np.array([0.0, -0.0, 1e-45, -1e-45, 3.4e38, -3.4e38, 1.0, -1.0], np.float32)])
    vals = vals.astype(np.float32)
    idx = rng.integers(0, 1 << 32, size=len(vals))
    keys = [D.pack_key(float(e), int(i)) for e, i in zip(vals, idx)]
    order_k = sorted(range(len(vals)), key=lambda j: keys[j])
    canon = [0.0 if v == 0 else float(v) for v in vals]
    order_l = sorted(range(len(vals)), key=lambda j: (canon[j], int(idx[j])))
    assert order_k == order_l
    for k, e, i in zip(keys, canon, idx):
        ee, ii = D.unpack_key(k)
        assert ii == i and struct.pack("<f", ee) == struct.pack("<f", e)
    with pytest.raises(ValueError):
        D.pack_key(float("nan"), 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _OracleShardSearch:
    """Adapter with HoboTensor.search's signature backed by the oracle replay (test only)."""

    def __init__(self, o):
        self.o, self.N = o, o.N

    def search(self, seed, batch, iters, chain0, nchains, p0, p1):
        r = self.o.search(seed, chain0, nchains, iters, p0, p1, nthreads=1)
        c = r["best_chain"]
        return r["chain_xbest"][c - chain0], float(np.float32(r["e_best"])), c


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import Oracle
    from workloads import random_integer_problem, seating
    out = {}
    # (1) combine of per-rank energy minima == global lexicographic min
    o = Oracle.from_problem(seating(4))
    from workloads import x_bits
    total = 1024
    lo, hi = D.shard(total, rank, world)
    E = o.energy(x_bits(1, hi - lo, 16, row0=lo))
    j = int(np.argmin(E))
    out["best"] = D.combine_best(float(E[j]), lo + j)
    # (2) sharded search (oracle-backed shards) == one search over all chains
    p = random_integer_problem(3, 14, 5, nterms=120)
    t = _OracleShardSearch(Oracle.from_problem(p))
    x, e, c = D.search_sharded(t, 7, 97, 6, rank, world)
    out["search"] = (x.tolist(), e, c)
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_combine_and_sharded_search(world):
    from oracle import Oracle
    from workloads import random_integer_problem, seating, x_bits
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process truth
    o = Oracle.from_problem(seating(4))
    E = o.energy(x_bits(1, 1024, 16))
    truth = (float(E.min()), int(np.argmin(E)))
    op = Oracle.from_problem(random_integer_problem(3, 14, 5, nterms=120))
    r = op.search(7, 0, 97, 6)
    for rank in range(world):
        assert res[rank]["best"] == truth
        x, e, c = res[rank]["search"]
        assert (e, c) == (float(np.float32(r["e_best"])), r["best_chain"])
        assert x == r["chain_xbest"][c].tolist()


def test_bench_reference_arm_under_torchrun_world2():
    """The driver's launch of the reference arm at N=2 (torchrun, one process per rank):
    rank 0 alone times the oracle and stdout carries exactly one JSON line; the other rank
    exits 0 without work.  CPU only (the reference arm never touches a GPU)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, NCCL_DEBUG="WARN")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29611", "bench.py", "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "0"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
