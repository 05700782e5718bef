"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs.  Bars (BASELINE.json north_star): bit-exact on integer-coefficient instances;
|dE|, |dG| <= tau = 1e-5 * sum|H| for fp32 coefficients; argmin exact when the energy gap
exceeds 2 tau (reading 11), else the returned candidate is within 2 tau."""
import contextlib
import os

import numpy as np
import pytest

from oracle import Oracle
from workloads import (cfg3_problem, exhaustive_X, h, int_twin_cells, paper_grids, pythagoras,
                       random_integer_problem, seating, tsp, uniform_cells, x_bits)
from workloads.gen import canonical_cells_all, int_encoded_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as _t
    assert _t.cuda.is_available(), "GPU tests need a CUDA device"
    return _t


@pytest.fixture(scope="module")
def H():
    from paper_2407_19987_b200 import build
    build.build()
    from paper_2407_19987_b200 import hobo
    return hobo


def dev(torch, X):
    return torch.from_numpy(np.ascontiguousarray(X, np.uint8)).cuda()


def energies(H, torch, t, X, row0=0):
    E, best = t.energy(dev(torch, X), row0=row0)
    torch.cuda.synchronize()
    return E.cpu().numpy().astype(np.float64), best


def fields(H, torch, t, X):
    G, E = t.local_field(dev(torch, X))
    torch.cuda.synchronize()
    return G.cpu().numpy().astype(np.float64), E.cpu().numpy().astype(np.float64)


@contextlib.contextmanager
def env(name, value):
    """Set a kernel-choice override (include/hobo.h) for the tensors built inside the block."""
    old = os.environ.get(name)
    os.environ[name] = value
    try:
        yield
    finally:
        if old is None:
            del os.environ[name]
        else:
            os.environ[name] = old


def f32(a):
    """The oracle's exact (long double) values rounded once to fp32, as float64."""
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


def check_argmin(best, E_or, tau, row0=0):
    order = np.argsort(E_or, kind="stable")
    e1 = E_or[order[0]]
    nxt = E_or[E_or > e1]
    gap = (nxt.min() - e1) if nxt.size else np.inf
    if gap > 2 * tau:
        assert best[1] == row0 + int(np.flatnonzero(E_or == e1)[0])
    else:
        assert E_or[best[1] - row0] <= e1 + 2 * tau


# ---- energies on integer instances: bit-exact ---------------------------------------------
def test_energy_seating4_exhaustive(H, torch):
    p = seating(4)
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    X = exhaustive_X(16)
    E, best = energies(H, torch, t, X)
    assert np.array_equal(E, o.energy(X))
    assert best == (-11.0, 46811)


def test_energy_cfg1(H, torch):
    p = seating(4)
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    X = x_bits(1, 1024, 16)
    E, best = energies(H, torch, t, X)
    assert np.array_equal(E, o.energy(X)) and best == (-10.0, 551)


def test_energy_paper_problems(H, torch):
    t = H.HoboTensor.from_problem(seating(5))
    E, _ = energies(H, torch, t, paper_grids())
    assert np.all(E == -17.0)
    for p, emin, arg in ((pythagoras(), -30.0, 1332), (tsp(), -360.0, 27)):
        t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
        X = exhaustive_X(p.N)
        E, best = energies(H, torch, t, X)
        assert np.array_equal(E, o.energy(X)), p.name
        assert best == (emin, arg), p.name


def test_energy_seating5_full_space(H, torch):
    """2^25 candidates in one batch: min -17 at the lowest ground-state index."""
    t = H.HoboTensor.from_problem(seating(5))
    b = torch.arange(1 << 25, device="cuda", dtype=torch.int64)[:, None]
    X = ((b >> torch.arange(25, device="cuda")[None, :]) & 1).to(torch.uint8).contiguous()
    E, best = t.energy(X)
    torch.cuda.synchronize()
    assert best == (-17.0, 14539195)
    assert int((E == -17.0).sum()) == 5


@pytest.mark.parametrize("order,N,B,seed", [(1, 37, 129, 1), (2, 100, 1000, 2), (3, 33, 127, 3), (3, 100, 300, 4),
                                            (3, 257, 130, 5), (4, 40, 200, 6), (5, 14, 256, 7), (6, 9, 100, 8),
                                            (2, 1, 5, 9), (3, 3, 1, 10)])
def test_energy_integer_dense(H, torch, order, N, B, seed):
    if order <= 4 and N >= 20:
        idx, val = int_twin_cells(order, N, seed)
        t, o = H.HoboTensor.import_cells(order, N, idx, val), Oracle.from_cells(order, N, idx, val)
    else:
        p = random_integer_problem(order, N, seed, nterms=300)
        t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    X = x_bits(seed, B, N)
    E, best = energies(H, torch, t, X, row0=7)
    Eo = o.energy(X)
    assert np.array_equal(E, Eo)
    check_argmin(best, Eo, 0.0, row0=7)


# ---- fp32 coefficients: tolerance -----------------------------------------------------------
@pytest.mark.parametrize("order,N,B,seed", [(2, 300, 700, 11), (3, 130, 500, 12), (3, 256, 256, 13), (4, 30, 300, 14)])
def test_energy_fp32(H, torch, order, N, B, seed):
    idx, val = uniform_cells(order, N, seed)
    t, o = H.HoboTensor.import_cells(order, N, idx, val), Oracle.from_cells(order, N, idx, val)
    assert t.limbs == 3
    X = x_bits(seed, B, N)
    E, best = energies(H, torch, t, X)
    Eo = o.energy(X)
    assert np.max(np.abs(E - Eo)) <= o.tau
    check_argmin(best, Eo, o.tau)


# ---- local fields ---------------------------------------------------------------------------
@pytest.mark.parametrize("order,N,B,seed", [(1, 40, 64, 1), (2, 70, 300, 2), (3, 50, 200, 3), (3, 300, 129, 4),
                                            (4, 24, 150, 5), (5, 12, 100, 6), (6, 8, 64, 7)])
def test_field_integer(H, torch, order, N, B, seed):
    p = random_integer_problem(order, N, seed, nterms=400)
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    X = x_bits(seed, B, N)
    G, E = fields(H, torch, t, X)
    assert np.array_equal(G, o.field(X))
    assert np.array_equal(E, o.energy(X))


def test_field_paper_problems(H, torch):
    for p in (seating(4), pythagoras(), tsp()):
        t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
        X = exhaustive_X(p.N)
        G, E = fields(H, torch, t, X)
        assert np.array_equal(G, o.field(X)), p.name
        assert np.array_equal(E, o.energy(X)), p.name


@pytest.mark.parametrize("order,N,B,seed", [(2, 260, 300, 21), (3, 100, 257, 22), (4, 20, 130, 23)])
def test_field_fp32(H, torch, order, N, B, seed):
    idx, val = uniform_cells(order, N, seed)
    t, o = H.HoboTensor.import_cells(order, N, idx, val), Oracle.from_cells(order, N, idx, val)
    X = x_bits(seed, B, N)
    G, E = fields(H, torch, t, X)
    assert np.max(np.abs(G - o.field(X))) <= o.tau
    assert np.max(np.abs(E - o.energy(X))) <= o.tau


# ---- full-size configs, sampled -------------------------------------------------------------
# Rows are sampled with a stride co-prime to 128 (the candidate block = TMEM lanes): row
# r_i = i * stride covers every TMEM lane (r mod 128) and both CTAs of a pair (r // 128 odd and
# even), plus the last row of the batch.
def sample_rows(B, stride, n=None):
    assert np.gcd(stride, 128) == 1
    rows = np.arange(0, B, stride)[:n]
    return np.unique(np.concatenate([rows, [B - 1]]))


def assert_lanes_covered(rows, B):
    if B >= 4 * 128:
        assert len(set((rows % 128).tolist())) == 128 or len(rows) < 128
        assert {0, 1} <= set(((rows // 128) % 2).tolist())


def test_cfg3_full_batch(H, torch):
    """BASELINE config 3 at its full size (B=65536) in the bench's launch configuration.
    Energies of ALL 65,536 candidates and the full-batch argmin equal the oracle's (integer
    instance: bit-exact, lowest index on ties); fields of 256 rows spread over every TMEM lane
    and both CTAs of each pair equal the oracle's."""
    p = cfg3_problem()
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    B = 65536
    X = x_bits(3, B, 512)
    G, E = fields(H, torch, t, X)
    rows = sample_rows(B, 257)
    assert_lanes_covered(rows, B)
    assert np.array_equal(G[rows], o.field(X[rows]))
    Eo = o.energy(X)                                   # the whole batch (~8 s on 16 cores)
    assert np.array_equal(E, Eo)
    Ee, best = energies(H, torch, t, X)
    assert np.array_equal(Ee, Eo)                      # energy mode == field mode == oracle
    assert best == (Eo.min(), int(np.argmin(Eo)))      # np.argmin: the lowest index on ties


def test_cfg2_full_batch(H, torch):
    """BASELINE config 2: QUBO N=1024 U(-1,1), B=65536.  Every energy against the float64
    closed form x^T Q x (numpy matmul over the oracle's dense Q), the full-batch argmin against
    it (reading 11: exact when the gap exceeds 2 tau), and 256 strided rows against the oracle."""
    idx, val = uniform_cells(2, 1024, 2)
    t, o = H.HoboTensor.import_cells(2, 1024, idx, val), Oracle.from_cells(2, 1024, idx, val)
    B = 65536
    X = x_bits(2, B, 1024)
    E, best = energies(H, torch, t, X)
    Q = o.dense().astype(np.float64)
    ref = np.empty(B)
    for lo in range(0, B, 8192):
        Xc = X[lo:lo + 8192].astype(np.float64)
        ref[lo:lo + 8192] = np.einsum("bi,bi->b", Xc @ Q, Xc)
    assert np.max(np.abs(E - ref)) <= o.tau
    check_argmin(best, ref, o.tau)
    rows = sample_rows(B, 257)
    assert_lanes_covered(rows, B)
    assert np.max(np.abs(E[rows] - o.energy(X[rows]))) <= o.tau
    assert np.allclose(E[:4], [225.87784564495087, 211.0458381175995, 31.37024474143982, 149.2058583498001],
                       rtol=0, atol=o.tau)


# ---- search ---------------------------------------------------------------------------------
def test_search_finds_brute_force_optimum(H, torch):
    for p, emin, nch, it in ((seating(4), -11.0, 1024, 64), (pythagoras(), -30.0, 2048, 64), (tsp(), -360.0, 256, 32)):
        t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
        x, e, c = t.search(1, nch, it)
        assert e == emin, p.name
        assert o.energy(x[None])[0] == e, p.name          # energy honesty


def test_search_replays_oracle_exactly(H, torch):
    """Integer instance: the device search and the oracle replay agree chain for chain."""
    p = random_integer_problem(3, 40, 77, nterms=500)
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    for chain0, n, iters in ((0, 300, 20), (1000, 129, 7), (5, 1, 0)):
        x, e, c = t.search(9, None, iters, chain0=chain0, nchains=n)
        r = o.search(9, chain0, n, iters)
        assert (e, c) == (r["e_best"], r["best_chain"])
        assert np.array_equal(x, r["chain_xbest"][c - chain0])


def test_search_graph_replay(H, torch):
    """The search loop runs as one CUDA graph per (chains, iterations, buffers) with seed, chain0
    and the P_t table in device memory: replays with other seeds / shards / schedules equal the
    directly launched loop (HOBO_GRAPH=0) and the oracle."""
    p = random_integer_problem(3, 40, 78, nterms=500)
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    runs = [(9, 0, 200, 12, 0.5, 0.005), (10, 0, 200, 12, 0.5, 0.005), (11, 300, 200, 12, 0.3, 0.01),
            (9, 0, 200, 12, 0.5, 0.005), (12, 7, 64, 3, 0.5, 0.005), (12, 7, 64, 3, 0.5, 0.005)]
    for seed, c0, n, it, p0, p1 in runs:
        x, e, c = t.search(seed, None, it, chain0=c0, nchains=n, p0=p0, p1=p1)
        with env("HOBO_GRAPH", "0"):
            x0, e0, c0_ = t.search(seed, None, it, chain0=c0, nchains=n, p0=p0, p1=p1)
        r = o.search(seed, c0, n, it, p0, p1)
        assert (e, c) == (e0, c0_) == (r["e_best"], r["best_chain"]) and np.array_equal(x, x0)
        assert np.array_equal(x, r["chain_xbest"][c - c0])


@pytest.mark.parametrize("case", ["cfg3_small", "qubo_persist", "splitk"])
def test_call_graph_replay(H, torch, case):
    """Energy / field calls replay a captured CUDA graph when the same call repeats (same
    buffers and batch): new candidate contents in the same buffers, profiling on and off, the
    per-tile, persistent and split-K paths -- all equal to direct launches (HOBO_GRAPH=0) and
    to the oracle."""
    if case == "cfg3_small":
        p = cfg3_problem()
        t, o, B = H.HoboTensor.from_problem(p), Oracle.from_problem(p), 3000
    elif case == "qubo_persist":
        idx, val = int_twin_cells(2, 1024, 61)
        t, o, B = H.HoboTensor.import_cells(2, 1024, idx, val), Oracle.from_cells(2, 1024, idx, val), 20000
    else:
        p = random_integer_problem(3, 200, 62, nterms=800)
        t, o, B = H.HoboTensor.from_problem(p), Oracle.from_problem(p), 40
    Xd = torch.empty(B, t.N, dtype=torch.uint8, device="cuda")
    G = torch.empty(B, t.N, dtype=torch.float32, device="cuda")
    E = torch.empty(B, dtype=torch.float32, device="cuda")
    for rep, seed in enumerate((71, 72, 73, 71)):
        X = x_bits(seed, B, t.N)
        Xd.copy_(torch.from_numpy(X))
        t.set_profiling(rep == 2)
        _, be = t.energy(Xd, E, row0=5)
        Ee = E.cpu().numpy().astype(np.float64)
        t.local_field(Xd, G, E, row0=5)
        Gf, Ef = G.cpu().numpy().astype(np.float64), E.cpu().numpy().astype(np.float64)
        if rep == 2:
            assert t.launch_stats()["kernel_ms"] > 0
        with env("HOBO_GRAPH", "0"):
            E0, b0 = t.energy(Xd, row0=5)
            G0, E1 = t.local_field(Xd, row0=5)
        assert np.array_equal(Ee, E0.cpu().numpy()) and be == b0
        assert np.array_equal(Gf, G0.cpu().numpy()) and np.array_equal(Ef, E1.cpu().numpy())
        rows = sample_rows(B, 37, 40)
        assert np.array_equal(Ee[rows], o.energy(X[rows])) and np.array_equal(Gf[rows], o.field(X[rows]))
    t.set_profiling(False)


def test_search_shard_invariance(H, torch):
    p = seating(4)
    t = H.HoboTensor.from_problem(p)
    full = t.search(3, 512, 16)
    a = t.search(3, None, 16, chain0=0, nchains=256)
    b = t.search(3, None, 16, chain0=256, nchains=256)
    win = min((a[1], a[2], 0), (b[1], b[2], 1))
    assert (full[1], full[2]) == win[:2]


# ---- remaining BASELINE configs at full size, sampled ----------------------------------------
# cfg3-fp32, cfg4 and cfg5 take the int8 digit-plane path (reading 24): the contraction
# is exact integer arithmetic rounded once, so energies and fields must EQUAL the oracle's exact
# (long double) values rounded once to fp32 -- not merely lie within tau.
def test_cfg5_full_batch_sampled(H, torch):
    """BASELINE config 5 at one GPU's full size: order 3, N=1024, all 178,957,824 canonical
    cells U(-1,1), B = 2^20 candidates, energies + argmin in the energy-mode layout (int8).
    Strided rows (every TMEM lane, both CTAs of a pair) equal fp32(oracle); the 16 lowest
    energies of the batch (the argmin among them) are re-evaluated by the oracle."""
    from oracle import colex_energy
    from workloads import uniform_colex
    N, B = 1024, 1 << 20
    v = uniform_colex(3, N, 5)
    t = H.HoboTensor.import_colex(3, N, v)
    # 178,957,824 canonical cells; the U(-1,1) draw hits exactly 0 for ~2^-24 of them
    assert t.limbs == 3 and t.ncells == sum(int(np.count_nonzero(a)) for a in v)
    assert sum(a.size for a in v) == 178957824
    Xd = torch.empty(B, N, dtype=torch.uint8, device="cuda")
    for lo in range(0, B, 1 << 17):
        Xd[lo:lo + (1 << 17)] = torch.from_numpy(x_bits(5, 1 << 17, N, row0=lo)).cuda()
    E, best = t.energy(Xd)
    torch.cuda.synchronize()
    assert t.launch_stats()["i8_planes"] == 3
    Eh = E.cpu().numpy().astype(np.float64)
    rows = sample_rows(B, 16411, 48)
    low = np.argsort(Eh, kind="stable")[:16]
    rows = np.unique(np.concatenate([rows, low]))
    Xs = Xd[torch.from_numpy(rows).cuda()].cpu().numpy()
    ref = colex_energy(3, N, v, Xs)
    assert np.array_equal(Eh[rows], f32(ref))
    assert best == (Eh.min(), int(np.argmin(Eh))) and best[1] == int(low[0])


def test_cfg4_full_batch_sampled(H, torch):
    """BASELINE config 4: order 4, N=128, all canonical cells U(-1,1), B=262,144 (int8):
    local fields + energies at full size; 64 strided rows (every lane class, both CTAs) and the
    argmin row equal fp32(oracle)."""
    from oracle import colex_energy, colex_field
    from workloads import uniform_colex
    N, B = 128, 262144
    v = uniform_colex(4, N, 4)
    t = H.HoboTensor.import_colex(4, N, v)
    X = x_bits(4, B, N)
    Xd = dev(torch, X)
    G, E, best = t.local_field(Xd, want_best=True)
    torch.cuda.synchronize()
    assert t.launch_stats()["i8_planes"] == 3
    G, E = G.cpu().numpy().astype(np.float64), E.cpu().numpy().astype(np.float64)
    rows = np.unique(np.concatenate([sample_rows(B, 4099, 64), [best[1]]]))
    assert np.array_equal(E[rows], f32(colex_energy(4, N, v, X[rows])))
    assert np.array_equal(G[rows], f32(colex_field(4, N, v, X[rows])))
    assert best == (E.min(), int(np.argmin(E)))


def test_cfg3_fp32_companion_sampled(H, torch):
    """cfg3-fp32: order 3, N=512, all 22,370,048 canonical cells U(-1,1), B=65,536 (int8):
    256 strided rows equal fp32(oracle) in energy and field; the argmin row too."""
    from oracle import colex_energy, colex_field
    from workloads import uniform_colex
    N, B = 512, 65536
    v = uniform_colex(3, N, 3)
    t = H.HoboTensor.import_colex(3, N, v)
    X = x_bits(3, B, N)
    G, E, best = t.local_field(dev(torch, X), want_best=True)
    torch.cuda.synchronize()
    assert t.launch_stats()["i8_planes"] == 3
    G, E = G.cpu().numpy().astype(np.float64), E.cpu().numpy().astype(np.float64)
    rows = np.unique(np.concatenate([sample_rows(B, 257), [best[1]]]))
    assert_lanes_covered(rows, B)
    assert np.array_equal(E[rows], f32(colex_energy(3, N, v, X[rows])))
    assert np.array_equal(G[rows], f32(colex_field(3, N, v, X[rows])))
    assert best == (E.min(), int(np.argmin(E)))


# ---- the persistent energy kernel (persist.cuh): short K loops, double-buffered accumulators ----
@pytest.mark.parametrize("i8", ["1", "0"])
@pytest.mark.parametrize("case", ["int_qubo", "int_o3", "fp32_qubo", "int_qubo_words"])
def test_persistent_energy_kernel(H, torch, case, i8):
    """The persistent energy kernels (HOBO_PERSIST=1; the default for cfg2-like tiles): int8 digit
    planes (kr_persist_i8_kernel, exact: energies equal fp32(oracle)) and bf16 limbs
    (kr_persist_kernel, HOBO_PERSIST_I8=0: within tau, exact on integer instances), against the
    oracle and the per-tile kernel (HOBO_PERSIST=0), at batches giving odd candidate-block counts,
    ragged blocks, fewer items than CTA pairs and several candidate blocks per pair."""
    if case == "int_qubo":
        idx, val = int_twin_cells(2, 300, 51)
        t, o = H.HoboTensor.import_cells(2, 300, idx, val), Oracle.from_cells(2, 300, idx, val)
    elif case == "int_o3":
        p = random_integer_problem(3, 70, 52, nterms=900)
        t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    elif case == "fp32_qubo":
        idx, val = uniform_cells(2, 520, 53)
        t, o = H.HoboTensor.import_cells(2, 520, idx, val), Oracle.from_cells(2, 520, idx, val)
    else:   # whole 32-bit rows (the vectorised pack kernel feeds the persistent one)
        idx, val = int_twin_cells(2, 256, 55)
        t, o = H.HoboTensor.import_cells(2, 256, idx, val), Oracle.from_cells(2, 256, idx, val)
    for B in (1, 129, 300, 5000, 40000):
        X = x_bits(54, B, t.N)
        with env("HOBO_PERSIST", "1"), env("HOBO_PERSIST_I8", i8):
            E1, b1 = energies(H, torch, t, X, row0=3)
            kind = t.launch_stats()["i8_planes"]
        with env("HOBO_PERSIST", "0"):
            E0, b0 = energies(H, torch, t, X, row0=3)
        assert (kind > 0) == (i8 == "1")
        rows = np.arange(B) if B <= 5000 else sample_rows(B, 129)
        Eo = o.energy(X[rows])
        if t.is_integer or kind:
            assert np.array_equal(E1[rows], f32(Eo)), B
        else:
            assert np.max(np.abs(E1[rows] - Eo)) <= o.tau, B
        if t.is_integer:
            assert np.array_equal(E1, E0) and b1 == b0, B
        else:
            assert np.max(np.abs(E1 - E0)) <= 2 * o.tau, B
        check_argmin(b1, E1, 0.0, row0=3)


# ---- stream-K (CTA-pair field launches: whole waves in place, the leftover tiles split) ------
@pytest.mark.parametrize("case", ["int_cfg3", "fp32_bf16"])
def test_stream_k_matches_data_parallel(H, torch, case):
    """The stream-K schedule (leftover tiles cut into 74 equal K ranges, partials summed in K
    order) against the plain one-tile-per-pair launch (HOBO_SK=0) and the oracle: 8,192
    candidates (one GPU's share at 8 GPUs: every tile split), 20,000 (two whole waves + 10
    split tiles) and 65,536 (cfg3's launch: 6 waves + 68 leftover tiles, which the schedule now
    leaves data-parallel: a 92%-full leftover wave gains less than its partial sums cost)."""
    if case == "int_cfg3":
        p = cfg3_problem()
        t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
        sizes = (8192, 20000, 65536)
    else:
        idx, val = uniform_cells(3, 300, 81)
        t = H.HoboTensor.import_cells(3, 300, idx, val)     # HOBO_I8=0 below: the bf16 limbs (L = 3)
        o = Oracle.from_cells(3, 300, idx, val)
        sizes = (8192, 20000)
    for B in sizes:
        X = x_bits(82, B, t.N)
        Xd = dev(torch, X)
        with env("HOBO_I8", "0"):
            G1, E1, b1 = t.local_field(Xd, row0=9, want_best=True)
            with env("HOBO_SK", "0"):
                G0, E0, b0 = t.local_field(Xd, row0=9, want_best=True)
        torch.cuda.synchronize()
        G1, E1, G0, E0 = (a.cpu().numpy().astype(np.float64) for a in (G1, E1, G0, E0))
        rows = sample_rows(B, 257, 64)
        Go, Eo = o.field(X[rows]), o.energy(X[rows])
        if t.is_integer:
            assert np.array_equal(G1, G0) and np.array_equal(E1, E0) and b1 == b0, B
            assert np.array_equal(G1[rows], Go) and np.array_equal(E1[rows], Eo), B
        else:
            assert np.max(np.abs(G1[rows] - Go)) <= o.tau and np.max(np.abs(E1[rows] - Eo)) <= o.tau, B
            assert np.max(np.abs(G1 - G0)) <= 2 * o.tau and np.max(np.abs(E1 - E0)) <= 2 * o.tau, B


# ---- split-K (small batches) -----------------------------------------------------------------
@pytest.mark.parametrize("B", [1, 16, 200])
def test_small_batch_split_k_matches(H, torch, B):
    """Small batches split the K schedule across CTAs (HBM-bound regime); on an integer
    instance the fields and energies are bit-identical to the unsplit full-batch run and to
    the oracle."""
    p = cfg3_problem()
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    X = x_bits(3, B, 512)
    G, E = fields(H, torch, t, X)
    assert np.array_equal(G, o.field(X)) and np.array_equal(E, o.energy(X))
    Ee, best = energies(H, torch, t, X)
    assert np.array_equal(Ee, E) and best == (E.min(), int(np.argmin(E)))


def test_small_batch_split_k_fp32(H, torch):
    idx, val = uniform_cells(3, 300, 41)
    t, o = H.HoboTensor.import_cells(3, 300, idx, val), Oracle.from_cells(3, 300, idx, val)
    X = x_bits(41, 37, 300)
    G, E = fields(H, torch, t, X)
    assert np.max(np.abs(G - o.field(X))) <= o.tau and np.max(np.abs(E - o.energy(X))) <= o.tau
    Ee, _ = energies(H, torch, t, X)
    assert np.max(np.abs(Ee - o.energy(X))) <= o.tau


# ---- result aggregation (the paper's Energy / Occurrence listing) ---------------------------
@pytest.mark.parametrize("name,batch,iters,topk", [("seating4", 1024, 16, 8), ("pythagoras", 3000, 24, 10),
                                                   ("tsp", 2000, 6, 6), ("rand", 5000, 9, 50)])
def test_search_samples_match_oracle(H, torch, name, batch, iters, topk):
    from oracle import aggregate
    p = {"seating4": seating(4), "pythagoras": pythagoras(), "tsp": tsp(),
         "rand": random_integer_problem(3, 18, 4, nterms=200)}[name]
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    got = t.search_samples(7, batch, iters, topk)
    r = o.search(7, 0, batch, iters)
    want = aggregate(r["chain_xbest"], r["chain_ebest"], topk)
    assert len(got) == len(want)
    for (gx, ge, gc), (wx, we, wc) in zip(got, want):
        assert np.array_equal(gx, wx) and ge == we and gc == wc


# ---- multilinear relaxation at real p (gradient descent's hot path) --------------------------
def _p_bf16(torch, seed, B, N):
    u = ((h(seed, 3, np.arange(B, dtype=np.uint64)[:, None], np.arange(N, dtype=np.uint64)[None, :]) >> np.uint64(40))
         .astype(np.float64) * 2.0 ** -24)
    Pd = torch.from_numpy(u.astype(np.float32)).cuda().to(torch.bfloat16).contiguous()
    return Pd, Pd.float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("kind,order,N,B,seed", [("int", 3, 40, 300, 1), ("int", 2, 100, 129, 2), ("int", 4, 20, 200, 3),
                                                 ("u", 3, 130, 257, 4), ("u", 3, 512, 64, 5), ("u", 2, 300, 500, 6),
                                                 ("cfg3", 3, 512, 1000, 7), ("int", 3, 37, 131, 8)])   # odd N
def test_multilinear_field(H, torch, kind, order, N, B, seed):
    from workloads import h  # noqa: F401
    if kind == "int":
        p = random_integer_problem(order, N, seed, nterms=300)
        t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    elif kind == "cfg3":
        p = cfg3_problem()
        t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    else:
        idx, val = uniform_cells(order, N, seed)
        t, o = H.HoboTensor.import_cells(order, N, idx, val), Oracle.from_cells(order, N, idx, val)
    Pd, P = _p_bf16(torch, seed, B, N)
    G, E = t.multilinear_field(Pd)   # N=512 at L=3 runs on the 128-column-tile layout
    torch.cuda.synchronize()
    Gr, Er = o.mfield(P), o.menergy(P)
    assert np.max(np.abs(G.cpu().numpy() - Gr)) <= o.tau
    assert np.max(np.abs(E.cpu().numpy() - Er)) <= o.tau


def test_multilinear_field_binary_points_exact(H, torch):
    """At p in {0,1} the relaxation is the binary field: bit-exact on an integer instance."""
    p = random_integer_problem(3, 60, 9, nterms=400)
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    X = x_bits(9, 200, 60)
    G, E = t.multilinear_field(torch.from_numpy(X).cuda().to(torch.bfloat16))
    torch.cuda.synchronize()
    assert np.array_equal(G.cpu().numpy().astype(np.float64), o.field(X))
    assert np.array_equal(E.cpu().numpy().astype(np.float64), o.energy(X))


# ---- gradient descent: quality and honesty of the returned states -------------
@pytest.mark.parametrize("name,shots,steps,eta", [("tsp", 2000, 30, 0.05), ("seating4", 2000, 30, 0.2),
                                                  ("pythagoras", 4000, 40, 1e-4), ("rand", 1000, 20, 0.05)])
def test_gd_run(H, torch, name, shots, steps, eta):
    p = {"seating4": seating(4), "pythagoras": pythagoras(), "tsp": tsp(),
         "rand": random_integer_problem(3, 18, 4, nterms=200)}[name]
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    res = t.gd_run(11, shots, steps, eta, topk=20)
    assert 1 <= len(res) <= 20 and sum(c for _, _, c in res) <= shots
    X = np.stack([x for x, _, _ in res])
    E = o.energy(X)
    assert np.array_equal(E, np.array([e for _, e, _ in res], np.float64))       # honest energies
    G = o.field(X)
    assert np.all((1 - 2 * X.astype(np.float64)) * G >= 0)                          # greedy local minima
    assert list(E) == sorted(E)
    assert E[0] == o.brute()["emin"]                                                # finds the optimum


# ---- Tensor-Train form ---------------------------------------------------
@pytest.mark.parametrize("name", ["tsp", "seating4", "pythagoras", "rand"])
def test_tt_energy(H, torch, name):
    p = {"tsp": tsp(), "seating4": seating(4), "pythagoras": pythagoras(),
         "rand": random_integer_problem(3, 10, 3, nterms=60)}[name]
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    t.tt_build(0.0)
    X = exhaustive_X(p.N)
    E, best = t.tt_energy(dev(torch, X))
    torch.cuda.synchronize()
    Eo = o.energy(X)
    assert np.max(np.abs(E.cpu().numpy().astype(np.float64) - Eo)) <= o.tau
    check_argmin(best, Eo, o.tau)


# ---- simulated annealing (SPEC sa_run S:447-453) -------------------------
def _linear_problem():
    from workloads import TermBuilder
    tb = TermBuilder()
    for m, c in enumerate([3, -2, 0, 5, -7, 1, 2, -1, 4]):
        if c:
            tb.add(float(c), [(0.0, [(m, 1.0)])])
    return tb.problem(1, 9)


def _wide_int_problem(N=200, seed=36):
    """Integer cells needing 3 bf16 limbs (a 3-box W stream per K-block) at N in (128, 256]."""
    from workloads import TermBuilder
    rng = np.random.default_rng(seed)
    tb = TermBuilder()
    for i in range(600):
        r = int(rng.integers(1, 4))
        vs = rng.choice(N, size=r, replace=False)
        # 262657 = 2^18 + 2^9 + 1: hi = 2^18, mid = 2^9, lo = 1 -> three bf16 limbs
        c = float(rng.integers(-9, 10)) if i % 50 else float(rng.choice([-1, 1]) * 262657)
        tb.add(c, [(0.0, [(int(v), 1.0)]) for v in vs])
    return tb.problem(3, N)


SA_CASES = {
    "seating4": lambda: seating(4),
    "pythagoras": pythagoras,                                   # L = 2 limbs
    "tsp": tsp,                                                 # order 6: site tensors of order 5
    "o3n40": lambda: random_integer_problem(3, 40, 31, 400),   # two bit words per chain
    "o4n20": lambda: random_integer_problem(4, 20, 32, 300),
    "o2n70": lambda: random_integer_problem(2, 70, 33, 500),   # order 2: site tensors of order 1
    "linear": _linear_problem,                                  # order 1: fields never change
    "o2n600": lambda: random_integer_problem(2, 600, 34, 900),  # N > 512: the per-site launch path
    "o3n520": lambda: random_integer_problem(3, 520, 35, 900),
    "wide3limb": _wide_int_problem,
    "o3n300": lambda: random_integer_problem(3, 300, 37, 700),  # two column tiles (box ring)
    "o2n400": lambda: random_integer_problem(2, 400, 38, 700),
}


@pytest.mark.parametrize("name", list(SA_CASES))
def test_sa_replays_oracle_exactly(H, torch, name):
    """Integer instances: final states, tracked and fresh energies equal the oracle's replay."""
    p = SA_CASES[name]()
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    t0 = t.default_t_start()
    for chain0, n, sweeps in ((0, 300, 6), (4000, 129, 2), (7, 1, 0)):
        X, E, Et = t.sa_shard(11, chain0, n, sweeps, t0, 0.05)
        torch.cuda.synchronize()
        xs, es = o.sa(11, chain0, n, sweeps, t0, 0.05)
        assert np.array_equal(X.cpu().numpy(), xs), (name, chain0)
        assert np.array_equal(Et.cpu().numpy(), es), (name, chain0)
        assert np.array_equal(E.cpu().numpy().astype(np.float64), es), (name, chain0)


@pytest.mark.parametrize("kind", ["ring", "stage", "pair"])
@pytest.mark.parametrize("name", ["o4n20", "o3n300"])
def test_sa_kernel_variants_replay_oracle(H, torch, kind, name):
    """Every persistent annealing kernel (HOBO_SA_KERNEL override: box ring, staged, CTA pair;
    a kernel that does not fit the shape falls back to the box ring) replays the oracle."""
    p = SA_CASES[name]()
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    t0 = t.default_t_start()
    with env("HOBO_SA_KERNEL", kind):
        X, E, Et = t.sa_shard(5, 100, 300, 3, t0, 0.05)
        torch.cuda.synchronize()
    xs, es = o.sa(5, 100, 300, 3, t0, 0.05)
    assert np.array_equal(X.cpu().numpy(), xs) and np.array_equal(Et.cpu().numpy(), es)


def test_sa_shard_invariance(H, torch):
    p = random_integer_problem(3, 24, 5, 200)
    t = H.HoboTensor.from_problem(p)
    Xa, Ea, _ = t.sa_shard(2, 0, 400, 4)
    Xb, Eb, _ = t.sa_shard(2, 150, 100, 4)
    torch.cuda.synchronize()
    assert torch.equal(Xa[150:250], Xb) and torch.equal(Ea[150:250], Eb)


def test_sa_cfg3_full_batch_sampled(H, torch):
    """BASELINE config 3 (order 3, N=512, integer, L=1) at its full 65,536 chains, one sweep
    (512 site launches): sampled chains against the oracle replay, bit for bit."""
    p = cfg3_problem()
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    B = 65536
    t0 = t.default_t_start()
    X, E, Et = t.sa_shard(3, 0, B, 1, t0, t0 / 10)
    torch.cuda.synchronize()
    Xh, Eh, Eth = X.cpu().numpy(), E.cpu().numpy().astype(np.float64), Et.cpu().numpy()
    assert np.array_equal(Eh, Eth)                               # incremental = fresh (integer)
    for c0 in (0, 777, B - 16):
        xs, es = o.sa(3, c0, 16, 1, t0, t0 / 10)
        assert np.array_equal(Xh[c0:c0 + 16], xs) and np.array_equal(Eth[c0:c0 + 16], es)


def test_sa_fp32_instance_is_honest(H, torch):
    """fp32 coefficients (L = 3): decisions follow the fp32 fields, so states are checked by
    invariants: fresh energies equal the oracle's energy of the returned states within tau,
    and the tracked energies stay within tau of them."""
    idx, val = uniform_cells(3, 30, 8)
    t, o = H.HoboTensor.import_cells(3, 30, idx, val), Oracle.from_cells(3, 30, idx, val)
    X, E, Et = t.sa_shard(4, 0, 500, 8, 5.0, 0.01)
    torch.cuda.synchronize()
    Eo = o.energy(X.cpu().numpy())
    assert np.max(np.abs(E.cpu().numpy() - Eo)) <= o.tau
    assert np.max(np.abs(Et.cpu().numpy() - Eo)) <= o.tau
    # converged chains (T_end = 0.01) are single-flip local minima up to tau
    G = o.field(X.cpu().numpy())
    assert np.all((1 - 2 * X.cpu().numpy().astype(np.float64)) * G >= -2 * o.tau)


@pytest.mark.parametrize("name,emin", [("seating4", -11.0), ("pythagoras", -30.0), ("tsp", -360.0)])
def test_sa_run_sample_set(H, torch, name, emin):
    """SPEC sa_run on the paper's problems: the SampleSet equals the oracle's aggregation of
    its replayed final states, occurrences sum to shots, and the ground energy is reached."""
    from oracle import aggregate
    p = SA_CASES[name]()
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    shots, sweeps = 1000, 200
    got = t.sa_run(7, shots, sweeps, topk=5)
    xs, es = o.sa(7, 0, shots, sweeps, t.default_t_start(), 0.01)
    want = aggregate(xs, es.astype(np.float32), 5)
    assert len(got) == len(want)
    for (gx, ge, gc), (wx, we, wc) in zip(got, want):
        assert np.array_equal(gx, wx) and ge == we and gc == wc
    assert got[0][1] == emin
    assert sum(c for _, _, c in t.sa_run(7, shots, sweeps, topk=1 << 12)) == shots


# ---- host-buffer entry points (the e2e path): chunked copies overlapped with compute ---------
def test_host_entry_points_match_device_path(H, torch):
    """cfg3 at the full 65,536 (4 chunks, ragged last) and small / offset batches: energies
    and argmin from host buffers equal the device-buffer calls bit for bit."""
    p = cfg3_problem()
    t = H.HoboTensor.from_problem(p)
    for B, row0, pinned in ((65536, 0, True), (1000, 5, False), (1, 0, False), (19000, 77, True)):
        Xh = x_bits(3, B, t.N)
        Xd = dev(torch, Xh)
        G, E, best = t.local_field(Xd, row0=row0, want_best=True)
        Ed, bestd = t.energy(Xd, row0=row0)
        torch.cuda.synchronize()
        src = torch.from_numpy(Xh).pin_memory() if pinned else Xh
        Eh, besth = t.local_field_host(src, row0=row0)
        assert np.array_equal(Eh, E.cpu().numpy()) and besth == best
        Eh2, besth2 = t.energy_host(src, row0=row0)
        assert np.array_equal(Eh2, Ed.cpu().numpy()) and besth2 == bestd
        # the fields delivered to host memory (double-buffered copy-out), pinned or pageable
        Gh = torch.empty(B, t.N, dtype=torch.float32).pin_memory() if pinned else np.empty((B, t.N), np.float32)
        Gh.fill(np.nan) if not pinned else Gh.fill_(float("nan"))
        Eh3, besth3 = t.local_field_host(src, row0=row0, G=Gh)
        Gh = Gh.numpy() if pinned else Gh
        assert np.array_equal(Gh, G.cpu().numpy()) and np.array_equal(Eh3, Eh) and besth3 == best
        if B >= 1000:
            rows = sample_rows(B, 129, 64)
            assert np.array_equal(Gh[rows].astype(np.float64), Oracle.from_problem(p).field(Xh[rows]))



# ---- packed candidates (hobo_*_bits): B x ceil(N/32) words instead of B x N bytes ------------
@pytest.mark.parametrize("case", ["cfg3", "ragged", "fp32"])
def test_packed_entry_points_match_byte_path(H, torch, case):
    """Every *_bits call (device and host buffers) equals its byte-input call bit for bit, on
    the packed rows of the same candidates; garbage in the pad bits past N is ignored.  Byte
    path results are themselves pinned to the oracle by the tests above; here the oracle is
    checked again on the packed call."""
    if case == "cfg3":
        p = cfg3_problem()
        t, o = H.HoboTensor.from_problem(p), None
        B, row0 = 20000, 11
    elif case == "ragged":
        p = random_integer_problem(3, 300, 41, nterms=800)          # N = 300: a 12-bit last word
        t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
        B, row0 = 1000, 0
    else:
        idx, val = uniform_cells(3, 130, 12)                       # int8 planes, 2-bit last word
        t, o = H.HoboTensor.import_cells(3, 130, idx, val), Oracle.from_cells(3, 130, idx, val)
        B, row0 = 500, 3
    Xh = x_bits(21, B, t.N)
    Xp = H.pack_rows(Xh)
    assert Xp.shape == (B, (t.N + 31) // 32) and Xp.dtype == np.uint32
    if t.N % 32:
        Xp[:, -1] |= np.uint32(0xFFFFFFFF) << np.uint32(t.N % 32)   # pad bits set: must be ignored
    Xd, Xpd = dev(torch, Xh), torch.from_numpy(Xp.view(np.int32)).cuda()
    G, E, best = t.local_field(Xd, row0=row0, want_best=True)
    Ee, beste = t.energy(Xd, row0=row0)
    Gb, Eb, bestb = t.local_field_bits(Xpd, row0=row0, want_best=True)
    Eeb, besteb = t.energy_bits(Xpd, row0=row0)
    torch.cuda.synchronize()
    assert torch.equal(G, Gb) and torch.equal(E, Eb) and best == bestb
    assert torch.equal(Ee, Eeb) and beste == besteb
    pinned = torch.from_numpy(Xp.view(np.int32)).pin_memory()
    for src in (Xp, pinned):
        Eh, besth = t.local_field_host_bits(src, row0=row0)
        assert np.array_equal(Eh, E.cpu().numpy()) and besth == best
        Gh = np.full((len(Eh), t.N), np.nan, np.float32)
        Eh1, besth1 = t.local_field_host_bits(src, row0=row0, G=Gh)
        assert np.array_equal(Gh, G.cpu().numpy()) and np.array_equal(Eh1, Eh) and besth1 == best
        Eh2, besth2 = t.local_field_host_bits(src, row0=row0, fields=False)
        assert np.array_equal(Eh2, Ee.cpu().numpy()) and besth2 == beste
    if o is not None:
        Eo = o.energy(Xh)
        if t.is_integer:
            assert np.array_equal(Eb.cpu().numpy(), Eo) and np.array_equal(Gb.cpu().numpy(), o.field(Xh))
        else:
            assert np.max(np.abs(Eeb.cpu().numpy() - Eo)) <= o.tau
    # empty batches
    none = (float("inf"), -1)
    assert t.energy_bits(Xpd[:0])[1] == none
    assert t.local_field_host_bits(Xp[:0])[1] == none


def test_stage_x_vectorised_and_bytewise_paths(H, torch):
    """Stage X: rows of whole words from a 16-byte aligned buffer take the
    vectorised packer, anything else the bytewise one; both give the same bits, so the same
    energies and fields (any nonzero byte counts as 1)."""
    p = random_integer_problem(3, 64, 17, nterms=400)            # N = 64: whole words
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    Xh = x_bits(23, 777, t.N)
    Xd = dev(torch, Xh * np.uint8(200))                           # nonzero bytes other than 1
    buf = torch.zeros(Xh.size + 1, dtype=torch.uint8, device="cuda")
    buf[1:].copy_(Xd.reshape(-1))
    Xu = buf[1:].view(777, t.N)                                    # unaligned: the bytewise path
    assert Xu.data_ptr() % 16 == 1
    Ga, Ea = t.local_field(Xd)
    Gu, Eu = t.local_field(Xu)
    Eo = o.energy(Xh)
    assert np.array_equal(Ea.cpu().numpy(), Eo) and torch.equal(Ea, Eu) and torch.equal(Ga, Gu)
    assert np.array_equal(Ga.cpu().numpy(), o.field(Xh))


# ---- the library's own NCCL communicator (hobo_dist_*), exercised at world size 1 -----------
def test_library_comm_world1_matches_single_gpu(H, torch):
    """With a communicator every best goes through ncclAllReduce(MIN) and hobo_search through
    the rank-sharded path + ncclBroadcast; at world 1 those are identities, so every result
    equals the communicator-free call and the oracle replay."""
    p = random_integer_problem(3, 40, 77, nterms=500)
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    ref_x, ref_e = t.search_global(9, 300, 20)
    r = o.search(9, 0, 300, 20)
    assert ref_e == r["e_best"] and np.array_equal(ref_x, r["chain_xbest"][r["best_chain"]])
    Xh = x_bits(5, 1000, 40)
    X = dev(torch, Xh)
    _, ref_b = t.energy(X, row0=3)
    dev_index = torch.cuda.current_device()
    uid = H.dist_unique_id()
    H.dist_init(0, 1, uid, dev_index)
    try:
        assert H.dist_info() == (0, 1)
        with pytest.raises(H.HoboError) as e:
            H.dist_init(0, 1, uid, dev_index)
        assert e.value.status == H.HOBO_ESTATE
        x, e = t.search_global(9, 300, 20)
        assert e == ref_e and np.array_equal(x, ref_x)
        assert t.energy(X, row0=3)[1] == ref_b
        assert t.local_field(X, row0=3, want_best=True)[2] == ref_b
        assert t.local_field_host(Xh, row0=3)[1] == ref_b
        Xp = H.pack_rows(Xh)
        assert t.local_field_host_bits(Xp, row0=3)[1] == ref_b
        assert t.energy_bits(torch.from_numpy(Xp.view(np.int32)).cuda(), row0=3)[1] == ref_b
        assert t.energy(X[:0])[1] == (float("inf"), -1)
    finally:
        H.dist_finalize()
    assert H.dist_info() == (0, 1)


# ---- edge cases of every batch entry point --------------------------------------------------
def test_empty_batches_and_argument_errors(H, torch):
    p = random_integer_problem(3, 24, 5, nterms=200)
    t = H.HoboTensor.from_problem(p)
    X0 = torch.empty(0, t.N, dtype=torch.uint8, device="cuda")
    none = (float("inf"), -1)
    assert t.energy(X0)[1] == none
    assert t.local_field(X0, want_best=True)[2] == none
    assert t.local_field_host(np.zeros((0, t.N), np.uint8))[1] == none
    assert t.energy_host(np.zeros((0, t.N), np.uint8))[1] == none
    with pytest.raises(H.HoboError) as e:                 # TT energies before the TT cores exist
        t.tt_energy(X0)
    assert e.value.status == H.HOBO_ESTATE
    t.tt_build(0.0)
    assert t.tt_energy(X0)[1] == none
    G, E = t.multilinear_field(torch.empty(0, t.N, dtype=torch.bfloat16, device="cuda"))
    assert G.shape == (0, t.N)
    # annealing and search arguments (0 < t_end <= t_start, >= 1 chain / shot, step > 0)
    for bad in (lambda: t.sa_shard(1, 0, 10, 2, 1.0, 2.0), lambda: t.sa_shard(1, 0, 0, 2, 2.0, 1.0),
                lambda: t.sa_shard(1, 0, 10, 2, 0.0, 0.0), lambda: t.sa_run(1, 0, 2),
                lambda: t.search(1, 0, 4), lambda: t.gd_run(1, 16, 4, 0.0),
                lambda: t.search_global(1, 0, 4)):
        with pytest.raises(H.HoboError) as e:
            bad()
        assert e.value.status == H.HOBO_EINVAL
    # device path limit: N <= 1024
    from workloads import TermBuilder
    tb = TermBuilder()
    tb.add(1.0, [(0.0, [(0, 1.0)]), (0.0, [(1024, 1.0)])])
    big = H.HoboTensor.from_problem(tb.problem(2, 1025))
    with pytest.raises(H.HoboError) as e:
        big.energy(torch.zeros(1, 1025, dtype=torch.uint8, device="cuda"))
    assert e.value.status == H.HOBO_EINVAL



def test_nan_energy_is_an_error(H, torch):
    """a NaN energy is an error, not a candidate.  Cells of +-3e38 at the
    all-ones candidate overflow the persistent kernel's fp32 chunk sums to +inf in one column
    tile and -inf in the other; their sum is NaN, and the argmin returns ERANGE (also through
    the library communicator at world 1).  Without the argmin the energies are still written."""
    N = 256
    idx = np.array([[0, 1], [0, 2], [0, 129], [0, 130]], np.int32)
    val = np.array([3e38, 3e38, -3e38, -3e38], np.float32)
    t = H.HoboTensor.import_cells(2, N, idx, val)
    X = torch.ones(64, N, dtype=torch.uint8, device="cuda")
    with env("HOBO_PERSIST", "1"):
        E, _ = t.energy(X, want_best=False)
        torch.cuda.synchronize()
        assert torch.isnan(E).all()
        with pytest.raises(H.HoboError) as e:
            t.energy(X)
        assert e.value.status == H.HOBO_ERANGE
        uid = H.dist_unique_id()
        H.dist_init(0, 1, uid, torch.cuda.current_device())
        try:
            with pytest.raises(H.HoboError) as e:
                t.energy(X)
            assert e.value.status == H.HOBO_ERANGE
        finally:
            H.dist_finalize()


# ---- CTA pairs (cta_group::2) and the single-CTA kernel, each forced on both limb regimes ----
@pytest.mark.parametrize("force", ["1", "0"])
def test_cta_pair_and_single_paths(H, torch, force):
    """HOBO_PAIR=1 runs every 256-column contraction on CTA pairs (M = 256 MMAs over two SMs),
    =0 on single CTAs: integer instances stay bit-exact, fp32 ones within tau, either way."""
    import os
    old = os.environ.get("HOBO_PAIR")
    os.environ["HOBO_PAIR"] = force
    try:
        for p in (random_integer_problem(3, 300, 41, nterms=800), cfg3_problem()):   # L = 1
            t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
            X = x_bits(6, 1000, t.N)                           # 8 candidate blocks: odd pairs too
            G, E = fields(H, torch, t, X)
            assert np.array_equal(E, o.energy(X)) and np.array_equal(G, o.field(X))
        idx, val = uniform_cells(3, 260, 3)                    # L = 3, two column tiles
        t, o = H.HoboTensor.import_cells(3, 260, idx, val), Oracle.from_cells(3, 260, idx, val)
        X = x_bits(7, 383, 260)                                # 3 candidate blocks: a lone last block
        G, E = fields(H, torch, t, X)
        assert np.max(np.abs(E - o.energy(X))) <= o.tau and np.max(np.abs(G - o.field(X))) <= o.tau
        Ee, _ = energies(H, torch, t, X)
        assert np.max(np.abs(Ee - o.energy(X))) <= o.tau
    finally:
        if old is None:
            del os.environ["HOBO_PAIR"]
        else:
            os.environ["HOBO_PAIR"] = old


# ---- column tiles longest-first (HOBO_CT_DESC) ---------------------------------------------
@pytest.mark.parametrize("desc", ["1", "0"])
def test_column_tile_order(H, torch, desc):
    """The triangular (energy-mode) schedules give later column tiles more K-blocks, so they
    are issued first by default; either order gives the same per-candidate results (each tile
    is one CTA's independent work): bit-exact on integer cells (bf16 and int8), within tau on
    fp32 cells, with several column tiles and a ragged candidate tail."""
    with env("HOBO_CT_DESC", desc):
        p = random_integer_problem(3, 300, 41, nterms=800)
        t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
        X = x_bits(9, 700, t.N)
        Ee, best = energies(H, torch, t, X)
        G, E = fields(H, torch, t, X)
        Eo = o.energy(X)
        assert np.array_equal(Ee, Eo) and np.array_equal(E, Eo) and np.array_equal(G, o.field(X))
        check_argmin(best, Eo, 0.0)
        for i8 in ("1", "0"):
            with env("HOBO_I8", i8):
                idx, val = uniform_cells(3, 300, 5)                # 2-3 column tiles
                t, o = H.HoboTensor.import_cells(3, 300, idx, val), Oracle.from_cells(3, 300, idx, val)
                X = x_bits(10, 300, 300)
                Ee, best = energies(H, torch, t, X)
                Eo = o.energy(X)
                if i8 == "1" and t.launch_stats()["i8_planes"]:
                    assert np.array_equal(Ee, f32(Eo))
                assert np.max(np.abs(Ee - Eo)) <= o.tau
                check_argmin(best, Eo, o.tau)


# ---- energy launches looping each CTA over several candidate blocks (HOBO_CB_ITERS) -------------
@pytest.mark.parametrize("iters", ["1", "2", "3", "8"])
def test_energy_multi_block_ctas(H, torch, iters):
    """A CTA that runs several candidate blocks back to back (the next block's W fill overlapping
    the previous epilogue; accumulator handed back through a barrier) gives the same energies
    and argmin: bit-exact on integer cells, within tau on fp32 cells; ragged block counts."""
    with env("HOBO_CB_ITERS", iters), env("HOBO_PAIR", "0"), env("HOBO_I8", "0"):
        p = random_integer_problem(3, 300, 41, nterms=800)
        t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
        for B in (1, 700, 1300):                                   # 1, 6, 11 candidate blocks
            X = x_bits(31, B, t.N)
            Ee, best = energies(H, torch, t, X, row0=5)
            Eo = o.energy(X)
            assert np.array_equal(Ee, Eo)
            check_argmin(best, Eo, 0.0, row0=5)
        idx, val = uniform_cells(2, 1024, 2)                       # cfg2's shape, 4 column tiles
        t, o = H.HoboTensor.import_cells(2, 1024, idx, val), Oracle.from_cells(2, 1024, idx, val)
        X = x_bits(32, 1500, 1024)
        Ee, best = energies(H, torch, t, X)
        Eo = o.energy(X)
        assert np.max(np.abs(Ee - Eo)) <= o.tau
        check_argmin(best, Eo, o.tau)


# ---- int8 digit planes (tcgen05.mma kind::i8): exact integer accumulation --------------------
@pytest.mark.parametrize("i8", ["1", "0"])
@pytest.mark.parametrize("order,N,B,seed", [(2, 300, 700, 11), (3, 130, 500, 12), (3, 260, 383, 13), (4, 30, 300, 14),
                                            (3, 300, 37, 41), (2, 1024, 1000, 2), (5, 16, 200, 15)])
def test_int8_digit_planes_fp32_cells(H, torch, order, N, B, seed, i8):
    """U(-1,1) cells lie on a 2^-23 fixed-point grid, so three int8 digit planes (unsigned low
    digits, signed top digit) hold every cell exactly and the s32 accumulators sum them without
    rounding: the int8 path's energies and fields equal the oracle's exact values rounded once
    to fp32 (reading 24).  HOBO_I8=0 keeps the bf16-limb path, within tau."""
    with env("HOBO_I8", i8):
        idx, val = uniform_cells(order, N, seed)
        t, o = H.HoboTensor.import_cells(order, N, idx, val), Oracle.from_cells(order, N, idx, val)
        X = x_bits(seed, B, N)
        G, E = fields(H, torch, t, X)
        assert t.launch_stats()["i8_planes"] == (3 if i8 == "1" else 0)
        Ee, best = energies(H, torch, t, X)
    Eo, Go = o.energy(X), o.field(X)
    if i8 == "1":
        assert np.array_equal(E, f32(Eo)) and np.array_equal(Ee, f32(Eo)) and np.array_equal(G, f32(Go))
    else:
        assert max(np.max(np.abs(E - Eo)), np.max(np.abs(Ee - Eo)), np.max(np.abs(G - Go))) <= o.tau
    check_argmin(best, Eo, o.tau)


@pytest.mark.parametrize("pair", ["1", "0"])
def test_int8_digit_planes_integer_instances(H, torch, pair):
    """Integer instances forced onto the int8 path (1 or 2 digit planes; CTA pairs forced on and
    off): bit-exact against the oracle like the bf16 path."""
    with env("HOBO_I8", "1"), env("HOBO_PAIR", pair):
        cases = [(cfg3_problem(), 1000, 2), (random_integer_problem(3, 300, 41, nterms=800), 1000, None),
                 (random_integer_problem(4, 40, 6, nterms=300), 200, None), (seating(4), 4096, 1), (tsp(), 64, None),
                 (random_integer_problem(2, 37, 9, nterms=200), 5, None)]
        for p, B, want in cases:
            t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
            X = x_bits(8, B, t.N)
            G, E = fields(H, torch, t, X)
            planes = t.launch_stats()["i8_planes"]
            assert planes >= 1 and (want is None or planes == want), (p.name, planes)
            Ee, best = energies(H, torch, t, X)
            Eo = o.energy(X)
            assert np.array_equal(G, o.field(X)) and np.array_equal(E, Eo) and np.array_equal(Ee, Eo), p.name
            check_argmin(best, Eo, 0.0)


def test_int8_digit_planes_choice(H, torch):
    """The automatic choice: int8 when it costs fewer tensor-core cycles (3 digit planes at twice
    the rate vs 3 bf16 limbs; 1 digit vs 1 limb) over K loops of >= 64 K-blocks; bf16 when it
    does not (cfg3: 2 digits vs 1 limb), for short K loops (N=64 at order 3: 33 K-blocks), and
    when the cells are not a <= 3-byte fixed-point grid."""
    X = x_bits(1, 256, 200)
    for make, want in ((lambda: H.HoboTensor.import_cells(3, 200, *uniform_cells(3, 200, 1)), 3),
                       (lambda: H.HoboTensor.import_cells(3, 200, *int_twin_cells(3, 200, 1)), 1),
                       (lambda: H.HoboTensor.from_problem(random_integer_problem(3, 200, 2, nterms=50)), None)):
        t = make()
        t.energy(dev(torch, X))
        got = t.launch_stats()["i8_planes"]
        assert (got == want) if want is not None else got in (0, 1, -1, -2, -3)
    p = cfg3_problem()
    t = H.HoboTensor.from_problem(p)
    t.local_field(dev(torch, x_bits(3, 128, 512)))
    assert t.launch_stats()["i8_planes"] == -2             # e4m3 limbs (two planes, the second sparse)
    with env("HOBO_F8", "0"):
        t = H.HoboTensor.from_problem(p)
        t.local_field(dev(torch, x_bits(3, 128, 512)))
        assert t.launch_stats()["i8_planes"] == 0
    t = H.HoboTensor.import_cells(3, 64, *uniform_cells(3, 64, 1))
    t.energy(dev(torch, x_bits(1, 256, 64)))
    assert t.launch_stats()["i8_planes"] == 0              # 33 K-blocks: bf16
    X = x_bits(1, 256, 64)
    idx, val = uniform_cells(2, 64, 3)
    val = val.copy()
    val[np.flatnonzero(idx[:, 0] != idx[:, 1])[0]] = np.float32(3.0e-12)   # a degree-2 cell with a ~2^-62
    # quantum next to O(1) cells: no 3-byte fixed-point grid holds both
    with env("HOBO_I8", "1"):                                # even when forced: not exact in 3 bytes
        t = H.HoboTensor.import_cells(2, 64, idx, val)
        t.energy(dev(torch, X))
    assert t.launch_stats()["i8_planes"] == 0


def test_int8_host_entry_points_and_search(H, torch):
    """The int8 path behind the host-buffer entry points (chunked copies, ragged last chunk)
    and inside the search loop: host calls equal the device calls bit for bit on U(-1,1)
    cells, and a forced-int8 search replays the oracle chain for chain on an integer
    instance."""
    idx, val = uniform_cells(3, 200, 17)
    t, o = H.HoboTensor.import_cells(3, 200, idx, val), Oracle.from_cells(3, 200, idx, val)
    for B, row0 in ((20000, 0), (333, 9)):
        Xh = x_bits(17, B, 200)
        Xd = dev(torch, Xh)
        G, E, best = t.local_field(Xd, row0=row0, want_best=True)
        assert t.launch_stats()["i8_planes"] == 3
        Ed, bestd = t.energy(Xd, row0=row0)
        torch.cuda.synchronize()
        Eh, besth = t.local_field_host(Xh, row0=row0)
        assert np.array_equal(Eh, E.cpu().numpy()) and besth == best
        Eh2, besth2 = t.energy_host(Xh, row0=row0)
        assert np.array_equal(Eh2, Ed.cpu().numpy()) and besth2 == bestd
        rows = np.arange(0, B, 97)
        assert np.array_equal(E.cpu().numpy().astype(np.float64)[rows], f32(o.energy(Xh[rows])))
    with env("HOBO_I8", "1"):
        p = random_integer_problem(3, 40, 77, nterms=500)
        t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
        x, e, c = t.search(9, None, 20, chain0=0, nchains=300)
        assert t.launch_stats()["i8_planes"] >= 1
    r = o.search(9, 0, 300, 20)
    assert (e, c) == (r["e_best"], r["best_chain"]) and np.array_equal(x, r["chain_xbest"][c])


# ---- e4m3 limbs (tcgen05.mma kind::f8f6f4): exact on integer-encoded instances --------------
def pow2_int_cells(order, N, seed, density=0.02, wide=0.0):
    """Sparse integer cells shaped like binary-integer encodings: s * m * 2^e with m in
    {1, 3, 5, 7} and e in [0, 8] (one e4m3 limb each); a fraction `wide` of them get a 9-12
    significant-bit m instead (second and third limbs).  Exact in fp32; sum |H| < 2^24."""
    idx = canonical_cells_all(order, N)
    cid = h(seed, 1, np.arange(len(idx), dtype=np.uint64), 0)
    keep = (cid % np.uint64(10000)) < np.uint64(int(density * 10000))
    idx = idx[keep]
    r = h(seed, 2, np.arange(len(idx), dtype=np.uint64), 0)
    m = np.array([1, 3, 5, 7], np.int64)[(r % np.uint64(4)).astype(np.int64)]
    e = ((r >> np.uint64(8)) % np.uint64(9)).astype(np.int64)
    wm = ((r >> np.uint64(16)) % np.uint64(3840)).astype(np.int64) + 257   # 9-12 significant bits
    is_wide = ((r >> np.uint64(32)) % np.uint64(10000)).astype(np.int64) < int(wide * 10000)
    mag = np.where(is_wide, wm, m << e)
    sgn = np.where((r >> np.uint64(48)) & np.uint64(1), -1, 1)
    return idx, (sgn * mag).astype(np.float32)


@pytest.mark.parametrize("pair", ["1", "0"])
def test_e4m3_limbs_integer_instances(H, torch, pair):
    """Integer instances on the e4m3-limb path (cfg3: 2 limb planes, the second needed by a
    few degree-2 cells only; wide cells: 3 planes): fields, energies (field and energy modes)
    and the argmin bit-exact against the oracle and equal to the bf16 path (HOBO_F8=0)."""
    cases = [("cfg3", None, None, cfg3_problem(), 1000, -2),
             ("pow2", 3, 200, pow2_int_cells(3, 200, 5), 700, -1),
             ("wide", 3, 200, pow2_int_cells(3, 200, 6, wide=0.0003), 383, -3),
             ("order4", 4, 60, pow2_int_cells(4, 60, 7, density=0.05), 300, None),
             ("ragged", 3, 300, pow2_int_cells(3, 300, 8, density=0.01), 1000, None)]   # N=300: padded tile

    def build(order, N, src):
        if order is None:
            return H.HoboTensor.from_problem(src), Oracle.from_problem(src)
        return H.HoboTensor.import_cells(order, N, *src), Oracle.from_cells(order, N, *src)

    with env("HOBO_PAIR", pair):
        for name, order, N, src, B, want in cases:
            t, o = build(order, N, src)
            X = x_bits(17, B, t.N)
            G, E = fields(H, torch, t, X)
            kind = t.launch_stats()["i8_planes"]
            assert kind < 0 and (want is None or kind == want), (name, kind)
            Ee, best = energies(H, torch, t, X, row0=3)
            assert t.launch_stats()["i8_planes"] < 0, name
            Eo, Go = o.energy(X), o.field(X)
            assert np.array_equal(G, Go) and np.array_equal(E, Eo) and np.array_equal(Ee, Eo), name
            check_argmin(best, Eo, 0.0, row0=3)
            with env("HOBO_F8", "0"):
                tb, _ = build(order, N, src)
                Gb, Eb = fields(H, torch, tb, X)
                assert tb.launch_stats()["i8_planes"] >= 0
                assert np.array_equal(Gb, G) and np.array_equal(Eb, E), name


def test_e4m3_limbs_choice(H, torch):
    """e4m3 limbs only where they pay: cells needing two limbs almost everywhere (5-8
    significant bits: one bf16 limb) fall back to bf16 after the limb scan; cells beyond three
    limbs (13+ bits) or non-integer cells never take them; HOBO_F8=1 forces an exact split of
    scaled fractions."""
    X = x_bits(2, 300, 200)
    idx = canonical_cells_all(3, 200)
    r = h(9, 3, np.arange(len(idx), dtype=np.uint64), 0)
    keep = (r % np.uint64(100)) < np.uint64(2)
    idx = idx[keep]
    mag = ((r[keep] >> np.uint64(8)) % np.uint64(120)).astype(np.int64) * 2 + 17   # odd, 5-8 bits
    t = H.HoboTensor.import_cells(3, 200, idx, mag.astype(np.float32))
    o = Oracle.from_cells(3, 200, idx, mag.astype(np.float32))
    E, _ = energies(H, torch, t, X)
    assert t.launch_stats()["i8_planes"] == 0 and np.array_equal(E, o.energy(X))
    big = ((r[keep] >> np.uint64(8)) % np.uint64(4096)).astype(np.int64) * 2 + 8193  # 14 bits
    t = H.HoboTensor.import_cells(3, 200, idx, big.astype(np.float32))
    energies(H, torch, t, X)
    assert t.launch_stats()["i8_planes"] >= 0
    # 1, 3, 5, 7 x 2^-e, e in [0, 12]: one e4m3 limb each (scaled by 2^5: 2^-7 .. 224), but a
    # 15-bit fixed-point grid (two int8 digits against one bf16 limb), so e4m3 pays
    fr = (((mag % 8) | 1).astype(np.float64) * 2.0 ** -(mag % 13).astype(np.float64)).astype(np.float32)
    with env("HOBO_F8", "1"):
        t = H.HoboTensor.import_cells(3, 200, idx, fr)
        o = Oracle.from_cells(3, 200, idx, fr)
        E, best = energies(H, torch, t, X)
        assert t.launch_stats()["i8_planes"] < 0
        assert np.max(np.abs(E - o.energy(X))) <= o.tau
    t = H.HoboTensor.import_cells(3, 200, idx, fr)
    energies(H, torch, t, X)
    assert t.launch_stats()["i8_planes"] >= 0                               # not integer: default off


def test_e4m3_limbs_split_schedules(H, torch):
    """The e4m3-limb contraction under the stream-K schedule (partial wave: leftover tiles cut
    into K ranges), under split-K (tiny batches) and in the search loop: bit-exact against the
    oracle and against the data-parallel schedule."""
    p = cfg3_problem()
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    for B in (5000, 64, 1):
        X = x_bits(23, B, 512)
        G, E = fields(H, torch, t, X)
        assert t.launch_stats()["i8_planes"] == -2
        with env("HOBO_SK", "0"):
            G0, E0 = fields(H, torch, t, X)
        assert np.array_equal(G, G0) and np.array_equal(E, E0)
        rows = sample_rows(B, 129, 64) if B >= 64 else np.arange(B)
        assert np.array_equal(G[rows], o.field(X[rows])) and np.array_equal(E[rows], o.energy(X[rows]))
    x, e, c = t.search(9, None, 2, chain0=0, nchains=64)
    r = o.search(9, 0, 64, 2)
    assert (e, c) == (r["e_best"], r["best_chain"]) and np.array_equal(x, r["chain_xbest"][c])


@pytest.mark.parametrize("N", [128, 193, 200, 255])
def test_e4m3_segment_tails(H, torch, N):
    """Segments whose K-block count is odd end in a pair holding one K-block of tuples and one of
    zero padding; e4m3 stages take two pairs, so such a pair can be a stage's second.  Two-bit
    candidates x_a = x_b = 1 select single tuples {a, b} (plus degree-2 ones) across the whole
    last stretch of the order-3 segment: fields bit-exact against the oracle."""
    idx, val = pow2_int_cells(3, N, 5)
    t, o = H.HoboTensor.import_cells(3, N, idx, val), Oracle.from_cells(3, N, idx, val)
    prs = [(a, b) for b in range(max(1, N - 12), N) for a in range(b)]
    X = np.zeros((len(prs) + 2, N), np.uint8)
    for r, (a, b) in enumerate(prs):
        X[r, a] = X[r, b] = 1
    X[-2, :] = 1
    X[-1, 1::2] = 1
    G, E = fields(H, torch, t, X)
    assert t.launch_stats()["i8_planes"] < 0
    assert np.array_equal(G, o.field(X)) and np.array_equal(E, o.energy(X))


def test_e4m3_n1024_integer_encoded(H, torch):
    """cfg3's recipe at N = 1024 (256 four-bit variables, the device path's largest N): the
    e4m3-limb path in field and energy mode, strided rows and the argmin bit-exact against
    the oracle (sum |H| < 2^24, so the exactness guard admits it)."""
    p = int_encoded_problem(256, 4, 2048, 4096, 7)
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    X = x_bits(5, 4096, p.N)
    G, E = fields(H, torch, t, X)
    assert t.launch_stats()["i8_planes"] < 0
    rows = sample_rows(4096, 97)
    assert np.array_equal(G[rows], o.field(X[rows])) and np.array_equal(E[rows], o.energy(X[rows]))
    Ee, best = energies(H, torch, t, X)
    assert np.array_equal(Ee, E)
    assert best == (E.min(), int(np.argmin(E)))


def test_bench_line_contract(H, torch):
    """`python bench.py` (the driver's command, few steps) prints one JSON line carrying the
    contract's keys, consistent with each other: value = units / step time, the roofline
    fraction = achieved / peak, the e2e byte counts of the host-buffer call, the clocks."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3"], cwd=root,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["higher_is_better"] is True
    assert abs(d["value"] - d["config"]["global_batch"] / (d["ms_per_step"] / 1e3)) <= 1e-6 * d["value"]
    r = d["roofline"]
    assert r["bound"] in ("tensor", "hbm") and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert 0.0 < r["frac"] <= 1.0 and r["kernel_ms"] > 0
    e = d["e2e"]
    B, N = d["config"]["global_batch"], d["config"]["N"]
    assert e["h2d_bytes_per_step"] == B * N and e["d2h_bytes_per_step"] == B * 4 + B * N * 4 + 16
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["gpu_launches"] > 0 and isinstance(d["clocks"], dict)
