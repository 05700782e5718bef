"""Pins of the CPU oracle (oracle/) against what the paper and the mathematics fix.

None of these checks re-types the oracle's formulas: energies are compared with the
paper's printed values, with the UNEXPANDED Hamiltonians of PAPER.md 5 evaluated
directly, with library linear algebra (numpy matmul / SVD), with exhaustive
enumeration, and with identities (flip identity, linearity, special cases).
"""
import numpy as np
import pytest

from oracle import Oracle, hash4, search_thresholds, splitmix64
from workloads import (canonical_cells_all, cfg3_problem, exhaustive_X, h, int_twin_cells,
                       paper_grids, pyth_bits, pythagoras, random_integer_problem, seating,
                       tsp, tsp_bits, uniform_cells, x_bits)


# ---- direct (unexpanded) evaluation of the paper's Hamiltonians --------------------------
def f_seating(X, n, weight=10.0):
    """PAPER.md:177-192 evaluated as written: -sum q + weight * sum of 3-windows."""
    q = X.reshape(-1, n, n).astype(np.int64)
    h2 = sum(q[:, i, j] * q[:, i, j + 1] * q[:, i, j + 2] for i in range(n) for j in range(n - 2))
    h2 = h2 + sum(q[:, i, j] * q[:, i + 1, j] * q[:, i + 2, j] for j in range(n) for i in range(n - 2))
    return -q.sum(axis=(1, 2)) + weight * h2


def f_pythagoras(X, weight=10.0):
    """PAPER.md:283-298 as written: (x^2+y^2-z^2)^2 + weight*sum prod(1-q)."""
    X = X.astype(np.int64)
    v = [sum(X[:, 4 * i + k] << k for k in range(4)) for i in range(3)]
    zero = sum((v[i] == 0).astype(np.int64) for i in range(3))
    return (v[0] ** 2 + v[1] ** 2 - v[2] ** 2) ** 2 + weight * zero


def f_tsp(X, weight=10.0):
    """PAPER.md:371-380 as written: weight*(xB*xC*xD - 6)^2, xB = 2 q0_0 + q0_1."""
    X = X.astype(np.int64)
    v = [2 * X[:, 2 * i] + X[:, 2 * i + 1] for i in range(3)]
    return weight * (v[0] * v[1] * v[2] - 6) ** 2


# ---- paper printouts --------------------------------------------------------------------
def test_offsets_printed(pins):
    for name, p in (("seating5x5", seating(5)), ("pythagoras", pythagoras()), ("tsp", tsp())):
        assert Oracle.from_problem(p).offset == pins["offsets"][name]["value"], name


def test_printed_energies(pins):
    pe = pins["printed_energies"]
    assert np.all(Oracle.from_problem(seating(5)).energy(paper_grids()) == pe["seating5x5_grids"]["value"])
    X = np.stack([pyth_bits(*t) for t in pe["pythagoras_triples"]["triples"]])
    assert np.all(Oracle.from_problem(pythagoras()).energy(X) == pe["pythagoras_triples"]["value"])
    X = np.stack([tsp_bits(*t) for t in pe["tsp_assignments"]["assignments"]])
    assert np.all(Oracle.from_problem(tsp()).energy(X) == pe["tsp_assignments"]["value"])


def test_tsp_tensor_shape_and_tt_ranks(pins):
    """Dense TSP tensor is (6,)*6; sequential SVD without truncation gives
    the core shapes printed at P:560.  This pins the smallest-subscript-FIRST replication rule:
    other placements give other ranks."""
    H = Oracle.from_problem(tsp()).dense().astype(np.float64)
    assert list(H.shape) == pins["tensor_shape_tsp"]["value"]
    shapes, r, A = [], 1, H
    for k in range(5):
        M = A.reshape(r * 6, -1)
        U, S, Vt = np.linalg.svd(M, full_matrices=False)
        rk = int((S > 1e-12 * S[0]).sum())
        shapes.append([6, rk] if k == 0 else [r, 6, rk])
        A = (S[:rk, None] * Vt[:rk])
        r = rk
    shapes.append([r, 6])
    assert shapes == pins["tt_core_shapes_tsp"]["value"]


# ---- tensor form vs the unexpanded formulas, exhaustively ----------------------------------
@pytest.mark.parametrize("name", ["seating4", "pythagoras", "tsp"])
def test_energy_plus_offset_equals_formula(name):
    p, f = {"seating4": (seating(4), lambda X: f_seating(X, 4)),
            "pythagoras": (pythagoras(), f_pythagoras), "tsp": (tsp(), f_tsp)}[name]
    o = Oracle.from_problem(p)
    X = exhaustive_X(p.N)
    E = o.energy(X)
    assert np.array_equal(E + o.offset, f(X).astype(np.float64))
    # O4' (literal sum over all N^k cells) agrees with the term-by-term O4 everywhere
    if p.N ** p.order * len(X) <= 3e8:
        assert np.array_equal(o.energy_tensor(X), E)


def test_energy_tensor_seating5_printed():
    """P:65 literal contraction of the (25,25,25) tensor at the printed grids."""
    o = Oracle.from_problem(seating(5))
    assert np.all(o.energy_tensor(paper_grids()) == -17.0)


def test_cancellation_above_the_order_is_dropped_not_an_error():
    """O1 before O2 (reading 7): a degree-4 monomial that cancels to
    zero is dropped before the degree check, so an order-2 build succeeds; one that survives
    is an error."""
    from workloads import TermBuilder
    tb = TermBuilder()
    tb.add(1.0, [(0.0, [(i, 1.0)]) for i in range(4)])
    tb.add(-1.0, [(0.0, [(i, 1.0)]) for i in range(4)])
    tb.add(2.0, [(0.0, [(0, 1.0)])])
    o = Oracle.from_problem(tb.problem(2, 4))
    assert o.ncells == 1 and o.cells()[1].tolist() == [2.0]
    tb.add(1.0, [(0.0, [(i, 1.0)]) for i in range(4)])
    with pytest.raises(Exception):
        Oracle.from_problem(tb.problem(2, 4))


def test_nonzero_cells(pins):
    for name, p in (("seating5x5", seating(5)), ("pythagoras", pythagoras()), ("tsp", tsp())):
        assert Oracle.from_problem(p).ncells == pins["nonzero_cells"][name]["value"], name


def test_canonical_index_examples(pins):
    for ex in pins["canonical_index"]["examples"]:
        order, s = ex["order"], ex["set"]
        N = max(s) + 1
        # present the set as a scrambled tuple of the right length; the oracle must place it
        tup = (s + [s[-1]] * order)[:order][::-1]
        o = Oracle.from_cells(order, N, np.array([tup], np.int32), np.array([3.0], np.float32))
        idx, val = o.cells()
        assert idx.tolist() == [ex["cell"]] and val.tolist() == [3.0]


def test_from_cells_canonicalises_by_index_set():
    """(i,j,j) and (j,i,i) both land on the canonical cell of {i,j}; energies on binary x are
    the full N^k contraction of the raw tensor (a closed-form: einsum over a random tensor)."""
    rng = np.random.default_rng(0)
    N, k = 6, 3
    T = rng.integers(-3, 4, size=(N,) * k).astype(np.float32)
    idx = np.stack(np.meshgrid(*[np.arange(N)] * k, indexing="ij"), -1).reshape(-1, k).astype(np.int32)
    o = Oracle.from_cells(k, N, idx, T.reshape(-1))
    X = exhaustive_X(N)
    ref = np.einsum("ijk,bi,bj,bk->b", T.astype(np.float64), X, X, X)
    assert np.array_equal(o.energy(X), ref)
    for tup, _ in zip(*o.cells()):
        tup = list(tup)
        rest = [v for v in tup if v != tup[0]]      # repeats only of the smallest, at the front
        assert tup == sorted(tup) and tup == [tup[0]] * (len(tup) - len(rest)) + rest
        assert len(set(rest)) == len(rest)


# ---- brute force ------------------------------------------------------------------------
def test_brute_force_table(pins):
    bf = pins["brute_force"]
    r = Oracle.from_problem(seating(4)).brute()
    assert (r["emin"], r["argmin"], r["next_level"]) == (bf["seating4x4"]["emin"], bf["seating4x4"]["argmin"],
                                                         bf["seating4x4"]["next_level"])
    assert r["ground"].tolist() == bf["seating4x4"]["ground"]
    for name, p in (("pythagoras", pythagoras()), ("tsp", tsp())):
        r = Oracle.from_problem(p).brute()
        assert (r["emin"], r["argmin"], r["n_ground"], r["next_level"]) == (
            bf[name]["emin"], bf[name]["argmin"], bf[name]["n_ground"], bf[name]["next_level"]), name
    # TSP ground states are exactly the permutations of (1,2,3)
    r = Oracle.from_problem(tsp()).brute()
    perms = {(1, 2, 3), (1, 3, 2), (2, 1, 3), (2, 3, 1), (3, 1, 2), (3, 2, 1)}
    dec = {tuple(2 * ((t >> (2 * i)) & 1) + ((t >> (2 * i + 1)) & 1) for i in range(3)) for t in r["ground"]}
    assert dec == perms


@pytest.mark.slow
def test_brute_force_seating5(pins):
    r = Oracle.from_problem(seating(5)).brute()
    bf = pins["brute_force"]["seating5x5"]
    assert (r["emin"], r["argmin"], r["n_ground"]) == (bf["emin"], bf["argmin"], bf["n_ground"])
    # the three printed grids are ground states
    idx = paper_grids().astype(np.int64) @ (1 << np.arange(25, dtype=np.int64))
    assert set(idx.tolist()) <= set(r["ground"].tolist())


def test_all_ones_and_zero(pins):
    ao = pins["all_ones_energy"]
    for name, p in (("seating4x4", seating(4)), ("pythagoras", pythagoras()), ("tsp", tsp())):
        o = Oracle.from_problem(p)
        E = o.energy(np.stack([np.zeros(p.N, np.uint8), np.ones(p.N, np.uint8)]))
        assert E[0] == 0.0 and E[1] == ao[name], name


# ---- closed forms via library linear algebra ----------------------------------------------
def test_qubo_energy_is_xQx():
    idx, val = uniform_cells(2, 64, 11)
    o = Oracle.from_cells(2, 64, idx, val)
    Q = o.dense().astype(np.float64)
    X = x_bits(7, 300, 64)
    ref = np.einsum("bi,ij,bj->b", X.astype(np.float64), Q, X.astype(np.float64))
    assert np.allclose(o.energy(X), ref, rtol=0, atol=1e-9 * o.sum_abs)


def test_order3_energy_batched_matmul():
    idx, val = uniform_cells(3, 24, 12)
    o = Oracle.from_cells(3, 24, idx, val)
    H = o.dense().astype(np.float64)
    X = x_bits(8, 200, 24).astype(np.float64)
    inner = np.einsum("ijk,bk->bij", H, X)                  # H_i x
    ref = np.einsum("bi,bj,bij->b", X, X, inner)            # sum_i x_i x^T H_i x
    assert np.allclose(o.energy(X.astype(np.uint8)), ref, rtol=0, atol=1e-9 * o.sum_abs)


def test_linearity():
    idx, val = uniform_cells(3, 12, 13)
    o1 = Oracle.from_cells(3, 12, idx, val)
    o2 = Oracle.from_cells(3, 12, idx, val * 2)              # exact scaling in fp32
    X = exhaustive_X(12)
    assert np.array_equal(o2.energy(X), 2 * o1.energy(X))


# ---- local field ------------------------------------------------------------------------
@pytest.mark.parametrize("order,seed", [(2, 1), (3, 2), (4, 3), (5, 4)])
def test_field_flip_identity(order, seed):
    """g_m = E(x|x_m=1) - E(x|x_m=0): E(x xor e_m) - E(x) = (1-2x_m) g_m, all x, all m."""
    p = random_integer_problem(order, 8, seed, nterms=60)
    o = Oracle.from_problem(p)
    X = exhaustive_X(8)
    E = o.energy(X)
    G = o.field(X)
    t = np.arange(256)
    for m in range(8):
        flipped = t ^ (1 << m)
        assert np.array_equal(E[flipped] - E, (1 - 2 * X[:, m].astype(np.float64)) * G[:, m])


def test_field_special_cases():
    # at x = 0 the field is the linear coefficient: seating -1 everywhere, TSP 0 (min degree 3)
    assert np.all(Oracle.from_problem(seating(4)).field(np.zeros((1, 16), np.uint8)) == -1.0)
    assert np.all(Oracle.from_problem(tsp()).field(np.zeros((1, 6), np.uint8)) == 0.0)
    # at every ground state no single flip lowers the energy
    for p in (seating(4), pythagoras(), tsp()):
        o = Oracle.from_problem(p)
        g = o.brute()["ground"]
        X = ((g[:, None] >> np.arange(p.N)[None, :]) & 1).astype(np.uint8)
        assert np.all((1 - 2 * X.astype(np.float64)) * o.field(X) >= 0)


def test_field_matches_qubo_gradient_closed_form():
    """For a QUBO with upper-triangular Q: g_m = Q_mm + sum_{j != m} (Q_mj + Q_jm) x_j."""
    idx, val = uniform_cells(2, 40, 21)
    o = Oracle.from_cells(2, 40, idx, val)
    Q = o.dense().astype(np.float64)
    S = Q + Q.T
    np.fill_diagonal(S, 0)
    X = x_bits(9, 100, 40)
    ref = np.diag(Q)[None, :] + X.astype(np.float64) @ S
    assert np.allclose(o.field(X), ref, rtol=0, atol=1e-9 * o.sum_abs)


# ---- generators (known answers) -------------------------------------------------------------
def test_generator_known_answers(pins):
    g = pins["generator"]
    from workloads import splitmix64 as wl_splitmix64
    assert splitmix64(0) == int(g["splitmix64_0"], 16) == wl_splitmix64(0)
    assert hash4(1, 1, 0, 0) == int(g["h_1_1_0_0"], 16) == h(1, 1, 0, 0)
    X = x_bits(1, 2, 16)
    assert "".join(map(str, X[0])) == g["xbits_seed1_b0"] and "".join(map(str, X[1])) == g["xbits_seed1_b1"]
    _, v2 = uniform_cells(2, 1024, 2)
    idx2 = canonical_cells_all(2, 1024)
    pos = {tuple(r): i for i, r in enumerate(idx2[:3000].tolist())}
    assert v2[pos[(0, 0)]] == np.float32(g["U_2_00_1024"]) and v2[pos[(0, 1)]] == np.float32(g["U_2_01_1024"])
    q = (h(5, 0, 0 + 1 * 1024 + 2 * 1024 ** 2, 0) >> 40)
    assert (q - (1 << 23)) * 2.0 ** -23 == g["U_5_012_1024"]


def test_cfg1_known_answers(pins):
    o = Oracle.from_problem(seating(4))
    E = o.energy(x_bits(1, 1024, 16))
    c = pins["cfg1"]
    assert E[:8].tolist() == c["E_head"] and E.sum() == c["E_sum"]
    assert int(np.argmin(E)) == c["argmin"] and E.min() == c["emin"] and (E == E.min()).sum() == 1


def test_cfg2_known_answers(pins):
    c = pins["cfg2"]
    X = x_bits(2, 4, 1024)
    o = Oracle.from_cells(2, 1024, *uniform_cells(2, 1024, 2))
    assert np.allclose(o.energy(X), c["E_head"], rtol=0, atol=1e-9)
    assert abs(o.sum_abs - c["sum_abs"]) < 0.01
    t = Oracle.from_cells(2, 1024, *int_twin_cells(2, 1024, 2))
    assert t.energy(X).tolist() == c["twin_E_head"] and t.sum_abs == c["twin_sum_abs"]


def test_cfg3_known_answers(pins):
    c = pins["cfg3"]
    o = Oracle.from_problem(cfg3_problem())
    deg, _, val = o.monomials()
    assert o.ncells == c["ncells"] and np.bincount(deg, minlength=4)[1:].tolist() == c["by_degree"]
    assert o.sum_abs == c["sum_abs"] and np.abs(val).max() == c["max_abs"] and o.offset == c["offset"]
    assert o.is_integer and o.sum_abs < 2 ** 24


# ---- search replay rule ------------------------------------------------------------------
def test_search_thresholds():
    P = search_thresholds(64, 0.5, 0.005)
    assert P[0] == 2 ** 31 and P[-1] == int(np.floor(2 ** 32 * 0.005))
    assert np.all(np.diff(P.astype(np.int64)) <= 0)
    assert search_thresholds(1, 0.5, 0.005).tolist() == [2 ** 31]


def test_search_oracle_finds_brute_optimum_and_is_honest():
    o = Oracle.from_problem(seating(4))
    r = o.search(1, 0, 1024, 64)
    assert r["e_best"] == -11.0
    xb = r["chain_xbest"]
    assert np.array_equal(o.energy(xb), r["chain_ebest"])        # energy honesty
    # chain-sharding invariance: two halves give the same per-chain results
    a, b = o.search(1, 0, 512, 64), o.search(1, 512, 512, 64)
    assert np.array_equal(np.concatenate([a["chain_ebest"], b["chain_ebest"]]), r["chain_ebest"])
    # iters = 0 returns the best random initial candidate
    r0 = o.search(1, 0, 1024, 0)
    X0 = np.stack([[(hash4(1, 1, c, m >> 6) >> (m & 63)) & 1 for m in range(16)] for c in range(1024)]).astype(np.uint8)
    E0 = o.energy(X0)
    assert r0["e_best"] == E0.min() and r0["best_chain"] == int(np.argmin(E0))


def test_search_rule_golden_trace():
    """O8 against a hand-checkable trace written from the rule text (tests/golden/search_trace.json,
    tests/golden/make_search_trace.py): every state, flipped site and per-chain best of 2 chains x 4
    iterations.  The trace exercises each branch a plausible slip would change: the strict
    "(r>>32) < P_t" (chain 0, t=0 sits exactly on P_0), the lowest-m tie-break (chain 1, t=3), the
    "Delta_min >= 0 -> random" fallback (Delta_min = 0 at chain 1, t=1) and the earliest-t best on
    an equal-energy revisit (chain 1: E=-1 at t=1 and t=4, different states)."""
    import json
    import os
    from workloads import TermBuilder
    with open(os.path.join(os.path.dirname(__file__), "golden", "search_trace.json")) as f:
        g = json.load(f)
    assert all(g["coverage"].values())
    tb = TermBuilder()
    for c, S in g["monomials"]:
        tb.add(float(c), [(0.0, [(v, 1.0)]) for v in S])
    o = Oracle.from_problem(tb.problem(g["order"], g["N"]))
    X = exhaustive_X(g["N"])
    for t, e in zip(range(16), o.energy(X)):
        assert g["energy_table"]["".join(str((t >> m) & 1) for m in range(4))] == e
    assert search_thresholds(g["iters"], g["p0"], g["p1"]).tolist() == g["P"]
    r = o.search_trace(g["seed"], 0, g["nchains"], g["iters"], g["p0"], g["p1"])
    for i, ch in enumerate(g["chains"]):
        assert r["x_trace"][i].tolist() == [s["x"] for s in ch["steps"]], f"chain {i} states"
        assert r["m_trace"][i].tolist() == [s["m_star"] for s in ch["steps"][:-1]], f"chain {i} moves"
        assert r["chain_ebest"][i] == ch["E_best"] and r["chain_xbest"][i].tolist() == ch["x_best"]
    best = min((ch["E_best"], ch["chain"]) for ch in g["chains"])
    assert (r["e_best"], r["best_chain"]) == best
    # the plain search returns the same per-chain results as its traced form
    r2 = o.search(g["seed"], 0, g["nchains"], g["iters"], g["p0"], g["p1"])
    assert np.array_equal(r2["chain_xbest"], r["chain_xbest"]) and np.array_equal(r2["chain_ebest"], r["chain_ebest"])


# ---- the colex-array oracle entry points used at full size ----------------------------------
def test_colex_energy_qubo_closed_form():
    """E = x^T Q x with Q_ii = c({i}), Q_ij = c({i,j}) (i<j): numpy float64 matmul."""
    from oracle import colex_energy
    from workloads import colex_rank, uniform_colex
    N = 48
    v = uniform_colex(2, N, 31)
    Q = np.zeros((N, N))
    for i in range(N):
        Q[i, i] = v[0][i]
        for j in range(i + 1, N):
            Q[i, j] = v[1][colex_rank([i, j])]
    X = x_bits(5, 200, N)
    ref = np.einsum("bi,ij,bj->b", X.astype(np.float64), Q, X.astype(np.float64))
    assert np.allclose(colex_energy(2, N, v, X), ref, rtol=0, atol=1e-9 * np.abs(Q).sum())


@pytest.mark.parametrize("order", [3, 4])
def test_colex_field_flip_identity(order):
    from oracle import colex_energy, colex_field
    from workloads import int_twin_colex
    N = 9
    v = int_twin_colex(order, N, 17)
    X = exhaustive_X(N)
    E = colex_energy(order, N, v, X)
    G = colex_field(order, N, v, X)
    t = np.arange(1 << N)
    for m in range(N):
        assert np.array_equal(E[t ^ (1 << m)] - E, (1 - 2 * X[:, m].astype(np.float64)) * G[:, m])


def test_colex_matches_cell_list():
    from oracle import colex_energy, colex_field
    from workloads import uniform_colex
    v = uniform_colex(3, 26, 4)
    o = Oracle.from_cells(3, 26, *uniform_cells(3, 26, 4))
    X = x_bits(2, 64, 26)
    assert np.array_equal(colex_energy(3, 26, v, X), o.energy(X))
    assert np.array_equal(colex_field(3, 26, v, X), o.field(X))


# ---- result aggregation (SPEC S:472-480 examples) ---------------------------------------------
def test_aggregate_examples():
    from oracle import aggregate
    r = aggregate(np.array([[0, 1], [0, 1], [1, 0]], np.uint8), [-1.0, -1.0, 0.0])
    assert [(x.tolist(), e, c) for x, e, c in r] == [([0, 1], -1.0, 2), ([1, 0], 0.0, 1)]
    assert aggregate(np.zeros((0, 3), np.uint8), []) == []
    # ties in energy: occurrence descending, then assignment lexicographic
    r = aggregate(np.array([[1, 0], [0, 1], [0, 1], [1, 1]], np.uint8), [0.0, 0.0, 0.0, 0.0])
    assert [(x.tolist(), c) for x, _, c in r] == [([0, 1], 2), ([1, 0], 1), ([1, 1], 1)]


def test_aggregate_occurrences_sum_to_shots():
    from oracle import aggregate
    o = Oracle.from_problem(tsp())
    r = o.search(3, 0, 500, 8)
    agg = aggregate(r["chain_xbest"], r["chain_ebest"])
    assert sum(c for _, _, c in agg) == 500
    assert agg[0][1] == r["e_best"] == -360.0
    for x, e, _ in agg:
        assert o.energy(x[None])[0] == e          # energy honesty


# ---- multilinear relaxation (gradient descent) ----------------
def test_menergy_is_the_multilinear_extension():
    """E(p) = sum over all binary x of E(x) prod p^x (1-p)^(1-x): the expectation of the
    (pinned) binary energy under independent Bernoulli(p) bits, exhaustively for N = 9."""
    p_ = random_integer_problem(3, 9, 12, nterms=80)
    o = Oracle.from_problem(p_)
    X = exhaustive_X(9).astype(np.float64)
    Ex = o.energy(X.astype(np.uint8))
    rng = np.random.default_rng(1)
    P = rng.random((20, 9))
    w = np.prod(np.where(X[None, :, :] == 1, P[:, None, :], 1 - P[:, None, :]), axis=2)   # 20 x 512
    assert np.allclose(o.menergy(P), w @ Ex, rtol=0, atol=1e-9 * o.sum_abs)


def test_mfield_central_differences():
    """the gradient matches central finite differences of E(p)."""
    idx, val = uniform_cells(4, 10, 3)
    o = Oracle.from_cells(4, 10, idx, val)
    rng = np.random.default_rng(2)
    P = rng.random((6, 10))
    G = o.mfield(P)
    h_ = 1e-5
    for m in range(10):
        Pp, Pm = P.copy(), P.copy()
        Pp[:, m] += h_
        Pm[:, m] -= h_
        fd = (o.menergy(Pp) - o.menergy(Pm)) / (2 * h_)
        assert np.allclose(G[:, m], fd, rtol=1e-6, atol=1e-7 * o.sum_abs)


def test_mfield_qubo_closed_form_and_binary_points():
    idx, val = uniform_cells(2, 30, 8)
    o = Oracle.from_cells(2, 30, idx, val)
    Q = o.dense().astype(np.float64)
    S = Q + Q.T
    np.fill_diagonal(S, 0)
    P = np.random.default_rng(3).random((7, 30))
    assert np.allclose(o.mfield(P), np.diag(Q)[None, :] + P @ S, rtol=0, atol=1e-9 * o.sum_abs)
    X = x_bits(4, 50, 30)
    assert np.array_equal(o.mfield(X.astype(np.float64)), o.field(X))
    assert np.array_equal(o.menergy(X.astype(np.float64)), o.energy(X))


# ---- simulated annealing (SPEC sa_run) -------------------------
def test_sa_temps_geometric_endpoints():
    from oracle import sa_temps
    T = sa_temps(5, 100.0, 0.01)
    assert T[0] == 100.0 and abs(T[-1] - 0.01) < 1e-15 and np.allclose(T[1:] / T[:-1], 0.1)
    assert sa_temps(1, 3.0, 1.0)[0] == 3.0


@pytest.mark.parametrize("maker", [lambda: seating(4), pythagoras, lambda: random_integer_problem(3, 14, 8, 60)])
def test_sa_infinite_temperature_flips_every_bit(maker):
    """T -> inf: min(1, exp(-d/T)) = 1, every proposal is accepted, so one sweep maps x to 1-x
    and the tracked energy must equal the fresh energy of 1-x."""
    o = Oracle.from_problem(maker())
    xs, es = o.sa(5, 0, 16, 1, 1e300, 1e300)
    x0 = np.array([[(h(5, 1, c, m >> 6) >> np.uint64(m & 63)) & np.uint64(1) for m in range(o.N)]
                   for c in range(16)], dtype=np.uint8)
    assert np.array_equal(xs, 1 - x0)
    assert np.array_equal(es, o.energy(1 - x0))


@pytest.mark.parametrize("maker", [lambda: seating(4), pythagoras, lambda: random_integer_problem(4, 12, 3, 80)])
def test_sa_zero_temperature_is_monotone_and_honest(maker):
    """T -> 0: only d <= 0 moves are accepted, so energies never rise from one sweep to the next
    (a run of s+1 sweeps extends the run of s sweeps: same counters, same T)."""
    o = Oracle.from_problem(maker())
    prev = None
    for s in range(0, 5):
        xs, es = o.sa(9, 0, 32, s, 1e-300, 1e-300)
        assert np.array_equal(es, o.energy(xs))
        if prev is not None:
            assert np.all(es <= prev)
        prev = es
    # converged chains sit in single-flip local minima
    G = o.field(xs)
    assert np.all((1 - 2 * xs.astype(np.float64)) * G >= 0)


def test_sa_replay_by_energy_differences():
    """The sweep rule replayed with d = E(x with x_m flipped) - E(x) from exhaustive energy
    evaluation (no local field), on a small integer instance."""
    import math
    p = random_integer_problem(3, 8, 21, 40)
    o = Oracle.from_problem(p)
    Eall = o.energy(exhaustive_X(o.N))
    idx = lambda x: int(sum(int(v) << m for m, v in enumerate(x)))  # noqa: E731
    T = [4.0 * (0.05 / 4.0) ** (s / 2) for s in range(3)]
    xs, es = o.sa(13, 3, 6, 3, 4.0, 0.05)
    for i, c in enumerate(range(3, 9)):
        x = [int((h(13, 1, c, 0) >> np.uint64(m)) & np.uint64(1)) for m in range(o.N)]
        for s in range(3):
            for m in range(o.N):
                y = list(x)
                y[m] ^= 1
                d = Eall[idx(y)] - Eall[idx(x)]
                u = int(h(13, 4, c, s * o.N + m) >> np.uint64(11)) * 2.0 ** -53
                if d <= 0 or u < math.exp(-d / T[s]):      # min(1, exp(-dE/T))
                    x = y
        assert list(xs[i]) == x and es[i] == Eall[idx(x)]


def test_sa_acceptance_is_the_metropolis_probability():
    """The oracle's acceptance decision (log form) equals SPEC's min(1, exp(-d/T)) test
    (S:450), u < exp(-d/T), on a grid of (d, T, u) away from the decision boundary."""
    import math
    from oracle import sa_accept
    rng = np.random.default_rng(5)
    n = 0
    for d in np.concatenate([[-3.0, -0.5, 0.0, 1e-9], rng.uniform(-5, 40, 60)]):
        for T in (1e-3, 0.05, 0.7, 3.0, 25.0, 1e4):
            for u in np.concatenate([[1e-300, 2.0 ** -53, 0.5, 1 - 2.0 ** -53], rng.random(20)]):
                ref = bool(d <= 0 or u < math.exp(-d / T))
                if d > 0 and abs(u - math.exp(-d / T)) <= 1e-12 * max(u, 1e-300):
                    continue                      # on the boundary the two forms may round apart
                assert sa_accept(float(d), T, float(u)) == ref, (d, T, u)
                n += 1
    assert n > 9000


def test_sa_spec_examples():
    """SPEC sa_run examples: H = q0 -> q0 = 0 at energy 0; the three paper problems reach
    their brute-force ground energies (-11 seating 4x4, -30 Pythagoras P:322, -360 TSP P:402)."""
    from workloads import TermBuilder
    tb = TermBuilder()
    tb.add(1.0, [(0.0, [(0, 1.0)])])
    o = Oracle.from_problem(tb.problem(1, 1))
    xs, es = o.sa(1, 0, 100, 1000, 10.0, 0.01)
    assert np.all(xs == 0) and np.all(es == 0)
    for p, emin in [(seating(4), -11.0), (pythagoras(), -30.0), (tsp(), -360.0)]:
        o = Oracle.from_problem(p)
        _, v = o.cells()
        xs, es = o.sa(7, 0, 1000, 200, 10 * float(np.abs(v).max()), 0.01)
        assert es.min() == emin == o.brute()["emin"]
        assert np.array_equal(o.energy(xs), es)
