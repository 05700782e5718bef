"""CPU tests of the product's host side: the C-ABI library loads and exports every symbol
of include/hobo.h, and its compiler (hobo_tensor_build / import_cells) produces exactly the
oracle's canonical cells.  No GPU compute is called here."""
import os
import re

import numpy as np
import pytest

from oracle import Oracle
from workloads import (TermBuilder, cfg3_problem, int_twin_cells, pythagoras, random_integer_problem,
                       seating, tsp, uniform_cells)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def H():
    from paper_2407_19987_b200 import build
    build.build()
    from paper_2407_19987_b200 import hobo
    return hobo


def test_library_exports_every_header_symbol(H):
    import ctypes
    hdr = open(os.path.join(ROOT, "include", "hobo.h")).read()
    names = set(re.findall(r"^\s*(?:hobo_status|const char\*)\s+(hobo_\w+)\s*\(", hdr, re.M))
    assert len(names) >= 12
    L = H.lib()
    for n in names:
        assert hasattr(L, n), n
    assert set(H.EXPORTED) == names
    # the library must link no oracle code
    so = open(H.LIB_PATH, "rb").read()
    assert b"or_energy" not in so and b"hobo_oracle" not in so
    assert isinstance(ctypes.CDLL(H.LIB_PATH), ctypes.CDLL)


def _same_cells(t, o):
    i1, v1 = t.cells()
    i2, v2 = o.cells()
    assert np.array_equal(i1, i2)
    assert np.array_equal(v1.view(np.uint32), v2.view(np.uint32))   # bit-exact fp32 cells


@pytest.mark.parametrize("maker", [lambda: seating(5), pythagoras, tsp, cfg3_problem,
                                   lambda: random_integer_problem(3, 20, 5, 200),
                                   lambda: random_integer_problem(4, 9, 6, 300),
                                   lambda: random_integer_problem(2, 30, 7, 400)])
def test_build_matches_oracle_cells(H, maker):
    p = maker()
    t = H.HoboTensor.from_problem(p)
    o = Oracle.from_problem(p)
    _same_cells(t, o)
    assert t.offset == o.offset and t.ncells == o.ncells
    assert t.is_integer == o.is_integer and t.sum_abs == o.sum_abs


def test_build_non_integer_terms_matches_oracle(H):
    rng = np.random.default_rng(3)
    tb = TermBuilder()
    for _ in range(300):
        k = int(rng.integers(0, 4))
        facs = []
        for _ in range(k):
            if rng.random() < 0.5:
                facs.append((float(rng.normal()), [(int(rng.integers(0, 12)), float(rng.normal()))]))
            else:
                facs.append((0.0, [(int(rng.integers(0, 12)), 1.0)]))
        tb.add(float(rng.normal()), facs)
    p = tb.problem(3, 12)
    t, o = H.HoboTensor.from_problem(p), Oracle.from_problem(p)
    i1, v1 = t.cells()
    i2, v2 = o.cells()
    assert np.array_equal(i1, i2)
    # both expand in long double and round once; allow 1 ulp where the summation order differs
    assert np.all(np.abs(v1.view(np.int32) - v2.view(np.int32)) <= 1)
    assert abs(t.offset - o.offset) <= 1e-12 * max(1, abs(o.offset))


@pytest.mark.parametrize("order,N,seed,kind", [(2, 64, 2, "u"), (3, 24, 5, "u"), (4, 10, 4, "u"), (3, 30, 9, "int")])
def test_import_cells_matches_oracle(H, order, N, seed, kind):
    idx, val = (uniform_cells if kind == "u" else int_twin_cells)(order, N, seed)
    # scramble index order inside each cell: import must canonicalise by index set
    rng = np.random.default_rng(seed)
    idx = np.take_along_axis(idx, rng.permuted(np.tile(np.arange(order), (len(idx), 1)), axis=1), axis=1)
    t = H.HoboTensor.import_cells(order, N, idx, val)
    o = Oracle.from_cells(order, N, idx, val)
    _same_cells(t, o)


def test_dense_export_matches_oracle(H):
    p = tsp()
    assert np.array_equal(H.HoboTensor.from_problem(p).dense(), Oracle.from_problem(p).dense())


def test_limb_counts(H):
    assert H.HoboTensor.from_problem(seating(4)).limbs == 1
    assert H.HoboTensor.from_problem(tsp()).limbs == 1
    assert H.HoboTensor.from_problem(cfg3_problem()).limbs == 1
    assert H.HoboTensor.from_problem(pythagoras()).limbs == 2     # 14-bit coefficients
    assert H.HoboTensor.import_cells(3, 20, *uniform_cells(3, 20, 1)).limbs == 3


def test_int8_digit_decomposition(H):
    """The fixed-point grid behind the int8 path (host side, no GPU): U(-1,1) cells are
    (q - 2^23) 2^-23, so 3 bytes at 2^-23; cfg3's integer cells (|c| <= 1216, lowest set bit
    2^0 somewhere) need 2 bytes at 2^0; seating's +10 cubic cells fit 1 byte (the -1 cells
    are degree 1, held in fp32 beside the planes); a 2^-62-quantum cell next to O(1) cells
    fits no 3-byte grid."""
    assert H.HoboTensor.import_cells(3, 20, *uniform_cells(3, 20, 1)).digits() == (3, -23)
    assert H.HoboTensor.from_problem(cfg3_problem()).digits() == (2, 0)
    d, q = H.HoboTensor.from_problem(seating(4)).digits()
    assert d == 1 and 10 * 2.0 ** -q < 128 and (10 * 2.0 ** -q) == int(10 * 2.0 ** -q)
    idx, val = uniform_cells(2, 16, 3)
    val = val.copy()
    val[np.flatnonzero(idx[:, 0] != idx[:, 1])[0]] = np.float32(3.0e-12)
    assert H.HoboTensor.import_cells(2, 16, idx, val).digits()[0] == 0
    # exactness of the decomposition: every cell = q 2^qexp with q in the d-byte range
    idx, val = uniform_cells(3, 24, 5)
    t = H.HoboTensor.import_cells(3, 24, idx, val)
    d, q = t.digits()
    deg = np.array([len(set(r)) for r in idx])
    qs = val[deg >= 2].astype(np.float64) * 2.0 ** -q
    assert np.array_equal(qs, np.round(qs)) and qs.min() >= -2 ** (8 * d - 1) and qs.max() <= 2 ** (8 * d - 1) - 1


def test_errors(H):
    tb = TermBuilder()
    tb.add(1.0, [(0.0, [(0, 1.0)]), (0.0, [(1, 1.0)]), (0.0, [(2, 1.0)])])
    p = tb.problem(2, 3)                    # degree 3 > order 2
    with pytest.raises(H.HoboError) as e:
        H.HoboTensor.from_problem(p)
    assert e.value.status == H.HOBO_EINVAL
    tb = TermBuilder()
    tb.add(1.0, [(0.0, [(5, 1.0)])])        # id outside [0, N)
    with pytest.raises(H.HoboError):
        H.HoboTensor.from_problem(tb.problem(2, 3))
    tb = TermBuilder()
    tb.add(float("nan"), [(0.0, [(0, 1.0)])])
    with pytest.raises(H.HoboError):
        H.HoboTensor.from_problem(tb.problem(2, 3))
    tb = TermBuilder()
    tb.add(1e300, [(0.0, [(0, 1.0)])])
    with pytest.raises(H.HoboError) as e:
        H.HoboTensor.from_problem(tb.problem(2, 3))
    assert e.value.status == H.HOBO_ERANGE
    # cancellation to zero is fine even above the order
    tb = TermBuilder()
    tb.add(1.0, [(0.0, [(i, 1.0)]) for i in range(4)])
    tb.add(-1.0, [(0.0, [(i, 1.0)]) for i in range(4)])
    tb.add(2.0, [(0.0, [(0, 1.0)])])
    assert H.HoboTensor.from_problem(tb.problem(2, 4)).ncells == 1


def test_tt_build_reproduces_paper_core_shapes(H, pins):
    """the TSP tensor (6,)*6 decomposes without approximation into cores
    [(6,2),(2,6,3),(3,6,4),(4,6,4),(4,6,2),(2,6)] — the product's own Jacobi TT-SVD."""
    t = H.HoboTensor.from_problem(tsp())
    r = t.tt_build(0.0)
    shapes = [[6, r[1]]] + [[r[p], 6, r[p + 1]] for p in range(1, 5)] + [[r[5], 6]]
    assert shapes == pins["tt_core_shapes_tsp"]["value"] and r[0] == r[6] == 1


def test_dist_entry_points_validate_arguments(H):
    """Multi-GPU communicator calls: argument checks happen before any NCCL or CUDA work."""
    assert H.dist_info() == (0, 1)
    for rank, world in ((1, 1), (-1, 2), (0, 0)):
        with pytest.raises(H.HoboError) as e:
            H.dist_init(rank, world, bytes(128), 0)
        assert e.value.status == H.HOBO_EINVAL
    H.dist_finalize()                      # no communicator: a no-op
    assert H.dist_info() == (0, 1)


@pytest.mark.parametrize("maker", [tsp, lambda: seating(4), lambda: random_integer_problem(3, 12, 2, 150)])
def test_import_dense_round_trip(H, maker):
    """Export the dense N^k tensor, import it back: the same canonical cells, bit for bit."""
    p = maker()
    t = H.HoboTensor.from_problem(p)
    back = H.HoboTensor.import_dense(t.order, t.N, t.dense())
    i1, v1 = t.cells()
    i2, v2 = back.cells()
    assert np.array_equal(i1, i2) and np.array_equal(v1.view(np.uint32), v2.view(np.uint32))


def test_import_dense_canonicalises_like_the_oracle(H):
    """A raw (non-canonical) dense tensor: every cell lands on the canonical cell of its index
    set, the same cells the oracle builds from the same raw cells."""
    rng = np.random.default_rng(9)
    order, N = 3, 7
    dense = np.where(rng.random((N,) * order) < 0.2, rng.integers(-5, 6, (N,) * order), 0).astype(np.float32)
    t = H.HoboTensor.import_dense(order, N, dense)
    nz = np.argwhere(dense != 0).astype(np.int32)
    o = Oracle.from_cells(order, N, nz, dense[tuple(nz.T)])
    _same_cells(t, o)


def test_pack_rows_bit_order(H):
    """hobo_*_bits row format (include/hobo.h): bit (m mod 32) of word m/32 is x_m, LSB first,
    pad bits zero.  Checked against the definition written out with Python integers."""
    rng = np.random.default_rng(5)
    for N in (1, 31, 32, 33, 300, 512):
        X = (rng.random((7, N)) < 0.5).astype(np.uint8)
        X[0] = 0
        X[1] = 1
        P = H.pack_rows(X * 3)                                      # any nonzero byte is a 1
        assert P.dtype == np.uint32 and P.shape == (7, (N + 31) // 32)
        for b in range(7):
            for w in range(P.shape[1]):
                want = sum(int(X[b, m]) << (m - 32 * w) for m in range(32 * w, min(N, 32 * w + 32)))
                assert int(P[b, w]) == want

