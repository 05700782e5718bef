"""Input generators: the paper's worked problems (PAPER.md 5) and the BASELINE.json
configs, written in the term format, plus seeded candidate batches.

The hash is SURVEY.md 8(d):
    splitmix64(z): z += 0x9E3779B97F4A7C15; z = (z^(z>>30))*0xBF58476D1CE4E5B9;
                   z = (z^(z>>27))*0x94D049BB133111EB; return z^(z>>31)
    h(s,a,b,c)   = splitmix64(splitmix64(splitmix64(s^a)^b)^c)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "LIN", "FAC", "TERM", "Problem", "TermBuilder", "splitmix64", "h", "x_bits",
    "seating", "pythagoras", "tsp", "cfg3_problem", "uniform_cells", "int_twin_cells",
    "canonical_cells_all", "subsets", "random_integer_problem", "exhaustive_X",
    "paper_grids", "pyth_bits", "tsp_bits", "colex_subsets", "uniform_colex", "int_twin_colex",
    "colex_rank",
]

# memory layout of hobo_lin / hobo_factor / hobo_term (16 bytes each, natural alignment)
LIN = np.dtype([("var", "<i4"), ("w", "<f8")], align=True)
FAC = np.dtype([("c0", "<f8"), ("nlin", "<i4"), ("lin0", "<i4")], align=True)
TERM = np.dtype([("coeff", "<f8"), ("nfac", "<i4"), ("fac0", "<i4")], align=True)
assert LIN.itemsize == FAC.itemsize == TERM.itemsize == 16

_M64 = (1 << 64) - 1


def splitmix64(z):
    """Vectorised over numpy uint64 arrays, or a Python int."""
    if isinstance(z, (int, np.integer)) and not isinstance(z, np.ndarray):
        z = (int(z) + 0x9E3779B97F4A7C15) & _M64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def h(s, a, b, c):
    """h(s,a,b,c); any argument may be a numpy array (broadcast)."""
    if all(isinstance(v, (int, np.integer)) and not isinstance(v, np.ndarray) for v in (s, a, b, c)):
        return splitmix64(splitmix64(splitmix64(int(s) ^ int(a)) ^ int(b)) ^ int(c))
    u = lambda v: np.asarray(v, dtype=np.uint64)  # noqa: E731
    return splitmix64(splitmix64(splitmix64(u(s) ^ u(a)) ^ u(b)) ^ u(c))


def x_bits(seed: int, B: int, N: int, row0: int = 0) -> np.ndarray:
    """Candidates x_bm = (h(seed,1,b,m>>6) >> (m&63)) & 1, i.i.d. Bernoulli(1/2); u8 B x N."""
    nw = (N + 63) // 64
    b = np.arange(row0, row0 + B, dtype=np.uint64)[:, None]
    w = np.arange(nw, dtype=np.uint64)[None, :]
    words = h(seed, 1, b, w)                                   # B x nw uint64
    bits = np.unpackbits(words.astype("<u8").view(np.uint8).reshape(B, nw, 8), axis=2,
                         bitorder="little").reshape(B, nw * 64)
    return np.ascontiguousarray(bits[:, :N]).astype(np.uint8)


def exhaustive_X(N: int) -> np.ndarray:
    """All 2^N assignments, row t has x_m = (t >> m) & 1."""
    t = np.arange(1 << N, dtype=np.int64)[:, None]
    return ((t >> np.arange(N)[None, :]) & 1).astype(np.uint8)


@dataclass
class Problem:
    order: int
    N: int
    terms: np.ndarray = field(repr=False)
    facs: np.ndarray = field(repr=False)
    lins: np.ndarray = field(repr=False)
    name: str = ""


class TermBuilder:
    """Collects terms coeff * prod_f (c0_f + sum_l w_l x_{v_l}) (include/hobo.h)."""

    def __init__(self):
        self.terms, self.facs, self.lins = [], [], []

    def add(self, coeff, factors):
        """factors: list of (c0, [(var, w), ...])."""
        fac0 = len(self.facs)
        for c0, lin in factors:
            lin0 = len(self.lins)
            self.lins.extend((int(v), float(w)) for v, w in lin)
            self.facs.append((float(c0), len(lin), lin0))
        self.terms.append((float(coeff), len(factors), fac0))

    def problem(self, order, N, name=""):
        t = np.array(self.terms, dtype=TERM) if self.terms else np.zeros(0, TERM)
        f = np.array(self.facs, dtype=FAC) if self.facs else np.zeros(0, FAC)
        l = np.array(self.lins, dtype=LIN) if self.lins else np.zeros(0, LIN)
        return Problem(order, N, t, f, l, name)


def _var(v):
    return (0.0, [(v, 1.0)])


def seating(n: int = 5, weight: float = 10.0) -> Problem:
    """H = -sum q + weight * (row and column windows of 3), q row-major."""
    tb = TermBuilder()
    q = lambda i, j: i * n + j  # noqa: E731  symbols_list([n,n]) row-major
    for i in range(n):
        for j in range(n):
            tb.add(-1.0, [_var(q(i, j))])
    for i in range(n):
        for j in range(n - 3 + 1):
            tb.add(weight, [_var(q(i, j + d)) for d in range(3)])
    for j in range(n):
        for i in range(n - 3 + 1):
            tb.add(weight, [_var(q(i + d, j)) for d in range(3)])
    return tb.problem(3, n * n, f"seating{n}x{n}")


def _int_factor(bits_weights):
    return (0.0, list(bits_weights))


def pythagoras(weight: float = 10.0) -> Problem:
    """x,y,z 4-bit LSB-first; H = (x^2+y^2-z^2)^2 + weight*sum prod(1-q)."""
    tb = TermBuilder()
    q = lambda i, k: i * 4 + k  # noqa: E731
    X, Y, Z = ([(q(i, k), 2.0 ** k) for k in range(4)] for i in range(3))
    parts = [(X, 1.0), (Y, 1.0), (Z, -1.0)]
    for u, su in parts:            # (x*x + y*y - z*z)^2 as a sum of 4-factor products
        for v, sv in parts:
            tb.add(su * sv, [_int_factor(u), _int_factor(u), _int_factor(v), _int_factor(v)])
    for i in range(3):             # prod (1 - q[i,:])
        tb.add(weight, [(1.0, [(q(i, k), -1.0)]) for k in range(4)])
    return tb.problem(4, 12, "pythagoras")


def tsp(weight: float = 10.0) -> Problem:
    """xB=2q0_0+q0_1 ... (MSB-first), H = weight*(xB*xC*xD - 6)^2.
    Only q0_0..q2_1 are used; they are ids 0..5 and N = 6 (the (6,...,6) tensor of P:531)."""
    tb = TermBuilder()
    xs = [[(2 * i, 2.0), (2 * i + 1, 1.0)] for i in range(3)]
    B_, C_, D_ = (_int_factor(x) for x in xs)
    tb.add(weight, [B_, B_, C_, C_, D_, D_])       # (xB xC xD)^2
    tb.add(-12.0 * weight, [B_, C_, D_])           # -2*6*xB xC xD
    tb.add(36.0 * weight, [])                      # 6^2 (constant -> offset)
    return tb.problem(6, 6, "tsp")


# printed solutions of the paper, as bit vectors in the id order above
def paper_grids():
    """The three 5x5 grids printed at PAPER.md:227-243 (row-major bits)."""
    g = [
        [[1, 1, 0, 1, 1], [1, 1, 0, 1, 1], [0, 0, 1, 0, 0], [1, 1, 0, 1, 1], [1, 1, 0, 1, 1]],
        [[1, 1, 0, 1, 1], [0, 1, 1, 0, 1], [1, 0, 1, 1, 0], [1, 1, 0, 1, 1], [0, 1, 1, 0, 1]],
        [[1, 1, 0, 1, 1], [1, 0, 1, 1, 0], [0, 1, 1, 0, 1], [1, 1, 0, 1, 1], [1, 0, 1, 1, 0]],
    ]
    return np.array(g, dtype=np.uint8).reshape(3, 25)


def pyth_bits(x, y, z):
    return np.array([(v >> k) & 1 for v in (x, y, z) for k in range(4)], dtype=np.uint8)


def tsp_bits(b, c, d):
    return np.array([(v >> s) & 1 for v in (b, c, d) for s in (1, 0)], dtype=np.uint8)


def cfg3_problem() -> Problem:
    """BASELINE config 3 as restated in SURVEY.md 8(d): 128 integer variables y_a of 4 bits
    (bit 4a+t has weight 2^t, the width of PAPER.md:283-286), cubic/quadratic/linear terms."""
    tb = TermBuilder()
    y = lambda a: _int_factor([(4 * a + t, 2.0 ** t) for t in range(4)])  # noqa: E731

    def distinct(tag, t, k):
        vals, j = [], 0
        while len(vals) < k:
            v = h(3, tag, t, j) % 128
            if v not in vals:
                vals.append(v)
            j += 1
        return sorted(vals)

    for t in range(2048):
        a, b, c = distinct(10, t, 3)
        w = 1.0 if (h(3, 12, t, 0) & 1) else -1.0
        tb.add(w, [y(a), y(b), y(c)])
    w2tab = [-4, -3, -2, -1, 1, 2, 3, 4]
    for t in range(4096):
        a, b = distinct(11, t, 2)
        tb.add(float(w2tab[h(3, 13, t, 0) % 8]), [y(a), y(b)])
    for a in range(128):
        tb.add(float((h(3, 14, a, 0) % 33) - 16), [y(a)])
    return tb.problem(3, 512, "cfg3")


def int_encoded_problem(nvars: int, bits: int, ncubic: int, nquad: int, seed: int) -> Problem:
    """cfg3's recipe at other sizes: nvars integer variables of `bits` bits (bit t weighs 2^t),
    ncubic +-1 cubic and nquad {+-1..+-4} quadratic terms over distinct variables (tests only)."""
    tb = TermBuilder()
    y = lambda a: _int_factor([(bits * a + t, 2.0 ** t) for t in range(bits)])  # noqa: E731

    def distinct(tag, t, k):
        vals, j = [], 0
        while len(vals) < k:
            v = int(h(seed, tag, t, j) % np.uint64(nvars))
            if v not in vals:
                vals.append(v)
            j += 1
        return sorted(vals)

    for t in range(ncubic):
        a, b, c = distinct(10, t, 3)
        tb.add(1.0 if (h(seed, 12, t, 0) & 1) else -1.0, [y(a), y(b), y(c)])
    for t in range(nquad):
        a, b = distinct(11, t, 2)
        tb.add(float([-4, -3, -2, -1, 1, 2, 3, 4][int(h(seed, 13, t, 0) % np.uint64(8))]), [y(a), y(b)])
    return tb.problem(3, nvars * bits, f"intenc{nvars}x{bits}")


def subsets(N: int, r: int) -> np.ndarray:
    """All r-subsets of range(N) as sorted rows, lexicographic order, int32 (C(N,r) x r)."""
    if r == 0:
        return np.zeros((1, 0), np.int32)
    if r == 1:
        return np.arange(N, dtype=np.int32)[:, None]
    out = []
    for first in range(N - r + 1):
        rest = subsets(N - first - 1, r - 1) + (first + 1)
        out.append(np.concatenate([np.full((rest.shape[0], 1), first, np.int32), rest], axis=1))
    return np.concatenate(out, axis=0) if out else np.zeros((0, r), np.int32)


def canonical_cells_all(order: int, N: int):
    """Index tuples of every canonical cell (one per nonempty subset of size <= order),
    smallest index repeated at the front.  Returns int32 (n x order)."""
    rows = []
    for r in range(1, order + 1):
        s = subsets(N, r)
        rows.append(np.concatenate([np.repeat(s[:, :1], order - r, axis=1), s], axis=1))
    return np.ascontiguousarray(np.concatenate(rows, axis=0).astype(np.int32))


def _cell_ids(idx: np.ndarray, N: int) -> np.ndarray:
    cid = np.zeros(idx.shape[0], dtype=np.uint64)
    for p in range(idx.shape[1]):
        cid += idx[:, p].astype(np.uint64) * np.uint64(N ** p)
    return cid


def uniform_cells(order: int, N: int, seed: int):
    """Every canonical cell U(-1,1) on the 2^-23 grid: q = h(seed,0,cid,0)>>40,
    value = (q - 2^23) * 2^-23 with cid = sum_p i_p N^(p-1) (exact in fp32)."""
    idx = canonical_cells_all(order, N)
    q = (h(seed, 0, _cell_ids(idx, N), 0) >> np.uint64(40)).astype(np.int64)
    val = ((q - (1 << 23)).astype(np.float64) * 2.0 ** -23).astype(np.float32)
    return idx, val


def int_twin_cells(order: int, N: int, seed: int, mod: int = 17, shift: int = 8):
    """Integer twin: cell = (h(seed,0,cid,0) mod 17) - 8."""
    idx = canonical_cells_all(order, N)
    v = (h(seed, 0, _cell_ids(idx, N), 0) % np.uint64(mod)).astype(np.int64) - shift
    return idx, v.astype(np.float32)


def random_integer_problem(order: int, N: int, seed: int, nterms: int, maxc: int = 9,
                           with_affine: bool = True) -> Problem:
    """Random small-integer polynomial with affine factors (tests only)."""
    rng = np.random.default_rng(seed)
    tb = TermBuilder()
    for _ in range(nterms):
        deg = int(rng.integers(0, order + 1))
        facs = []
        for _ in range(deg):
            if with_affine and rng.random() < 0.3:
                k = min(int(rng.integers(1, 3)), N)
                vs = rng.choice(N, size=k, replace=False)
                facs.append((float(rng.integers(-1, 2)), [(int(v), float(rng.integers(-2, 3) or 1)) for v in vs]))
            else:
                facs.append(_var(int(rng.integers(0, N))))
        tb.add(float(rng.integers(-maxc, maxc + 1)), facs)
    return tb.problem(order, N, f"randint{order}_{N}")


def colex_subsets(n: int, r: int) -> np.ndarray:
    """All r-subsets of range(n) in colex order (sorted rows; max element slowest), int32."""
    if r == 0:
        return np.zeros((1, 0), np.int32)
    if n < r:
        return np.zeros((0, r), np.int32)
    parts = []
    for m in range(r - 1, n):
        head = colex_subsets(m, r - 1) if r > 1 else np.zeros((1, 0), np.int32)
        parts.append(np.concatenate([head, np.full((head.shape[0], 1), m, np.int32)], axis=1))
    return np.concatenate(parts, axis=0)


def colex_rank(s) -> int:
    """colex_rank({a1<...<ar}) = sum_i C(a_i, i) (the index used by import_colex)."""
    return sum(math.comb(int(a), i + 1) for i, a in enumerate(sorted(s)))


def _colex_values(order, N, seed, fn, chunk_rows=1 << 22):
    """Per-degree arrays over colex r-subsets (r = 1..order): value of the canonical cell
    (s1 repeated order-r+1 times, s2..sr) with cell id sum_p t_p N^p, from fn(cid)."""
    out = []
    pw = np.array([N ** p for p in range(order)], dtype=np.uint64)
    for r in range(1, order + 1):
        vals = np.empty(math.comb(N, r), np.float32)
        pos = 0
        # colex order = for each max element m: the colex (r-1)-subsets of [0, m), then m
        prev = colex_subsets(N, r - 1) if r > 1 else np.zeros((1, 0), np.int32)
        for m in range(r - 1, N):
            cnt = math.comb(m, r - 1)
            head = prev[:cnt].astype(np.uint64)          # colex prefix = subsets of [0, m)
            if r == 1:
                tup_first = np.full(1, m, np.uint64)
                cid = tup_first * pw.sum()
            else:
                s1 = head[:, 0]
                cid = s1 * pw[: order - r + 1].sum()
                for i in range(1, r - 1):
                    cid = cid + head[:, i] * pw[order - r + i]
                cid = cid + np.uint64(m) * pw[order - 1]
            vals[pos:pos + cnt] = fn(cid)
            pos += cnt
        out.append(vals)
    return out


def uniform_colex(order: int, N: int, seed: int):
    """The U(-1,1) canonical cells of uniform_cells(), as per-degree colex arrays."""
    def fn(cid):
        q = (h(seed, 0, cid, 0) >> np.uint64(40)).astype(np.int64)
        return ((q - (1 << 23)).astype(np.float64) * 2.0 ** -23).astype(np.float32)
    return _colex_values(order, N, seed, fn)


def int_twin_colex(order: int, N: int, seed: int, mod: int = 17, shift: int = 8):
    def fn(cid):
        return ((h(seed, 0, cid, 0) % np.uint64(mod)).astype(np.int64) - shift).astype(np.float32)
    return _colex_values(order, N, seed, fn)
