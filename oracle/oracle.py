"""ctypes binding of oracle/liboracle.so (plain C++17, see hobo_oracle.cpp).

TEST INFRASTRUCTURE: imported only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / reference legs.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "hobo_oracle.cpp")


def build_oracle_lib(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", _LIB, _SRC, "-lpthread"])
    return _LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build_oracle_lib())
        P, I64, U64, D, I = C.c_void_p, C.c_int64, C.c_uint64, C.c_double, C.c_int
        _lib.or_build.argtypes = [I, I, P, I64, P, P, C.POINTER(P), C.POINTER(D)]
        _lib.or_from_cells.argtypes = [I, I, I64, P, P, C.POINTER(P)]
        _lib.or_free.argtypes = [P]
        _lib.or_free.restype = None
        _lib.or_info.argtypes = [P, C.POINTER(I), C.POINTER(I), C.POINTER(I64), C.POINTER(I), C.POINTER(D)]
        _lib.or_cells.argtypes = [P, P, P]
        _lib.or_monomials.argtypes = [P, P, P, P]
        _lib.or_export_dense.argtypes = [P, P]
        _lib.or_energy.argtypes = [P, P, I64, P, I]
        _lib.or_energy_tensor.argtypes = [P, P, I64, P]
        _lib.or_field.argtypes = [P, P, I64, P, I]
        _lib.or_brute.argtypes = [P, C.POINTER(D), C.POINTER(I64), C.POINTER(I64), C.POINTER(D), P, I64, I]
        _lib.or_search.argtypes = [P, U64, I64, I64, I64, D, D, P, P, C.POINTER(D), C.POINTER(I64), I]
        _lib.or_hash.argtypes = [U64, U64, U64, U64]
        _lib.or_hash.restype = U64
        _lib.or_splitmix64.argtypes = [U64]
        _lib.or_splitmix64.restype = U64
        _lib.or_search_thresholds.argtypes = [I64, D, D, P]
        _lib.or_colex_energy.argtypes = [I, I, P, P, I64, P, I]
        _lib.or_menergy.argtypes = [P, P, I64, P, I]
        _lib.or_mfield.argtypes = [P, P, I64, P, I]
        _lib.or_colex_field.argtypes = [I, I, P, P, I64, P, I]
        _lib.or_sa.argtypes = [P, U64, I64, I64, I64, D, D, P, P, I]
        _lib.or_search_trace.argtypes = [P, U64, I64, I64, I64, D, D, P, P, C.POINTER(D), C.POINTER(I64), I, P, P]
        _lib.or_sa_accept.argtypes = [D, D, D]
        _lib.or_sa_temps.argtypes = [I64, D, D, P]
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def hash4(s, a, b, c) -> int:
    return int(_L().or_hash(s, a, b, c))


def splitmix64(z) -> int:
    return int(_L().or_splitmix64(z))


def search_thresholds(iters: int, p0: float = 0.5, p1: float = 0.005) -> np.ndarray:
    out = np.zeros(max(iters, 1), np.uint32)
    _L().or_search_thresholds(iters, p0, p1, _ptr(out))
    return out[:iters]


def _nthreads(n):
    return n if n else (os.cpu_count() or 1)


class Oracle:
    """Handle over the oracle's compiled problem (O1-O3)."""

    def __init__(self, handle, offset=0.0):
        self._h = handle
        self.offset = offset
        o, n, nc, ii, sa = C.c_int(), C.c_int(), C.c_int64(), C.c_int(), C.c_double()
        _L().or_info(self._h, C.byref(o), C.byref(n), C.byref(nc), C.byref(ii), C.byref(sa))
        self.order, self.N, self.ncells = o.value, n.value, nc.value
        self.is_integer, self.sum_abs = bool(ii.value), sa.value

    @classmethod
    def from_problem(cls, p):
        h, off = C.c_void_p(), C.c_double()
        st = _L().or_build(p.order, p.N, _ptr(p.terms), len(p.terms), _ptr(p.facs), _ptr(p.lins),
                           C.byref(h), C.byref(off))
        if st:
            raise ValueError(f"or_build failed with status {st}")
        return cls(h, off.value)

    @classmethod
    def from_cells(cls, order, N, idx, val):
        idx = np.ascontiguousarray(idx, np.int32)
        val = np.ascontiguousarray(val, np.float32)
        h = C.c_void_p()
        st = _L().or_from_cells(order, N, len(val), _ptr(idx), _ptr(val), C.byref(h))
        if st:
            raise ValueError(f"or_from_cells failed with status {st}")
        return cls(h, 0.0)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.or_free(self._h)
            self._h = None

    @property
    def tau(self):
        """Parity tolerance 1e-5 * sum |H| (BASELINE.json north_star)."""
        return 1e-5 * self.sum_abs

    def cells(self):
        idx = np.zeros((self.ncells, self.order), np.int32)
        val = np.zeros(self.ncells, np.float32)
        _L().or_cells(self._h, _ptr(idx), _ptr(val))
        return idx, val

    def monomials(self):
        deg = np.zeros(self.ncells, np.int32)
        var = np.zeros((self.ncells, self.order), np.int32)
        val = np.zeros(self.ncells, np.float32)
        _L().or_monomials(self._h, _ptr(deg), _ptr(var), _ptr(val))
        return deg, var, val

    def dense(self):
        out = np.zeros((self.N,) * self.order, np.float32)
        if _L().or_export_dense(self._h, _ptr(out)):
            raise MemoryError("dense export too large")
        return out

    def energy(self, X, nthreads=0):
        X = np.ascontiguousarray(X, np.uint8)
        E = np.zeros(X.shape[0], np.float64)
        _L().or_energy(self._h, _ptr(X), X.shape[0], _ptr(E), _nthreads(nthreads))
        return E

    def energy_tensor(self, X):
        X = np.ascontiguousarray(X, np.uint8)
        E = np.zeros(X.shape[0], np.float64)
        if _L().or_energy_tensor(self._h, _ptr(X), X.shape[0], _ptr(E)):
            raise MemoryError("tensor-form energy too large")
        return E

    def field(self, X, nthreads=0):
        X = np.ascontiguousarray(X, np.uint8)
        G = np.zeros((X.shape[0], self.N), np.float64)
        _L().or_field(self._h, _ptr(X), X.shape[0], _ptr(G), _nthreads(nthreads))
        return G

    def menergy(self, P, nthreads=0):
        """E(p) of the multilinear relaxation at real p (rows of P)."""
        P = np.ascontiguousarray(P, np.float64)
        E = np.zeros(P.shape[0], np.float64)
        _L().or_menergy(self._h, _ptr(P), P.shape[0], _ptr(E), _nthreads(nthreads))
        return E

    def mfield(self, P, nthreads=0):
        """dE/dp of the multilinear relaxation at real p."""
        P = np.ascontiguousarray(P, np.float64)
        G = np.zeros((P.shape[0], self.N), np.float64)
        _L().or_mfield(self._h, _ptr(P), P.shape[0], _ptr(G), _nthreads(nthreads))
        return G

    def brute(self, max_ground=64, nthreads=0):
        emin, arg, ng, nxt = C.c_double(), C.c_int64(), C.c_int64(), C.c_double()
        ground = np.zeros(max_ground, np.int64)
        st = _L().or_brute(self._h, C.byref(emin), C.byref(arg), C.byref(ng), C.byref(nxt), _ptr(ground),
                           max_ground, _nthreads(nthreads))
        if st:
            raise MemoryError("brute force too large")
        return dict(emin=emin.value, argmin=arg.value, n_ground=ng.value, next_level=nxt.value,
                    ground=ground[: min(ng.value, max_ground)])

    def search(self, seed, chain0, nchains, iters, p0=0.5, p1=0.005, nthreads=0):
        eb = np.zeros(nchains, np.float64)
        xb = np.zeros((nchains, self.N), np.uint8)
        e, c = C.c_double(), C.c_int64()
        st = _L().or_search(self._h, seed, chain0, nchains, iters, p0, p1, _ptr(eb), _ptr(xb),
                            C.byref(e), C.byref(c), _nthreads(nthreads))
        if st:
            raise ValueError(f"or_search status {st}")
        return dict(e_best=e.value, best_chain=c.value, chain_ebest=eb, chain_xbest=xb)

    def search_trace(self, seed, chain0, nchains, iters, p0=0.5, p1=0.005):
        """or_search with its trajectory: adds x_trace (nchains x (iters+1) x N, the state
        evaluated at each t) and m_trace (nchains x iters, the flipped site)."""
        eb = np.zeros(nchains, np.float64)
        xb = np.zeros((nchains, self.N), np.uint8)
        xt = np.zeros((nchains, iters + 1, self.N), np.uint8)
        mt = np.zeros((nchains, max(iters, 1)), np.int32)
        e, c = C.c_double(), C.c_int64()
        st = _L().or_search_trace(self._h, seed, chain0, nchains, iters, p0, p1, _ptr(eb), _ptr(xb),
                                  C.byref(e), C.byref(c), 1, _ptr(xt), _ptr(mt))
        if st:
            raise ValueError(f"or_search_trace status {st}")
        return dict(e_best=e.value, best_chain=c.value, chain_ebest=eb, chain_xbest=xb, x_trace=xt,
                    m_trace=mt[:, :iters])

    def sa(self, seed, chain0, nchains, sweeps, t_start, t_end, nthreads=0):
        """SPEC sa_run replayed per chain: (final states nchains x N, tracked energies)."""
        xs = np.zeros((nchains, self.N), np.uint8)
        es = np.zeros(nchains, np.float64)
        st = _L().or_sa(self._h, C.c_uint64(seed), chain0, nchains, sweeps, C.c_double(t_start), C.c_double(t_end),
                        _ptr(xs), _ptr(es), _nthreads(nthreads))
        if st:
            raise ValueError(f"or_sa status {st}")
        return xs, es


def sa_accept(d, T, u) -> bool:
    """The oracle's Metropolis acceptance decision (or_sa_accept)."""
    return bool(_L().or_sa_accept(C.c_double(d), C.c_double(T), C.c_double(u)))


def sa_temps(sweeps, t_start, t_end):
    out = np.zeros(max(1, sweeps), np.float64)
    if _L().or_sa_temps(sweeps, C.c_double(t_start), C.c_double(t_end), _ptr(out)):
        raise ValueError("bad schedule")
    return out


def _colex_ptrs(by_degree):
    arrs = [np.ascontiguousarray(a, np.float32) for a in by_degree]
    return arrs, (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def colex_energy(order, N, by_degree, X, nthreads=0):
    """Energies of candidates X from per-degree colex canonical cells (large instances)."""
    arrs, ptrs = _colex_ptrs(by_degree)
    X = np.ascontiguousarray(X, np.uint8)
    E = np.zeros(X.shape[0], np.float64)
    _L().or_colex_energy(order, N, C.cast(ptrs, C.c_void_p), _ptr(X), X.shape[0], _ptr(E), _nthreads(nthreads))
    return E


def colex_field(order, N, by_degree, X, nthreads=0):
    arrs, ptrs = _colex_ptrs(by_degree)
    X = np.ascontiguousarray(X, np.uint8)
    G = np.zeros((X.shape[0], N), np.float64)
    _L().or_colex_field(order, N, C.cast(ptrs, C.c_void_p), _ptr(X), X.shape[0], _ptr(G), _nthreads(nthreads))
    return G


def aggregate(xs, es, topk=None):
    """The sampler's result list ("Energy e, Occurrence n"):
    distinct assignments with occurrence counts, ordered by energy ascending, occurrence
    descending, assignment lexicographic (x_0 first).  xs: (n, N) u8, es: (n,) energies."""
    groups = {}
    for x, e in zip(np.asarray(xs, np.uint8), es):
        k = bytes(x)
        if k in groups:
            groups[k][1] += 1
        else:
            groups[k] = [float(e), 1]
    out = sorted(((e, -c, k) for k, (e, c) in groups.items()))
    res = [(np.frombuffer(k, np.uint8).copy(), e, -c) for e, c, k in out]
    return res if topk is None else res[:topk]
