"""Thin ctypes binding of include/hobo.h (libhobo.so).  Argument marshalling only: every
step of the hot path runs in the library's CUDA kernels.  PyTorch provides device memory
and streams.  There is no CPU fallback: if the library is missing, importing raises."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "_lib", "libhobo.so")

HOBO_OK, HOBO_EINVAL, HOBO_ERANGE, HOBO_ENOMEM, HOBO_ECUDA, HOBO_ENCCL, HOBO_ESTATE = range(7)
_STATUS = {1: "EINVAL", 2: "ERANGE", 3: "ENOMEM", 4: "ECUDA", 5: "ENCCL", 6: "ESTATE"}

EXPORTED = [
    "hobo_tensor_build", "hobo_tensor_import_cells", "hobo_tensor_import_colex", "hobo_tensor_import_dense", "hobo_tensor_free", "hobo_tensor_info", "hobo_tensor_digits",
    "hobo_tensor_export_cells", "hobo_tensor_export_dense", "hobo_energy", "hobo_local_field", "hobo_local_field_host", "hobo_energy_host",
    "hobo_energy_bits", "hobo_local_field_bits", "hobo_energy_host_bits", "hobo_local_field_host_bits",
    "hobo_search", "hobo_search_shard", "hobo_search_samples", "hobo_multilinear_field",
    "hobo_gd_run", "hobo_tt_build", "hobo_tt_energy", "hobo_sa_shard", "hobo_sa_run", "hobo_last_launch_stats", "hobo_last_launch_kind",
    "hobo_set_profiling", "hobo_dist_unique_id", "hobo_dist_init", "hobo_dist_finalize", "hobo_dist_info",
    "hobo_shard", "hobo_shard_owner", "hobo_best_key", "hobo_best_from_key",
    "hobo_last_error",
]


class HoboError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class HoboBest(C.Structure):
    _fields_ = [("e", C.c_float), ("idx", C.c_int64)]


_lib = None


def lib():
    """Load libhobo.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2407_19987_b200.build` "
                              "(the HOBO hot path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P, I, I64, U64, D, SZ = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_double, C.c_size_t
        L.hobo_tensor_build.argtypes = [I, I, P, SZ, P, P, C.POINTER(P), C.POINTER(D)]
        L.hobo_tensor_import_cells.argtypes = [I, I, I64, P, P, C.POINTER(P)]
        L.hobo_tensor_import_colex.argtypes = [I, I, P, C.POINTER(P)]
        L.hobo_tensor_import_dense.argtypes = [I, I, P, C.POINTER(P)]
        L.hobo_tensor_free.argtypes = [P]
        L.hobo_tensor_digits.argtypes = [P, C.POINTER(I), C.POINTER(I)]
        L.hobo_tensor_info.argtypes = [P, C.POINTER(I), C.POINTER(I), C.POINTER(I64), C.POINTER(I),
                                       C.POINTER(D), C.POINTER(I), C.POINTER(D)]
        L.hobo_tensor_export_cells.argtypes = [P, P, P]
        L.hobo_tensor_export_dense.argtypes = [P, P]
        L.hobo_energy.argtypes = [P, P, I64, I64, P, C.POINTER(HoboBest), P]
        L.hobo_local_field.argtypes = [P, P, I64, I64, P, P, C.POINTER(HoboBest), P]
        L.hobo_local_field_host.argtypes = [P, P, I64, I64, P, P, C.POINTER(HoboBest), P]
        L.hobo_energy_host.argtypes = [P, P, I64, I64, P, C.POINTER(HoboBest), P]
        L.hobo_energy_bits.argtypes = [P, P, I64, I64, P, C.POINTER(HoboBest), P]
        L.hobo_local_field_bits.argtypes = [P, P, I64, I64, P, P, C.POINTER(HoboBest), P]
        L.hobo_energy_host_bits.argtypes = [P, P, I64, I64, P, C.POINTER(HoboBest), P]
        L.hobo_local_field_host_bits.argtypes = [P, P, I64, I64, P, P, C.POINTER(HoboBest), P]
        L.hobo_search.argtypes = [P, U64, I64, I64, P, C.POINTER(C.c_float), P]
        L.hobo_search_shard.argtypes = [P, U64, I64, I64, I64, D, D, P, C.POINTER(C.c_float),
                                        C.POINTER(I64), P]
        L.hobo_multilinear_field.argtypes = [P, P, I64, P, P, P]
        L.hobo_tt_build.argtypes = [P, D, P]
        L.hobo_tt_energy.argtypes = [P, P, I64, I64, P, C.POINTER(HoboBest), P]
        L.hobo_gd_run.argtypes = [P, U64, I64, I64, D, I64, I64, P, P, P, C.POINTER(I64), P]
        L.hobo_search_samples.argtypes = [P, U64, I64, I64, I64, P, P, P, C.POINTER(I64), P]
        L.hobo_sa_shard.argtypes = [P, U64, I64, I64, I64, D, D, P, P, P, P]
        L.hobo_sa_run.argtypes = [P, U64, I64, I64, D, D, I64, P, P, P, C.POINTER(I64), P]
        L.hobo_last_launch_stats.argtypes = [P, C.POINTER(I64), C.POINTER(D), C.POINTER(D), C.POINTER(D)]
        L.hobo_last_launch_kind.argtypes = [P, C.POINTER(I)]
        L.hobo_set_profiling.argtypes = [P, I]
        L.hobo_dist_unique_id.argtypes = [P]
        L.hobo_dist_init.argtypes = [I, I, P, I]
        L.hobo_dist_finalize.argtypes = []
        L.hobo_dist_info.argtypes = [C.POINTER(I), C.POINTER(I)]
        L.hobo_shard.argtypes = [I64, I, I, C.POINTER(I64), C.POINTER(I64)]
        L.hobo_shard_owner.argtypes = [I64, I, I64, C.POINTER(I)]
        L.hobo_best_key.argtypes = [C.c_float, I64, C.POINTER(U64)]
        L.hobo_best_from_key.argtypes = [U64, C.POINTER(HoboBest)]
        L.hobo_last_error.restype = C.c_char_p
        for name in EXPORTED:
            if name != "hobo_last_error":
                getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(st):
    if st != HOBO_OK:
        raise HoboError(st, lib().hobo_last_error().decode())


def _np_ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _stream_handle(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _dev_ptr(t, dtype, shape=None):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("expected a CUDA torch tensor")
    if t.dtype != dtype or not t.is_contiguous():
        raise TypeError(f"expected a contiguous {dtype} tensor, got {t.dtype}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"expected shape {shape}, got {tuple(t.shape)}")
    return C.c_void_p(t.data_ptr())


def pack_rows(X):
    """u8 candidates (numpy B x N, nonzero = 1) -> the packed rows the *_bits calls take:
    uint32 B x ceil(N/32), bit (m mod 32) of word m/32 = x_m.  Format conversion only."""
    X = np.ascontiguousarray(X)
    B, N = X.shape
    W = (N + 31) // 32
    Xp = np.zeros((B, W * 32), np.uint8)
    Xp[:, :N] = X != 0
    return np.packbits(Xp, axis=1, bitorder="little").view("<u4").reshape(B, W)


class HoboTensor:
    """Owner of one compiled problem (hobo_tensor*)."""

    def __init__(self, handle, offset=0.0):
        self._h = handle
        o, n, nc, ii, sa, lb, off = (C.c_int(), C.c_int(), C.c_int64(), C.c_int(), C.c_double(), C.c_int(),
                                     C.c_double())
        _check(lib().hobo_tensor_info(self._h, C.byref(o), C.byref(n), C.byref(nc), C.byref(ii), C.byref(sa),
                                      C.byref(lb), C.byref(off)))
        self.order, self.N, self.ncells = o.value, n.value, nc.value
        self.is_integer, self.sum_abs, self.limbs, self.offset = bool(ii.value), sa.value, lb.value, off.value

    def digits(self):
        """(digits, qexp): the cells of degree >= 2 are q * 2^qexp with q a `digits`-byte
        two's-complement integer (0: not representable in 3 bytes)."""
        d, q = C.c_int(), C.c_int()
        _check(lib().hobo_tensor_digits(self._h, C.byref(d), C.byref(q)))
        return d.value, q.value

    # -- construction ---------------------------------------------------------------------
    @classmethod
    def build(cls, order, N, terms, facs, lins):
        """hobo_tensor_build from numpy structured arrays (workloads.TERM/FAC/LIN layout)."""
        h, off = C.c_void_p(), C.c_double()
        _check(lib().hobo_tensor_build(order, N, _np_ptr(terms), len(terms), _np_ptr(facs), _np_ptr(lins),
                                       C.byref(h), C.byref(off)))
        return cls(h, off.value)

    @classmethod
    def from_problem(cls, p):
        return cls.build(p.order, p.N, p.terms, p.facs, p.lins)

    @classmethod
    def import_cells(cls, order, N, idx, val):
        idx = np.ascontiguousarray(idx, np.int32)
        val = np.ascontiguousarray(val, np.float32)
        h = C.c_void_p()
        _check(lib().hobo_tensor_import_cells(order, N, len(val), _np_ptr(idx), _np_ptr(val), C.byref(h)))
        return cls(h, 0.0)

    @classmethod
    def import_colex(cls, order, N, by_degree):
        """Canonical cells per degree r = 1..order, each a float32 array of C(N, r) in colex order."""
        arrs = [np.ascontiguousarray(a, np.float32) for a in by_degree]
        if len(arrs) != order:
            raise ValueError("need one array per degree 1..order")
        ptrs = (C.c_void_p * order)(*[a.ctypes.data for a in arrs])
        h = C.c_void_p()
        _check(lib().hobo_tensor_import_colex(order, N, C.cast(ptrs, C.c_void_p), C.byref(h)))
        return cls(h, 0.0)

    @classmethod
    def import_dense(cls, order, N, dense):
        """A dense N^order fp32 tensor (row-major, last index fastest), canonicalised by index set."""
        d = np.ascontiguousarray(dense, np.float32).reshape(-1)
        if d.size != N ** order:
            raise ValueError(f"expected {N}^{order} cells")
        h = C.c_void_p()
        _check(lib().hobo_tensor_import_dense(order, N, d.ctypes.data, C.byref(h)))
        return cls(h, 0.0)

    def close(self):
        if getattr(self, "_h", None):
            lib().hobo_tensor_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def tau(self):
        return 1e-5 * self.sum_abs

    # -- host exports -----------------------------------------------------------------------
    def cells(self):
        idx = np.zeros((self.ncells, self.order), np.int32)
        val = np.zeros(self.ncells, np.float32)
        _check(lib().hobo_tensor_export_cells(self._h, _np_ptr(idx), _np_ptr(val)))
        return idx, val

    def dense(self):
        out = np.zeros((self.N,) * self.order, np.float32)
        _check(lib().hobo_tensor_export_dense(self._h, _np_ptr(out)))
        return out

    # -- the hot path -------------------------------------------------------------------------
    def energy(self, X, E=None, row0=0, want_best=True, stream=None):
        """E_b for a CUDA u8 tensor X (B x N).  Returns (E, best) with best = (e, global idx)."""
        import torch
        B = X.shape[0]
        xp = _dev_ptr(X, torch.uint8, (B, self.N))
        if E is None:
            E = torch.empty(B, dtype=torch.float32, device=X.device)
        best = HoboBest()
        _check(lib().hobo_energy(self._h, xp, B, row0, _dev_ptr(E, torch.float32, (B,)),
                                 C.byref(best) if want_best else None, _stream_handle(stream)))
        return E, ((best.e, best.idx) if want_best else None)

    def local_field(self, X, G=None, E=None, row0=0, want_energy=True, want_best=False, stream=None):
        """G[b, m] = E(x_b | x_m=1) - E(x_b | x_m=0) (and E, and the argmin) for a CUDA u8 X.
        Returns (G, E) or, with want_best, (G, E, (e_best, global idx))."""
        import torch
        B = X.shape[0]
        xp = _dev_ptr(X, torch.uint8, (B, self.N))
        if G is None:
            G = torch.empty(B, self.N, dtype=torch.float32, device=X.device)
        if E is None and want_energy:
            E = torch.empty(B, dtype=torch.float32, device=X.device)
        best = HoboBest()
        _check(lib().hobo_local_field(self._h, xp, B, row0, _dev_ptr(G, torch.float32, (B, self.N)),
                                      _dev_ptr(E, torch.float32, (B,)) if E is not None else None,
                                      C.byref(best) if want_best else None, _stream_handle(stream)))
        return (G, E, (best.e, best.idx)) if want_best else (G, E)

    @staticmethod
    def _host_ptr(a, dtype, shape):
        """Host buffer address: a numpy array or a CPU torch tensor (ideally pinned)."""
        if a is None:
            return None
        if hasattr(a, "data_ptr"):
            if a.is_cuda or tuple(a.shape) != tuple(shape) or not a.is_contiguous() or \
                    a.element_size() != np.dtype(dtype).itemsize:
                raise ValueError(f"expected a contiguous CPU tensor of shape {shape} and {np.dtype(dtype)} width")
            return a.data_ptr()
        if a.dtype.itemsize != np.dtype(dtype).itemsize or a.dtype.kind != np.dtype(dtype).kind or \
                a.shape != tuple(shape) or not a.flags.c_contiguous:
            raise ValueError(f"expected a C-contiguous {np.dtype(dtype)} array of shape {shape}")
        return a.ctypes.data

    def local_field_host(self, X, E=None, row0=0, want_best=True, stream=None, fields=True, G=None):
        """hobo_local_field_host (fields=True) / hobo_energy_host (fields=False): candidates in
        host memory (numpy u8 B x N, or a CPU torch tensor, ideally pinned); energies into the
        host array E (f32, allocated if None); with G (host f32 B x N, ideally pinned) the local
        fields come back too.  Returns (E, best)."""
        B = X.shape[0]
        xp = self._host_ptr(X, np.uint8, (B, self.N))
        if E is None:
            E = np.empty(B, np.float32)
        ep = self._host_ptr(E, np.float32, (B,))
        best = HoboBest()
        bp = C.byref(best) if want_best else None
        if fields:
            _check(lib().hobo_local_field_host(self._h, xp, B, row0, self._host_ptr(G, np.float32, (B, self.N)), ep, bp,
                                               _stream_handle(stream)))
        else:
            if G is not None:
                raise ValueError("fields=False computes no fields")
            _check(lib().hobo_energy_host(self._h, xp, B, row0, ep, bp, _stream_handle(stream)))
        return E, ((best.e, best.idx) if want_best else None)

    def energy_host(self, X, E=None, row0=0, want_best=True, stream=None):
        return self.local_field_host(X, E, row0, want_best, stream, fields=False)

    # ---- packed candidates (hobo_*_bits): rows of ceil(N/32) words, see pack_rows ----
    def energy_bits(self, Xb, E=None, row0=0, want_best=True, stream=None):
        """hobo_energy_bits: E_b for a CUDA int32 tensor of packed rows (B x ceil(N/32))."""
        import torch
        B = Xb.shape[0]
        xp = _dev_ptr(Xb, torch.int32, (B, (self.N + 31) // 32))
        if E is None:
            E = torch.empty(B, dtype=torch.float32, device=Xb.device)
        best = HoboBest()
        _check(lib().hobo_energy_bits(self._h, xp, B, row0, _dev_ptr(E, torch.float32, (B,)),
                                      C.byref(best) if want_best else None, _stream_handle(stream)))
        return E, ((best.e, best.idx) if want_best else None)

    def local_field_bits(self, Xb, G=None, E=None, row0=0, want_best=False, stream=None):
        """hobo_local_field_bits: fields, energies (and the argmin) for packed CUDA rows."""
        import torch
        B = Xb.shape[0]
        xp = _dev_ptr(Xb, torch.int32, (B, (self.N + 31) // 32))
        if G is None:
            G = torch.empty(B, self.N, dtype=torch.float32, device=Xb.device)
        if E is None:
            E = torch.empty(B, dtype=torch.float32, device=Xb.device)
        best = HoboBest()
        _check(lib().hobo_local_field_bits(self._h, xp, B, row0, _dev_ptr(G, torch.float32, (B, self.N)),
                                           _dev_ptr(E, torch.float32, (B,)), C.byref(best) if want_best else None,
                                           _stream_handle(stream)))
        return (G, E, (best.e, best.idx)) if want_best else (G, E)

    def local_field_host_bits(self, Xb, E=None, row0=0, want_best=True, stream=None, fields=True, G=None):
        """hobo_local_field_host_bits (fields=True) / hobo_energy_host_bits: packed rows in host
        memory (numpy uint32 or a CPU int32 tensor, B x ceil(N/32), ideally pinned); G as in
        local_field_host."""
        W = (self.N + 31) // 32
        B = Xb.shape[0]
        if hasattr(Xb, "data_ptr"):
            if Xb.is_cuda or tuple(Xb.shape) != (B, W) or not Xb.is_contiguous() or Xb.element_size() != 4:
                raise ValueError(f"expected a contiguous 4-byte CPU tensor of shape {(B, W)}")
            xp = Xb.data_ptr()
        else:
            if Xb.dtype.itemsize != 4 or Xb.shape != (B, W) or not Xb.flags.c_contiguous:
                raise ValueError(f"expected a C-contiguous 4-byte array of shape {(B, W)}")
            xp = Xb.ctypes.data
        if E is None:
            E = np.empty(B, np.float32)
        ep = self._host_ptr(E, np.float32, (B,))
        best = HoboBest()
        bp = C.byref(best) if want_best else None
        if fields:
            _check(lib().hobo_local_field_host_bits(self._h, xp, B, row0, self._host_ptr(G, np.float32, (B, self.N)), ep,
                                                    bp, _stream_handle(stream)))
        else:
            if G is not None:
                raise ValueError("fields=False computes no fields")
            _check(lib().hobo_energy_host_bits(self._h, xp, B, row0, ep, bp, _stream_handle(stream)))
        return E, ((best.e, best.idx) if want_best else None)

    def multilinear_field(self, P, G=None, E=None, stream=None):
        """Gradient and value of the multilinear relaxation at real p (CUDA bf16 tensor B x N)."""
        import torch
        B = P.shape[0]
        pp = _dev_ptr(P, torch.bfloat16, (B, self.N))
        if G is None:
            G = torch.empty(B, self.N, dtype=torch.float32, device=P.device)
        if E is None:
            E = torch.empty(B, dtype=torch.float32, device=P.device)
        _check(lib().hobo_multilinear_field(self._h, pp, B, _dev_ptr(G, torch.float32, (B, self.N)),
                                            _dev_ptr(E, torch.float32, (B,)), _stream_handle(stream)))
        return G, E

    def search(self, seed, batch, iters, chain0=None, nchains=None, p0=0.5, p1=0.005, stream=None):
        """hobo_search (or the shard [chain0, chain0+nchains)).  Returns (x_best u8[N], e_best, chain)."""
        x = np.zeros(self.N, np.uint8)
        e = C.c_float()
        c = C.c_int64()
        if chain0 is None:
            chain0, nchains = 0, batch
        _check(lib().hobo_search_shard(self._h, seed, chain0, nchains, iters, p0, p1, _np_ptr(x), C.byref(e),
                                       C.byref(c), _stream_handle(stream)))
        return x, e.value, c.value

    def search_global(self, seed, batch, iters, stream=None):
        """hobo_search: the global batch of chains; with a library communicator (dist_init) the
        chains are sharded by rank and the winner combined over ranks.  Returns (x u8[N], e)."""
        x = np.zeros(self.N, np.uint8)
        e = C.c_float()
        _check(lib().hobo_search(self._h, seed, batch, iters, _np_ptr(x), C.byref(e), _stream_handle(stream)))
        return x, e.value

    def search_samples(self, seed, batch, iters, topk=10, stream=None):
        """hobo_search_samples: list of (x u8[N], energy, occurrence), the paper's result format."""
        x = np.zeros((topk, self.N), np.uint8)
        e = np.zeros(topk, np.float32)
        cnt = np.zeros(topk, np.int64)
        n = C.c_int64()
        _check(lib().hobo_search_samples(self._h, seed, batch, iters, topk, _np_ptr(x), _np_ptr(e), _np_ptr(cnt),
                                         C.byref(n), _stream_handle(stream)))
        return [(x[i], float(e[i]), int(cnt[i])) for i in range(n.value)]

    def gd_run(self, seed, shots, steps, step_size, greedy_iters=None, topk=10, stream=None):
        """hobo_gd_run: gradient descent on the relaxation + rounding + greedy descent, aggregated."""
        if greedy_iters is None:
            greedy_iters = self.N
        x = np.zeros((topk, self.N), np.uint8)
        e = np.zeros(topk, np.float32)
        cnt = np.zeros(topk, np.int64)
        n = C.c_int64()
        _check(lib().hobo_gd_run(self._h, seed, shots, steps, step_size, greedy_iters, topk, _np_ptr(x), _np_ptr(e),
                                 _np_ptr(cnt), C.byref(n), _stream_handle(stream)))
        return [(x[i], float(e[i]), int(cnt[i])) for i in range(n.value)]

    def default_t_start(self):
        """SPEC's default schedule start: 10 * max |coefficient| (t_end defaults to 0.01)."""
        if getattr(self, "_tmax", None) is None:
            _, v = self.cells()
            self._tmax = 10.0 * float(np.abs(v).max()) if len(v) else 1.0
        return self._tmax

    def sa_shard(self, seed, chain0, nchains, sweeps, t_start=None, t_end=0.01, device=None, stream=None):
        """hobo_sa_shard: annealed final states (u8, nchains x N), fresh energies (f32) and the
        incrementally tracked energies (f64), as CUDA tensors."""
        import torch
        t0 = self.default_t_start() if t_start is None else float(t_start)
        dev = torch.device("cuda") if device is None else torch.device(device)
        X = torch.empty(nchains, self.N, dtype=torch.uint8, device=dev)
        E = torch.empty(nchains, dtype=torch.float32, device=dev)
        Et = torch.empty(nchains, dtype=torch.float64, device=dev)
        _check(lib().hobo_sa_shard(self._h, seed, chain0, nchains, sweeps, t0, float(t_end), X.data_ptr(),
                                   E.data_ptr(), Et.data_ptr(), _stream_handle(stream)))
        return X, E, Et

    def sa_run(self, seed, shots, sweeps, t_start=None, t_end=0.01, topk=10, stream=None):
        """hobo_sa_run: SPEC sa_run's SampleSet — list of (x u8[N], energy, occurrence)."""
        t0 = self.default_t_start() if t_start is None else float(t_start)
        x = np.zeros((topk, self.N), np.uint8)
        e = np.zeros(topk, np.float32)
        cnt = np.zeros(topk, np.int64)
        n = C.c_int64()
        _check(lib().hobo_sa_run(self._h, seed, shots, sweeps, t0, float(t_end), topk, _np_ptr(x), _np_ptr(e),
                                 _np_ptr(cnt), C.byref(n), _stream_handle(stream)))
        return [(x[i], float(e[i]), int(cnt[i])) for i in range(n.value)]

    def tt_build(self, rel_tol=0.0):
        """Tensor-Train cores by sequential SVD; returns the bond ranks r_0..r_k."""
        ranks = np.zeros(self.order + 1, np.int32)
        _check(lib().hobo_tt_build(self._h, rel_tol, _np_ptr(ranks)))
        return ranks.tolist()

    def tt_energy(self, X, E=None, row0=0, want_best=True, stream=None):
        """Energies from the TT form (after tt_build)."""
        import torch
        B = X.shape[0]
        xp = _dev_ptr(X, torch.uint8, (B, self.N))
        if E is None:
            E = torch.empty(B, dtype=torch.float32, device=X.device)
        best = HoboBest()
        _check(lib().hobo_tt_energy(self._h, xp, B, row0, _dev_ptr(E, torch.float32, (B,)),
                                    C.byref(best) if want_best else None, _stream_handle(stream)))
        return E, ((best.e, best.idx) if want_best else None)

    def set_profiling(self, enable=True):
        _check(lib().hobo_set_profiling(self._h, 1 if enable else 0))

    def launch_stats(self):
        """Launches, executed MMA MACs, algorithmic MACs, (profiling on) kernel ms of the last call, and
        its MMA kind: i8_planes = int8 digit planes (kind::i8, MACs are 8-bit), minus the e4m3 limb
        planes (kind::f8f6f4, MACs are 8-bit), or 0 (bf16 limbs)."""
        n, mm, am, ms, i8 = C.c_int64(), C.c_double(), C.c_double(), C.c_double(), C.c_int()
        _check(lib().hobo_last_launch_stats(self._h, C.byref(n), C.byref(mm), C.byref(am), C.byref(ms)))
        _check(lib().hobo_last_launch_kind(self._h, C.byref(i8)))
        return dict(launches=n.value, mma_macs=mm.value, algo_macs=am.value, kernel_ms=ms.value, i8_planes=i8.value)


# ---- multi-GPU communicator of the library (include/hobo.h) ------------------
def dist_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().hobo_dist_unique_id(buf))
    return buf.raw


def dist_init(rank: int, world: int, uid: bytes, device: int):
    buf = C.create_string_buffer(bytes(uid), 128)
    _check(lib().hobo_dist_init(rank, world, buf, device))


def dist_finalize():
    _check(lib().hobo_dist_finalize())


def dist_info():
    r, w = C.c_int(), C.c_int()
    _check(lib().hobo_dist_info(C.byref(r), C.byref(w)))
    return r.value, w.value


# ---- multi-GPU host logic of the library (hobo_shard*, hobo_best_key; no device needed) -------
def shard(total: int, rank: int, world: int):
    """hobo_shard: this rank's contiguous range [lo, hi) of `total` items."""
    lo, n = C.c_int64(), C.c_int64()
    _check(lib().hobo_shard(total, rank, world, C.byref(lo), C.byref(n)))
    return lo.value, lo.value + n.value


def shard_owner(total: int, world: int, index: int) -> int:
    """hobo_shard_owner: the rank whose shard holds global item `index`."""
    o = C.c_int()
    _check(lib().hobo_shard_owner(total, world, index, C.byref(o)))
    return o.value


def best_key(e: float, idx: int) -> int:
    """hobo_best_key: the unsigned 64-bit argmin key of (e, idx) (HoboError on NaN)."""
    k = C.c_uint64()
    _check(lib().hobo_best_key(e, idx, C.byref(k)))
    return k.value


def best_from_key(key: int):
    """hobo_best_from_key: (e, idx); the empty key ~0 gives (inf, -1)."""
    b = HoboBest()
    _check(lib().hobo_best_from_key(key, C.byref(b)))
    return b.e, b.idx
