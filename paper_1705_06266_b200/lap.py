"""ctypes binding of liblap.so (include/lap.h): argument marshalling only.

Every step of setup and solve runs in the CUDA kernels of liblap.so; there is
no CPU fallback.  If the library is missing or fails to load, importing this
module raises.  Vectors may be numpy arrays (host) or CUDA torch tensors
(device pointers are passed straight through).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblap.so")

LAP_OK, LAP_EINVAL, LAP_EGRAPH, LAP_EDISCONNECTED, LAP_ENOMEM, LAP_ECUDA, LAP_ENCCL, LAP_ENOCONV, LAP_ESTALL = range(9)
KIND_AGG, KIND_ELIM, KIND_COARSEST = 0, 1, 2


class LapError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"liblap status {code}: {msg}")
        self.code = code


class lap_graph(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("row_ptr", ctypes.c_void_p), ("col", ctypes.c_void_p),
                ("w", ctypes.c_void_p), ("on_device", ctypes.c_int32)]


class lap_params(ctypes.Structure):
    _fields_ = [
        ("tol", ctypes.c_double), ("max_iters", ctypes.c_int32), ("cheby_degree", ctypes.c_int32),
        ("cheby_lo", ctypes.c_double), ("cheby_hi", ctypes.c_double), ("lanczos_steps", ctypes.c_int32),
        ("elim_max_degree", ctypes.c_int32), ("elim_enable", ctypes.c_int32), ("n_test_vectors", ctypes.c_int32),
        ("tv_sweeps", ctypes.c_int32), ("tv_omega", ctypes.c_double), ("vote_rounds", ctypes.c_int32),
        ("vote_threshold", ctypes.c_int32), ("coarse_nnz", ctypes.c_int64), ("max_levels", ctypes.c_int32),
        ("seed", ctypes.c_uint64), ("random_order", ctypes.c_int32), ("affinity_power", ctypes.c_int32),
        ("keep_strength", ctypes.c_int32), ("use_graphs", ctypes.c_int32), ("replicate_nnz", ctypes.c_int64),
        ("cycle", ctypes.c_int32), ("kcycle_inner", ctypes.c_int32), ("elim_rounds", ctypes.c_int32),
        ("keep_logical", ctypes.c_int32),
    ]


class lap_stats(ctypes.Structure):
    _fields_ = [("kernel_launches", ctypes.c_int64), ("spmv_edges", ctypes.c_int64), ("spmv_bytes", ctypes.c_int64),
                ("setup_ms", ctypes.c_double), ("solve_ms", ctypes.c_double), ("vcycles", ctypes.c_int32)]


EXPORTS = [
    "lap_params_default", "lap_last_error", "lap_version", "lap_setup", "lap_solve", "lap_free",
    "lap_num_levels", "lap_level_info", "lap_level_export", "lap_level_strength", "lap_coarse_pinv",
    "lap_perm", "lap_spmv", "lap_vcycle", "lap_kcycle", "lap_solve_block", "lap_get_stats", "lap_bench_op",
    "lap_nccl_unique_id", "lap_comm_create", "lap_comm_create_virtual", "lap_comm_info", "lap_comm_free",
    "lap_setup_dist", "lap_dist_index", "lap_pool_retain", "lap_random_stream",
    "lap_bench_gather", "lap_level_rows", "lap_import_hierarchy", "lap_setup_split",
]


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"liblap.so not built at {path}; run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    P, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    pi32, pi64, pdbl = ctypes.POINTER(i32), ctypes.POINTER(i64), ctypes.POINTER(dbl)
    sig = {
        "lap_params_default": (None, [ctypes.POINTER(lap_params)]),
        "lap_last_error": (ctypes.c_char_p, []),
        "lap_version": (ctypes.c_char_p, []),
        "lap_setup": (ctypes.c_int, [ctypes.POINTER(lap_graph), ctypes.POINTER(lap_params), P, ctypes.POINTER(P)]),
        "lap_solve": (ctypes.c_int, [P, P, P, dbl, pi32, pdbl, P]),
        "lap_free": (None, [P]),
        "lap_num_levels": (ctypes.c_int, [P, pi32]),
        "lap_level_info": (ctypes.c_int, [P, i32, pi32, pi64, pi64, pdbl]),
        "lap_level_export": (ctypes.c_int, [P, i32, P, P, P, P, P]),
        "lap_level_strength": (ctypes.c_int, [P, i32, P]),
        "lap_coarse_pinv": (ctypes.c_int, [P, P]),
        "lap_perm": (ctypes.c_int, [P, P]),
        "lap_spmv": (ctypes.c_int, [P, i32, P, P, P]),
        "lap_vcycle": (ctypes.c_int, [P, P, P, P]),
        "lap_kcycle": (ctypes.c_int, [P, i32, i32, P, P, P]),
        "lap_solve_block": (ctypes.c_int, [P, i32, P, P, ctypes.c_double, P, P, P]),
        "lap_get_stats": (ctypes.c_int, [P, ctypes.POINTER(lap_stats)]),
        "lap_bench_op": (ctypes.c_int, [P, i32, i32, i32, P, P, pdbl, pi64]),
        "lap_nccl_unique_id": (ctypes.c_int, [P]),
        "lap_comm_create": (ctypes.c_int, [P, i32, i32, i32, i32, ctypes.POINTER(P)]),
        "lap_comm_create_virtual": (ctypes.c_int, [i32, i32, ctypes.POINTER(P)]),
        "lap_comm_info": (ctypes.c_int, [P, pi32, pi32, pi32, pi32, pi32]),
        "lap_comm_free": (None, [P]),
        "lap_setup_dist": (ctypes.c_int, [ctypes.POINTER(lap_graph), ctypes.POINTER(lap_params), P, P, ctypes.POINTER(P)]),
        "lap_dist_index": (ctypes.c_int, [i64, i32, i64, P, P, pi64]),
        "lap_setup_split": (ctypes.c_int, [i64, P, i32, P]),
        "lap_pool_retain": (None, [ctypes.c_uint64]),
        "lap_random_stream": (ctypes.c_int, [i32, ctypes.c_uint64, i32, i32, i64, P, P]),
        "lap_bench_gather": (ctypes.c_int, [i64, i64, i32, P, P]),
        "lap_level_rows": (ctypes.c_int, [P, i32, i64, P, P, P, P]),
        "lap_import_hierarchy": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(lap_params), P, ctypes.POINTER(P)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = load()
    return _lib


def _check(rc, allow=()):
    if rc != LAP_OK and rc not in allow:
        raise LapError(rc, lib().lap_last_error().decode())
    return rc


def _ptr(a):
    """Device pointer of a CUDA tensor or host pointer of a numpy array."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return ctypes.c_void_p(a.data_ptr())
    return ctypes.c_void_p(a.ctypes.data)


_TORCH_DT = {np.float64: "torch.float64", np.int64: "torch.int64", np.int32: "torch.int32"}


def _arg(a, n: int, dt, name: str, out: bool = False):
    """Validate one array argument before its pointer crosses the ABI: the C
    side reads / writes exactly n elements of dtype dt, contiguously.  numpy
    inputs are converted (a copy if needed); numpy outputs and torch tensors
    must already match -- a mismatch raises ValueError instead of letting the
    library over-read host memory or fault on the device."""
    if hasattr(a, "data_ptr"):  # torch tensor (CUDA or CPU)
        if str(a.dtype) != _TORCH_DT[dt]:
            raise ValueError(f"{name}: dtype {a.dtype}, expected {_TORCH_DT[dt]}")
        if not a.is_contiguous():
            raise ValueError(f"{name}: tensor is not contiguous")
        if a.numel() != n:
            raise ValueError(f"{name}: {a.numel()} elements, expected {n}")
        return a
    if out:
        if not (isinstance(a, np.ndarray) and a.dtype == dt and a.flags.c_contiguous and a.flags.writeable):
            raise ValueError(f"{name}: output must be a writeable C-contiguous {np.dtype(dt).name} array")
        if a.size != n:
            raise ValueError(f"{name}: {a.size} elements, expected {n}")
        return a
    a = np.ascontiguousarray(a, dt)
    if a.size != n:
        raise ValueError(f"{name}: {a.size} elements, expected {n}")
    return a


def _stream(stream):
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


def random_stream(which: int, n: int, seed: int = 0, level: int = 0, attempt: int = 0, stream=None) -> np.ndarray:
    """lap_random_stream (test hook): 0 = h(i) (uint64), 1 = X0 rows (n x 4),
    2 = Lanczos start vector (unnormalised), 3 = mix64(i) (uint64)."""
    out = np.zeros(4 * n if which == 1 else n, np.uint64 if which in (0, 3) else np.float64)
    _check(lib().lap_random_stream(which, seed, level, attempt, n, _ptr(out), _stream(stream)))
    return out.reshape(n, 4) if which == 1 else out


def bench_gather(nx: int, m: int = 1 << 26, reps: int = 5, stream=None) -> np.ndarray:
    """lap_bench_gather: ms per launch of m random gathers from an nx-double x."""
    ms = np.zeros(reps)
    _check(lib().lap_bench_gather(int(nx), int(m), int(reps), _stream(stream), _ptr(ms)))
    return ms


def pool_retain(nbytes: int) -> None:
    """lap_pool_retain: bytes of pool reservation kept when no hierarchy is alive."""
    lib().lap_pool_retain(int(nbytes))


def lap_params_default(**kw) -> lap_params:
    p = lap_params()
    lib().lap_params_default(ctypes.byref(p))
    for k, v in kw.items():
        if not hasattr(p, k):
            raise AttributeError(k)
        setattr(p, k, v)
    return p


class Comm:
    """A pr x pc process grid for the sharded solve (lap_comm_create /
    lap_comm_create_virtual).  With nccl_id=None the whole grid is emulated in
    this process on the current GPU."""

    def __init__(self, grid_rows: int, grid_cols: int, nccl_id: bytes | None = None, rank: int = 0):
        self._c = ctypes.c_void_p()
        if nccl_id is None:
            _check(lib().lap_comm_create_virtual(grid_rows, grid_cols, ctypes.byref(self._c)))
        else:
            buf = (ctypes.c_uint8 * 128).from_buffer_copy(bytes(nccl_id).ljust(128, b"\0"))
            _check(lib().lap_comm_create(buf, rank, grid_rows * grid_cols, grid_rows, grid_cols,
                                         ctypes.byref(self._c)))
        self.grid = (grid_rows, grid_cols)

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        _check(lib().lap_nccl_unique_id(buf))
        return bytes(buf)

    def info(self):
        v = [ctypes.c_int32() for _ in range(5)]
        _check(lib().lap_comm_info(self._c, *[ctypes.byref(x) for x in v]))
        return dict(zip(["rank", "nranks", "grid_rows", "grid_cols", "virtual"], [x.value for x in v]))

    def close(self):
        if getattr(self, "_c", None):
            lib().lap_comm_free(self._c)
            self._c = None


def dist_index(n: int, nranks: int, rows) -> tuple:
    """Host-only piece map of a sharded level (lap_dist_index)."""
    rows = np.ascontiguousarray(rows, np.int64)
    out = np.zeros(len(rows), np.int64)
    S = ctypes.c_int64()
    _check(lib().lap_dist_index(n, nranks, len(rows), _ptr(rows), _ptr(out), ctypes.byref(S)))
    return out, S.value


def setup_split(cum, nranks: int) -> np.ndarray:
    """Host-only split rule of the distributed setup's term builds
    (lap_setup_split): cum[0..nout] term prefix -> bounds[0..nranks]."""
    cum = np.ascontiguousarray(cum, np.int64)
    out = np.zeros(nranks + 1, np.int64)
    _check(lib().lap_setup_split(len(cum) - 1, _ptr(cum), nranks, _ptr(out)))
    return out


class Hierarchy:
    """lap_setup(graph, params) -> hierarchy ; .solve(b) -> (x, iters, residual).
    With comm=Comm(...), lap_setup_dist: the fine levels are sharded over the grid."""

    def __init__(self, graph, params: lap_params | None = None, stream=None, comm: "Comm | None" = None, **kw):
        self.params = params if params is not None else lap_params_default(**kw)
        dev = hasattr(graph.row_ptr, "data_ptr") and getattr(graph.row_ptr, "is_cuda", False)
        n = int(graph.n)
        if n < 1:
            raise ValueError("graph.n must be >= 1")
        rp = _arg(graph.row_ptr, n + 1, np.int64, "row_ptr")
        nnz = int(rp[-1])  # one device read for a CUDA tensor
        if dev and not (getattr(graph.col, "is_cuda", False) and (graph.w is None or getattr(graph.w, "is_cuda", False))):
            raise ValueError("row_ptr, col and w must all be CUDA tensors or all host arrays")
        col = _arg(graph.col, nnz, np.int32, "col")
        w = None if graph.w is None else _arg(graph.w, nnz, np.float64, "w")
        self._keep = (rp, col, w)
        g = lap_graph(int(graph.n), _ptr(self._keep[0]), _ptr(self._keep[1]), _ptr(self._keep[2]), 1 if dev else 0)
        self._h = ctypes.c_void_p()
        self.comm = comm
        if comm is None:
            rc = lib().lap_setup(ctypes.byref(g), ctypes.byref(self.params), _stream(stream), ctypes.byref(self._h))
        else:
            rc = lib().lap_setup_dist(ctypes.byref(g), ctypes.byref(self.params), comm._c, _stream(stream),
                                      ctypes.byref(self._h))
        self.status = _check(rc, allow=(LAP_ESTALL,))
        self._keep = None
        self.n = n

    @classmethod
    def import_dir(cls, path: str, params: lap_params | None = None, stream=None, **kw) -> "Hierarchy":
        """lap_import_hierarchy: a hierarchy from the interchange directory."""
        self = cls.__new__(cls)
        self.params = params if params is not None else lap_params_default(**kw)
        self._h = ctypes.c_void_p()
        self.comm = None
        self._keep = None
        rc = lib().lap_import_hierarchy(os.fsencode(path), ctypes.byref(self.params), _stream(stream),
                                        ctypes.byref(self._h))
        self.status = _check(rc, allow=(LAP_ESTALL,))
        self.n = self.level_info(0)[1]
        return self

    def close(self):
        if getattr(self, "_h", None):
            lib().lap_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- the two calls of the method
    def solve(self, b, x=None, tol: float = 0.0, stream=None):
        if x is None:
            x = np.zeros(self.n) if not hasattr(b, "data_ptr") else b.new_zeros(self.n)
        b = _arg(b, self.n, np.float64, "b")
        x = _arg(x, self.n, np.float64, "x", out=True)
        it = ctypes.c_int32(0)
        rr = ctypes.c_double(0.0)
        rc = _check(lib().lap_solve(self._h, _ptr(b), _ptr(x), tol, ctypes.byref(it), ctypes.byref(rr),
                                    _stream(stream)), allow=(LAP_ENOCONV,))
        return x, int(it.value), float(rr.value), rc

    def solve_block(self, B, X=None, tol: float = 0.0, stream=None):
        """k right-hand sides at once (N4): B is (k, n) -- row j = right-hand
        side j, i.e. n x k column-major -- numpy or a torch CUDA tensor.
        Returns X (k, n), iters[k], rel_residual[k], status."""
        if not hasattr(B, "data_ptr"):
            B = np.ascontiguousarray(B, np.float64)
        if B.ndim != 2 or B.shape[1] != self.n:
            raise ValueError(f"B: shape {tuple(B.shape)}, expected (k, {self.n})")
        k = B.shape[0]
        if X is None:
            X = np.zeros((k, self.n)) if not hasattr(B, "data_ptr") else B.new_zeros((k, self.n))
        B = _arg(B, k * self.n, np.float64, "B")
        X = _arg(X, k * self.n, np.float64, "X", out=True)
        it = np.zeros(k, np.int32)
        rr = np.zeros(k, np.float64)
        rc = _check(lib().lap_solve_block(self._h, k, _ptr(B), _ptr(X), tol, _ptr(it), _ptr(rr), _stream(stream)),
                    allow=(LAP_ENOCONV,))
        return X, it, rr, rc

    # ---- introspection
    @property
    def nlev(self) -> int:
        v = ctypes.c_int32(0)
        _check(lib().lap_num_levels(self._h, ctypes.byref(v)))
        return v.value

    def level_info(self, l: int):
        k, n, z, lam = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
        _check(lib().lap_level_info(self._h, l, ctypes.byref(k), ctypes.byref(n), ctypes.byref(z), ctypes.byref(lam)))
        return k.value, n.value, z.value, lam.value

    def level(self, l: int) -> dict:
        kind, n, z, lam = self.level_info(l)
        rp = np.zeros(n + 1, np.int64)
        col = np.zeros(max(z, 1), np.int32)
        w = np.zeros(max(z, 1), np.float64)
        d = np.zeros(max(n, 1), np.float64)
        mp = np.zeros(max(n, 1), np.int32)
        _check(lib().lap_level_export(self._h, l, _ptr(rp), _ptr(col), _ptr(w), _ptr(d), _ptr(mp)))
        out = dict(kind=kind, n=n, nnz=z, lam=lam, row_ptr=rp, col=col[:z], w=w[:z], d=d[:n])
        if kind == KIND_AGG:
            out["agg"] = mp[:n]
            out["m"] = int(mp[:n].max()) + 1 if n else 0
        elif kind == KIND_ELIM:
            out["fmap"] = mp[:n]
            out["nF"] = int((mp[:n] < 0).sum())
        else:
            P = np.zeros(n * n)
            _check(lib().lap_coarse_pinv(self._h, _ptr(P)))
            out["pinv"] = P.reshape(n, n)
        return out

    def level_maps(self, l: int):
        """(d, map) of level l (map = agg or fmap; None for the coarsest) --
        available also when the logical CSR was released."""
        kind, n, z, lam = self.level_info(l)
        d = np.zeros(max(n, 1), np.float64)
        mp = np.zeros(max(n, 1), np.int32)
        _check(lib().lap_level_export(self._h, l, None, None, None, _ptr(d), _ptr(mp)))
        return d[:n], (mp[:n] if kind != KIND_COARSEST else None)

    def level_map(self, l: int) -> np.ndarray:
        """agg (aggregation level) or fmap (elimination level) of level l in the
        logical numbering; available also when the logical CSR was released."""
        _, n, _, _ = self.level_info(l)
        mp = np.zeros(max(n, 1), np.int32)
        _check(lib().lap_level_export(self._h, l, None, None, None, None, _ptr(mp)))
        return mp[:n]

    def level_degrees(self, l: int, rows) -> np.ndarray:
        """Stored entries of the given logical rows of level l (lap_level_rows
        without the column / weight copies)."""
        rows = np.ascontiguousarray(rows, np.int64)
        rp = np.zeros(len(rows) + 1, np.int64)
        _check(lib().lap_level_rows(self._h, l, len(rows), _ptr(rows), _ptr(rp), None, None))
        return np.diff(rp)

    def level_rows(self, l: int, rows):
        """Rows of level l's logical CSR rebuilt from the solve storage
        (lap_level_rows): returns (row_ptr[k+1], col, w)."""
        rows = np.ascontiguousarray(rows, np.int64)
        rp = np.zeros(len(rows) + 1, np.int64)
        _check(lib().lap_level_rows(self._h, l, len(rows), _ptr(rows), _ptr(rp), None, None))
        col = np.zeros(max(1, int(rp[-1])), np.int32)
        w = np.zeros(max(1, int(rp[-1])), np.float64)
        _check(lib().lap_level_rows(self._h, l, len(rows), _ptr(rows), _ptr(rp), _ptr(col), _ptr(w)))
        return rp, col[:rp[-1]], w[:rp[-1]]

    def strength(self, l: int) -> np.ndarray:
        _, n, z, _ = self.level_info(l)
        S = np.zeros(max(z, 1))
        _check(lib().lap_level_strength(self._h, l, _ptr(S)))
        return S[:z]

    def perm(self) -> np.ndarray:
        p = np.zeros(self.n, np.int64)
        _check(lib().lap_perm(self._h, _ptr(p)))
        return p

    def spmv(self, l: int, x, y=None, stream=None):
        n = self.level_info(l)[1]
        if y is None:
            y = np.zeros(n) if not hasattr(x, "data_ptr") else x.new_zeros(n)
        x = _arg(x, n, np.float64, "x")
        y = _arg(y, n, np.float64, "y", out=True)
        _check(lib().lap_spmv(self._h, l, _ptr(x), _ptr(y), _stream(stream)))
        return y

    def vcycle(self, r, z=None, stream=None):
        if z is None:
            z = np.zeros(self.n) if not hasattr(r, "data_ptr") else r.new_zeros(self.n)
        r = _arg(r, self.n, np.float64, "r")
        z = _arg(z, self.n, np.float64, "z", out=True)
        _check(lib().lap_vcycle(self._h, _ptr(r), _ptr(z), _stream(stream)))
        return z

    def kcycle(self, l: int, r, with_fcg: bool = False, z=None, stream=None):
        """z = K(l, r) on level l's internal numbering (N2); with_fcg: the
        level's inner FCG iterations around it (oracle.Hierarchy.kcoarse)."""
        n = self.level_info(l)[1]
        if z is None:
            z = np.zeros(n) if not hasattr(r, "data_ptr") else r.new_zeros(n)
        r = _arg(r, n, np.float64, "r")
        z = _arg(z, n, np.float64, "z", out=True)
        _check(lib().lap_kcycle(self._h, l, 1 if with_fcg else 0, _ptr(r), _ptr(z), _stream(stream)))
        return z

    def stats(self) -> dict:
        s = lap_stats()
        _check(lib().lap_get_stats(self._h, ctypes.byref(s)))
        return {k: getattr(s, k) for k, _ in s._fields_}

    def bench_op(self, which: int, level: int = 0, reps: int = 50, stream=None):
        """CUDA-event time of `reps` launches of an operation (lap_bench_op):
        which 0 = SpMV on `level`, 1 = fused Chebyshev step, 2 = V-cycle.
        Returns (ms per launch array, algorithmic bytes, edges) per launch."""
        ms = np.zeros(reps)
        by, ed = ctypes.c_double(), ctypes.c_int64()
        _check(lib().lap_bench_op(self._h, which, level, reps, _stream(stream), _ptr(ms), ctypes.byref(by),
                                  ctypes.byref(ed)))
        return ms, by.value, ed.value

    def first_agg_level(self) -> int:
        for l in range(self.nlev):
            if self.level_info(l)[0] == KIND_AGG:
                return l
        return -1
