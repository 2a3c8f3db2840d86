"""oracle -- ctypes wrapper over the plain-C CPU oracle (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg
(``cpu_baseline`` / ``--impl reference``) may import this package.  The
product library (paper_1705_06266_b200, liblap.so) never imports, links or
calls it.  See oracle/lap_oracle.h for the citations and what each function
computes.
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lap_oracle.c")
_HDR = os.path.join(_HERE, "lap_oracle.h")
_SO = os.path.join(_HERE, "liboracle.so")

ORC_OK, ORC_EINVAL, ORC_EGRAPH, ORC_EDISCONNECTED, ORC_ENOMEM, ORC_ENOCONV, ORC_ESTALL = 0, 1, 2, 3, 4, 7, 8
AGG, ELIM, COARSEST = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle (IEEE fp64, no FMA contraction, no fast-math)."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-std=gnu11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


class Params(ctypes.Structure):
    _fields_ = [
        ("tol", ctypes.c_double), ("max_iters", ctypes.c_int32), ("cheby_degree", ctypes.c_int32),
        ("cheby_lo", ctypes.c_double), ("cheby_hi", ctypes.c_double), ("lanczos_steps", ctypes.c_int32),
        ("elim_max_degree", ctypes.c_int32), ("elim_enable", ctypes.c_int32),
        ("n_test_vectors", ctypes.c_int32), ("tv_sweeps", ctypes.c_int32), ("tv_omega", ctypes.c_double),
        ("vote_rounds", ctypes.c_int32), ("vote_threshold", ctypes.c_int32), ("coarse_nnz", ctypes.c_int64),
        ("max_levels", ctypes.c_int32), ("seed", ctypes.c_uint64), ("random_order", ctypes.c_int32),
        ("affinity_power", ctypes.c_int32), ("cycle", ctypes.c_int32), ("kcycle_inner", ctypes.c_int32),
        ("elim_rounds", ctypes.c_int32),
    ]


class Level(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32), ("n", ctypes.c_int64), ("nnz", ctypes.c_int64),
        ("row_ptr", ctypes.POINTER(ctypes.c_int64)), ("col", ctypes.POINTER(ctypes.c_int32)),
        ("w", ctypes.POINTER(ctypes.c_double)), ("d", ctypes.POINTER(ctypes.c_double)),
        ("lam", ctypes.c_double), ("m", ctypes.c_int64), ("agg", ctypes.POINTER(ctypes.c_int32)),
        ("S", ctypes.POINTER(ctypes.c_double)), ("nF", ctypes.c_int64),
        ("fmap", ctypes.POINTER(ctypes.c_int32)), ("pinv", ctypes.POINTER(ctypes.c_double)),
    ]


_lib = None
P = ctypes.c_void_p


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        i64, i32, u64, dbl = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double
        sig = {
            "orc_params_default": (None, [P]),
            "orc_set_threads": (None, [i32]),
            "orc_get_threads": (i32, []),
            "orc_mix64": (u64, [u64]),
            "orc_salt": (u64, [u64, u64]),
            "orc_mix64_inverse": (u64, [u64]),
            "orc_canon_elo": (i32, [i32, i64]),
            "orc_canon_sum": (dbl, [P, i64, i32, i64]),
            "orc_ilogb": (i32, [dbl]),
            "orc_validate": (ctypes.c_int, [i64, P, P, P]),
            "orc_random_perm": (None, [i64, u64, P]),
            "orc_row_sums": (None, [i64, P, P, P]),
            "orc_relabel": (None, [i64, P, P, P, P, P, P, P]),
            "orc_spmv": (None, [i64, P, P, P, P, P, P]),
            "orc_elim_select": (i64, [i64, P, P, i32, u64, P, P]),
            "orc_schur": (i64, [i64, P, P, P, P, P, P, P, P, P, P]),
            "orc_test_vectors": (None, [i64, P, P, P, P, u64, i32, i32, i32, dbl, P]),
            "orc_test_vectors_from": (None, [i64, P, P, P, P, i32, dbl, P]),
            "orc_affinity": (None, [i64, P, P, P, i32, P]),
            "orc_normalize_strength": (None, [i64, P, P, P, P]),
            "orc_aggregate": (i64, [i64, P, P, P, i32, i32, P, P, P]),
            "orc_galerkin_count": (i64, [i64, P, P, P, i64]),
            "orc_galerkin": (i64, [i64, P, P, P, P, i64, P, P, P, P]),
            "orc_lanczos": (dbl, [i64, P, P, P, P, u64, i32, i32, P, P, P]),
            "orc_tridiag_max_eig": (dbl, [i32, P, P]),
            "orc_lanczos_start": (None, [i64, u64, i32, P]),
            "orc_elim_hash": (u64, [u64, u64]),
            "orc_coarse_pinv": (ctypes.c_int, [i64, P, P, P, P, P]),
            "orc_chebyshev": (None, [i64, P, P, P, P, dbl, dbl, dbl, i32, P, P, i32]),
            "orc_setup": (ctypes.c_int, [i64, P, P, P, P, ctypes.POINTER(P)]),
            "orc_free": (None, [P]),
            "orc_vcycle": (None, [P, i32, P, P]),
            "orc_kcycle": (None, [P, i32, P, P]),
            "orc_kcoarse": (None, [P, i32, P, P]),
            "orc_solve": (ctypes.c_int, [P, P, P, dbl, P, P]),
            "orc_nlev": (i32, [P]),
            "orc_get_level": (ctypes.POINTER(Level), [P, i32]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def default_params(**kw) -> Params:
    p = Params()
    lib().orc_params_default(ctypes.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


# ---------------------------------------------------------------- primitives

def set_threads(t: int) -> None:
    """OpenMP threads of the oracle; results are bitwise independent of it."""
    lib().orc_set_threads(int(t))


def get_threads() -> int:
    return int(lib().orc_get_threads())


def mix64(z: int) -> int:
    return lib().orc_mix64(z & 0xFFFFFFFFFFFFFFFF)


def mix64_inverse(z: int) -> int:
    return lib().orc_mix64_inverse(z & 0xFFFFFFFFFFFFFFFF)


def salt(seed: int, k: int) -> int:
    return lib().orc_salt(seed, k)


def canon_sum(terms, e_max: int, K: int) -> float:
    t = _c(terms, np.float64)
    return lib().orc_canon_sum(_p(t), len(t), e_max, K)


def canon_elo(e_max: int, K: int) -> int:
    return lib().orc_canon_elo(e_max, K)


def ilogb(x: float) -> int:
    return lib().orc_ilogb(x)


def validate(g) -> int:
    w = _c(g.w, np.float64) if g.w is not None else None
    return lib().orc_validate(g.n, _p(_c(g.row_ptr, np.int64)), _p(_c(g.col, np.int32)), _p(w))


def random_perm(n: int, seed: int = 0) -> np.ndarray:
    perm = np.zeros(n, dtype=np.int64)
    lib().orc_random_perm(n, seed, _p(perm))
    return perm


def relabel(g, perm):
    """O-S1: Pi L Pi^T of graph g (w None = unit) -> (row_ptr, col, w)."""
    rp = np.zeros(g.n + 1, np.int64)
    col = np.zeros(max(1, g.nnz), np.int32)
    w = np.zeros(max(1, g.nnz), np.float64)
    ww = None if g.w is None else _c(g.w, np.float64)
    lib().orc_relabel(g.n, _p(_c(g.row_ptr, np.int64)), _p(_c(g.col, np.int32)), _p(ww), _p(_c(perm, np.int64)),
                      _p(rp), _p(col), _p(w))
    return rp, col[:g.nnz], w[:g.nnz]


def row_sums(n, row_ptr, w) -> np.ndarray:
    d = np.zeros(n, dtype=np.float64)
    lib().orc_row_sums(n, _p(_c(row_ptr, np.int64)), _p(_c(w, np.float64)), _p(d))
    return d


def spmv(n, row_ptr, col, w, d, x) -> np.ndarray:
    y = np.zeros(n, dtype=np.float64)
    lib().orc_spmv(n, _p(_c(row_ptr, np.int64)), _p(_c(col, np.int32)), _p(_c(w, np.float64)),
                   _p(_c(d, np.float64)), _p(_c(x, np.float64)), _p(y))
    return y


def elim_select(n, row_ptr, col, max_degree=4, seed=0, hash_override=None):
    F = np.zeros(n, dtype=np.uint8)
    ho = _c(hash_override, np.uint64) if hash_override is not None else None
    nF = lib().orc_elim_select(n, _p(_c(row_ptr, np.int64)), _p(_c(col, np.int32)), max_degree, seed, _p(ho), _p(F))
    return F.astype(bool), int(nF)


def schur(n, row_ptr, col, w, d, F):
    """Returns (fmap, nrow_ptr, ncol, nw, nd)."""
    rp, c, ww, dd = _c(row_ptr, np.int64), _c(col, np.int32), _c(w, np.float64), _c(d, np.float64)
    Fu = _c(F, np.uint8)
    fmap = np.zeros(n, dtype=np.int32)
    nc = int(n - Fu.sum())
    nrp = np.zeros(nc + 1, dtype=np.int64)
    nnz = lib().orc_schur(n, _p(rp), _p(c), _p(ww), _p(dd), _p(Fu), _p(fmap), _p(nrp), None, None, None)
    ncol = np.zeros(max(nnz, 1), dtype=np.int32)
    nw = np.zeros(max(nnz, 1), dtype=np.float64)
    nd = np.zeros(max(nc, 1), dtype=np.float64)
    lib().orc_schur(n, _p(rp), _p(c), _p(ww), _p(dd), _p(Fu), _p(fmap), _p(nrp), _p(ncol), _p(nw), _p(nd))
    return fmap, nrp, ncol[:nnz], nw[:nnz], nd[:nc]


def test_vectors(n, row_ptr, col, w, d, seed=0, level=0, attempt=0, sweeps=3, omega=2.0 / 3.0):
    X = np.zeros((n, 4), dtype=np.float64)
    lib().orc_test_vectors(n, _p(_c(row_ptr, np.int64)), _p(_c(col, np.int32)), _p(_c(w, np.float64)),
                           _p(_c(d, np.float64)), seed, level, attempt, sweeps, omega, _p(X))
    return X


def test_vectors_from(n, row_ptr, col, w, d, X0, sweeps=3, omega=2.0 / 3.0):
    X = np.array(X0, dtype=np.float64, order="C").reshape(n, 4).copy()
    lib().orc_test_vectors_from(n, _p(_c(row_ptr, np.int64)), _p(_c(col, np.int32)), _p(_c(w, np.float64)),
                                _p(_c(d, np.float64)), sweeps, omega, _p(X))
    return X


def affinity(n, row_ptr, col, X, power=1):
    C = np.zeros(int(row_ptr[-1]), dtype=np.float64)
    lib().orc_affinity(n, _p(_c(row_ptr, np.int64)), _p(_c(col, np.int32)), _p(_c(X, np.float64)), power, _p(C))
    return C


def normalize_strength(n, row_ptr, col, C):
    S = np.zeros(int(row_ptr[-1]), dtype=np.float64)
    lib().orc_normalize_strength(n, _p(_c(row_ptr, np.int64)), _p(_c(col, np.int32)), _p(_c(C, np.float64)), _p(S))
    return S


def aggregate(n, row_ptr, col, S, rounds=10, threshold=8):
    agg = np.zeros(n, dtype=np.int32)
    st = np.zeros(n, dtype=np.int8)
    votes = np.zeros(n, dtype=np.int32)
    m = lib().orc_aggregate(n, _p(_c(row_ptr, np.int64)), _p(_c(col, np.int32)), _p(_c(S, np.float64)),
                            rounds, threshold, _p(agg), _p(st), _p(votes))
    return agg, int(m), st, votes


def galerkin(n, row_ptr, col, w, agg, m):
    rp, c, ww, a = _c(row_ptr, np.int64), _c(col, np.int32), _c(w, np.float64), _c(agg, np.int32)
    cnnz = lib().orc_galerkin_count(n, _p(rp), _p(c), _p(a), m)
    crp = np.zeros(m + 1, dtype=np.int64)
    ccol = np.zeros(max(cnnz, 1), dtype=np.int32)
    cw = np.zeros(max(cnnz, 1), dtype=np.float64)
    cd = np.zeros(max(m, 1), dtype=np.float64)
    lib().orc_galerkin(n, _p(rp), _p(c), _p(ww), _p(a), m, _p(crp), _p(ccol), _p(cw), _p(cd))
    return crp, ccol[:cnnz], cw[:cnnz], cd[:m]


def lanczos(n, row_ptr, col, w, d, seed=0, level=0, steps=10):
    al = np.zeros(64)
    be = np.zeros(64)
    k = ctypes.c_int32(0)
    lam = lib().orc_lanczos(n, _p(_c(row_ptr, np.int64)), _p(_c(col, np.int32)), _p(_c(w, np.float64)),
                            _p(_c(d, np.float64)), seed, level, steps, _p(al), _p(be), ctypes.byref(k))
    return lam, al[:k.value], be[:k.value]


def lanczos_start(n, seed=0, level=0):
    """Unnormalised Lanczos start vector of level `level` (O-S6, reading R-U')."""
    v = np.zeros(n)
    lib().orc_lanczos_start(n, seed, level, _p(v))
    return v


def elim_hash(j: int, seed: int = 0) -> int:
    """h(j) = mix64(j XOR salt_2) (O-R17)."""
    return lib().orc_elim_hash(j, seed)


def tridiag_max_eig(alpha, beta):
    a = _c(alpha, np.float64)
    b = _c(np.concatenate([beta, [0.0]]), np.float64)
    return lib().orc_tridiag_max_eig(len(a), _p(a), _p(b))


def coarse_pinv(n, row_ptr, col, w, d):
    pinv = np.zeros((n, n), dtype=np.float64)
    rc = lib().orc_coarse_pinv(n, _p(_c(row_ptr, np.int64)), _p(_c(col, np.int32)), _p(_c(w, np.float64)),
                               _p(_c(d, np.float64)), _p(pinv))
    return rc, pinv


def chebyshev(n, row_ptr, col, w, d, lam, b, x=None, lo=0.3, hi=1.1, degree=2):
    xx = np.zeros(n) if x is None else np.array(x, dtype=np.float64, copy=True)
    lib().orc_chebyshev(n, _p(_c(row_ptr, np.int64)), _p(_c(col, np.int32)), _p(_c(w, np.float64)),
                        _p(_c(d, np.float64)), lam, lo, hi, degree, _p(_c(b, np.float64)), _p(xx),
                        1 if x is None else 0)
    return xx


# ---------------------------------------------------------------- hierarchy

@dataclass
class LevelData:
    kind: int
    n: int
    nnz: int
    row_ptr: np.ndarray
    col: np.ndarray
    w: np.ndarray
    d: np.ndarray
    lam: float = 0.0
    m: int = 0
    agg: np.ndarray | None = None
    S: np.ndarray | None = None
    nF: int = 0
    fmap: np.ndarray | None = None
    pinv: np.ndarray | None = None


def _arr(ptr, n, dt):
    if n <= 0 or not ptr:
        return np.zeros(0, dtype=dt)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dt, copy=True)


class Hierarchy:
    """Oracle hierarchy (O-S9) with the solve (O-S7, O-S8)."""

    def __init__(self, g, params: Params | None = None, **kw):
        self.params = params if params is not None else default_params(**kw)
        self._h = ctypes.c_void_p()
        w = None if g.w is None else _c(g.w, np.float64)
        self._keep = (_c(g.row_ptr, np.int64), _c(g.col, np.int32), w)
        self.status = lib().orc_setup(g.n, _p(self._keep[0]), _p(self._keep[1]), _p(self._keep[2]),
                                      ctypes.byref(self.params), ctypes.byref(self._h))
        if not self._h:
            raise RuntimeError(f"orc_setup failed with status {self.status}")
        self.n = g.n

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_free(self._h)
            self._h = None

    @property
    def nlev(self) -> int:
        return lib().orc_nlev(self._h)

    def perm(self) -> np.ndarray:
        # orc_hier layout: nlev(i32), status(i32), n0(i64), perm(ptr)
        class _H(ctypes.Structure):
            _fields_ = [("nlev", ctypes.c_int32), ("status", ctypes.c_int32), ("n0", ctypes.c_int64),
                        ("perm", ctypes.POINTER(ctypes.c_int64))]
        hh = ctypes.cast(self._h, ctypes.POINTER(_H)).contents
        return _arr(hh.perm, hh.n0, np.int64)

    def level(self, l: int) -> LevelData:
        L = lib().orc_get_level(self._h, l).contents
        n, z = L.n, L.nnz
        ld = LevelData(L.kind, n, z, _arr(L.row_ptr, n + 1, np.int64), _arr(L.col, z, np.int32),
                       _arr(L.w, z, np.float64), _arr(L.d, n, np.float64))
        if L.kind == AGG:
            ld.lam, ld.m = L.lam, L.m
            ld.agg = _arr(L.agg, n, np.int32)
            ld.S = _arr(L.S, z, np.float64)
        elif L.kind == ELIM:
            ld.nF = L.nF
            ld.fmap = _arr(L.fmap, n, np.int32)
        else:
            ld.pinv = _arr(L.pinv, n * n, np.float64).reshape(n, n)
        return ld

    def levels(self):
        return [self.level(l) for l in range(self.nlev)]

    def level_view(self, l: int) -> LevelData:
        """level(l) without copies: numpy views into the oracle's memory, valid
        while this Hierarchy is alive (cfg 5 levels hold ~25 GB each)."""
        L = lib().orc_get_level(self._h, l).contents
        n, z = L.n, L.nnz

        def v(ptr, cnt, dt):
            if cnt <= 0 or not ptr:
                return np.zeros(0, dtype=dt)
            return np.ctypeslib.as_array(ptr, shape=(cnt,))
        ld = LevelData(L.kind, n, z, v(L.row_ptr, n + 1, np.int64), v(L.col, z, np.int32), v(L.w, z, np.float64),
                       v(L.d, n, np.float64))
        if L.kind == AGG:
            ld.lam, ld.m = L.lam, L.m
            ld.agg = v(L.agg, n, np.int32)
        elif L.kind == ELIM:
            ld.nF = L.nF
            ld.fmap = v(L.fmap, n, np.int32)
        else:
            ld.pinv = v(L.pinv, n * n, np.float64).reshape(n, n)
        return ld

    def export(self, path: str) -> None:
        """Write the hierarchy in the interchange format (
        include/lap.h lap_import_hierarchy): meta.json, perm.i64, and per level
        L<l>/meta.json, row_ptr.i64, col.i32, w.f64, d.f64 and agg.i32 /
        fmap.i32 / coarse_pinv.f64 (little-endian raw arrays)."""
        os.makedirs(path, exist_ok=True)
        p = self.params
        meta = {"format": "lap-hierarchy-v1", "producer": "oracle/lap_oracle.c", "nlev": self.nlev, "n0": self.n,
                "params": {f: getattr(p, f) for f, _ in p._fields_}}
        with open(os.path.join(path, "meta.json"), "w") as f:
            json.dump(meta, f)
        self.perm().astype("<i8").tofile(os.path.join(path, "perm.i64"))
        for l in range(self.nlev):
            L = self.level_view(l)
            d = os.path.join(path, f"L{l}")
            os.makedirs(d, exist_ok=True)
            lm = {"kind": L.kind, "n": L.n, "nnz": L.nnz}
            if L.kind == AGG:
                lm.update(**{"lambda": float(L.lam), "m": int(L.m)})
            elif L.kind == ELIM:
                lm["nF"] = int(L.nF)
            with open(os.path.join(d, "meta.json"), "w") as f:
                json.dump(lm, f)
            L.row_ptr.astype("<i8").tofile(os.path.join(d, "row_ptr.i64"))
            L.col.astype("<i4").tofile(os.path.join(d, "col.i32"))
            L.w.astype("<f8").tofile(os.path.join(d, "w.f64"))
            L.d.astype("<f8").tofile(os.path.join(d, "d.f64"))
            if L.kind == AGG:
                L.agg.astype("<i4").tofile(os.path.join(d, "agg.i32"))
            elif L.kind == ELIM:
                L.fmap.astype("<i4").tofile(os.path.join(d, "fmap.i32"))
            else:
                L.pinv.astype("<f8").tofile(os.path.join(d, "coarse_pinv.f64"))

    def vcycle(self, l: int, b) -> np.ndarray:
        n = self.level(l).n
        x = np.zeros(n)
        lib().orc_vcycle(self._h, l, _p(_c(b, np.float64)), _p(x))
        return x

    def kcycle(self, l: int, b) -> np.ndarray:
        """K-cycle at level l (N2): x = K_l b."""
        x = np.zeros(self.level(l).n)
        lib().orc_kcycle(self._h, l, _p(_c(b, np.float64)), _p(x))
        return x

    def kcoarse(self, l: int, b) -> np.ndarray:
        """The K-cycle's coarse problem at level l: kcycle_inner FCG(1)
        iterations preconditioned by K_l (aggregation levels), else K_l b."""
        x = np.zeros(self.level(l).n)
        lib().orc_kcoarse(self._h, l, _p(_c(b, np.float64)), _p(x))
        return x

    def solve(self, b, tol: float | None = None):
        tol = self.params.tol if tol is None else tol
        x = np.zeros(self.n)
        it = ctypes.c_int32(0)
        rr = ctypes.c_double(0.0)
        rc = lib().orc_solve(self._h, _p(_c(b, np.float64)), _p(x), tol, ctypes.byref(it), ctypes.byref(rr))
        return x, int(it.value), float(rr.value), rc
