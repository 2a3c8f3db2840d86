"""lapgen -- seeded synthetic inputs for the graph-Laplacian hot path.

INPUT GENERATION ONLY: this module holds none of the solver method's
arithmetic (no hashing of vertex ids, no sums of Laplacian entries, no
aggregation or elimination logic).  It is the one module that both the CPU
oracle (``oracle/``) and the CUDA library (``paper_1705_06266_b200``) are fed
from, so that both sides read identical bytes.

Workloads (BASELINE.json ``configs``; recipes in DESIGN.md §Inputs):

  cfg 1  2D 5-point grid 64x64, unit weights
  cfg 2  3D 7-point grid 128^3, weights 10^(-3u), u ~ U[0,1) (default_rng(1))
  cfg 3  R-MAT scale 20, edge factor 16, (a,b,c,d)=(.57,.19,.19,.05), LCC, unit w
  cfg 4  Barabasi-Albert n=4,194,304, m=8, w ~ U[0.5,2) (default_rng(2))
  cfg 5  R-MAT scale 26 (counter-based generator), LCC, unit w

The paper's own graphs (UF collection, SNAP social graphs, P:268, P:738,
P:778-789) are not available; these synthetic graphs stand in for them.
RHS: ``default_rng(0).standard_normal(n)`` with the mean subtracted (P:670,
BASELINE.json configs[0], SURVEY O-R32).
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libgen.so")
GEN_VERSION = "lapgen-v1"


@dataclass
class Graph:
    """Symmetric off-diagonal adjacency in CSR (the lap_graph contract)."""
    n: int
    row_ptr: np.ndarray  # int64[n+1]
    col: np.ndarray      # int32[nnz], ascending per row, no self loops
    w: np.ndarray        # float64[nnz], w_ij == w_ji, > 0
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def degrees(self) -> np.ndarray:
        return np.diff(self.row_ptr)


def build_lib(force: bool = False) -> str:
    src = os.path.join(_HERE, "_gen.c")
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-shared", "-fPIC", "-o", _LIB, src])
    return _LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        build_lib()
        _lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        _lib.gen_barabasi_albert.restype = ctypes.c_int64
        _lib.gen_barabasi_albert.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, P, P, ctypes.c_int64]
        _lib.gen_rmat.restype = None
        _lib.gen_rmat.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                  ctypes.c_double, ctypes.c_uint64, P, P]
        _lib.gen_rmat_lcc_build.restype = ctypes.c_void_p
        _lib.gen_rmat_lcc_build.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                            ctypes.c_double, ctypes.c_uint64, P, P]
        _lib.gen_rmat_lcc_fetch.restype = None
        _lib.gen_rmat_lcc_fetch.argtypes = [ctypes.c_void_p, P, P]
        _lib.gen_csr_from_edges.restype = None
        _lib.gen_csr_from_edges.argtypes = [ctypes.c_int64, ctypes.c_int64, P, P, P, P, P, P]
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def csr_from_edges(n: int, u, v, w=None, name: str = "") -> Graph:
    """Undirected edge list (no self loops, no duplicates) -> symmetric CSR."""
    u = np.ascontiguousarray(u, dtype=np.int64)
    v = np.ascontiguousarray(v, dtype=np.int64)
    ne = len(u)
    if w is None:
        w = np.ones(ne, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    col = np.zeros(2 * ne, dtype=np.int32)
    val = np.zeros(2 * ne, dtype=np.float64)
    _L().gen_csr_from_edges(n, ne, _ptr(u), _ptr(v), _ptr(w), _ptr(row_ptr), _ptr(col), _ptr(val))
    return Graph(n, row_ptr, col, val, name)


def dedup_undirected(u, v):
    """Drop self loops, canonicalise (min,max), deduplicate."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    keep = u != v
    u, v = u[keep], v[keep]
    a = np.minimum(u, v)
    b = np.maximum(u, v)
    key = np.unique(a * (np.int64(1) << 32) + b)
    return key >> 32, key & 0xFFFFFFFF


def largest_component(g: Graph) -> Graph:
    """Largest connected component, vertices relabelled by ascending original id."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components
    m = csr_matrix((np.ones(g.nnz, dtype=np.int8), g.col, g.row_ptr), shape=(g.n, g.n))
    ncomp, lab = connected_components(m, directed=False)
    if ncomp == 1:
        return g
    big = np.argmax(np.bincount(lab))
    keep = lab == big
    newid = np.cumsum(keep) - 1
    rows = np.repeat(np.arange(g.n), g.degrees())
    sel = keep[rows] & (rows < g.col)  # one direction of every kept edge
    u = newid[rows[sel]]
    v = newid[g.col[sel]]
    return csr_from_edges(int(keep.sum()), u, v, g.w[sel], g.name)


# --------------------------------------------------------------------------
# BASELINE.json workloads
# --------------------------------------------------------------------------

def grid2d(nx: int = 64, ny: int = 64, name: str = "") -> Graph:
    """2D 5-point grid, id = x + nx*y, unit weights (configs[0])."""
    ids = np.arange(nx * ny, dtype=np.int64).reshape(ny, nx)
    u = np.concatenate([ids[:, :-1].ravel(), ids[:-1, :].ravel()])
    v = np.concatenate([ids[:, 1:].ravel(), ids[1:, :].ravel()])
    return csr_from_edges(nx * ny, u, v, None, name or f"grid2d_{nx}x{ny}")


def grid3d(n: int = 128, weighted: bool = True, seed: int = 1, name: str = "") -> Graph:
    """3D 7-point grid, id = x + n*y + n^2*z (configs[1]).

    Edge weights w_e = 10**(-3 u_e), u_e = default_rng(seed).random(|E|) drawn
    per undirected edge in the order x-edges, y-edges, z-edges, each by
    ascending lower endpoint (log-uniform on [1e-3, 1])."""
    ids = np.arange(n ** 3, dtype=np.int64).reshape(n, n, n)  # [z, y, x]
    ux, vx = ids[:, :, :-1].ravel(), ids[:, :, 1:].ravel()
    uy, vy = ids[:, :-1, :].ravel(), ids[:, 1:, :].ravel()
    uz, vz = ids[:-1, :, :].ravel(), ids[1:, :, :].ravel()
    u = np.concatenate([ux, uy, uz])
    v = np.concatenate([vx, vy, vz])
    w = None
    if weighted:
        w = 10.0 ** (-3.0 * np.random.default_rng(seed).random(len(u)))
    return csr_from_edges(n ** 3, u, v, w, name or f"grid3d_{n}")


def rmat(scale: int = 20, edge_factor: int = 16, abcd=(0.57, 0.19, 0.19, 0.05),
         seed: int = 0, name: str = "") -> Graph:
    """R-MAT (configs[2]); numpy PCG64(seed), one uniform per edge per level.

    Quadrant: u-bit set for c and d, v-bit for b and d.  Self loops dropped,
    duplicates merged, symmetrised, largest connected component, unit w."""
    a, b, c, _ = abcd
    ne = edge_factor << scale
    rng = np.random.default_rng(seed)
    u = np.zeros(ne, dtype=np.int64)
    v = np.zeros(ne, dtype=np.int64)
    for _lvl in range(scale):
        x = rng.random(ne)
        ub = x >= a + b
        vb = ((x >= a) & (x < a + b)) | (x >= a + b + c)
        u = (u << 1) | ub
        v = (v << 1) | vb
    u, v = dedup_undirected(u, v)
    g = csr_from_edges(1 << scale, u, v, None, name or f"rmat_s{scale}")
    return largest_component(g)


def rmat_large_reference(scale: int, edge_factor: int = 16, abcd=(0.57, 0.19, 0.19, 0.05),
                         seed: int = 0, name: str = "") -> Graph:
    """R-MAT from the counter-based C edge stream, post-processed in numpy /
    scipy (small scales: the check of rmat_large's C pipeline)."""
    a, b, c, _ = abcd
    ne = edge_factor << scale
    u = np.zeros(ne, dtype=np.int64)
    v = np.zeros(ne, dtype=np.int64)
    _L().gen_rmat(scale, ne, a, b, c, seed, _ptr(u), _ptr(v))
    u, v = dedup_undirected(u, v)
    g = csr_from_edges(1 << scale, u, v, None, name or f"rmat_s{scale}")
    return largest_component(g)


def rmat_large(scale: int = 26, edge_factor: int = 16, abcd=(0.57, 0.19, 0.19, 0.05),
               seed: int = 0, name: str = "", unit_weights_array: bool = False) -> Graph:
    """R-MAT with the counter-based C generator (configs[4]; scale 26): edge
    stream, dedup, LCC and symmetric CSR all in C/OpenMP (gen_rmat_lcc_build),
    identical to rmat_large_reference.  Unit weights: w is None (the lap_graph
    contract's NULL = unit) unless unit_weights_array."""
    a, b, c, _ = abcd
    ne = edge_factor << scale
    n = ctypes.c_int64()
    nnz = ctypes.c_int64()
    h = _L().gen_rmat_lcc_build(scale, ne, a, b, c, seed, ctypes.byref(n), ctypes.byref(nnz))
    row_ptr = np.empty(n.value + 1, np.int64)
    col = np.empty(nnz.value, np.int32)
    _L().gen_rmat_lcc_fetch(h, _ptr(row_ptr), _ptr(col))
    w = np.ones(nnz.value) if unit_weights_array else None
    return Graph(n.value, row_ptr, col, w, name or f"rmat_s{scale}")


def barabasi_albert(n: int = 4194304, m: int = 8, seed: int = 0, wseed: int = 2,
                    wlo: float = 0.5, whi: float = 2.0, name: str = "") -> Graph:
    """Barabasi-Albert (configs[3]): clique K_{m+1}, then m distinct
    degree-proportional targets per new vertex; w ~ U[wlo, whi) per edge from
    default_rng(wseed).  Connected by construction."""
    k0 = min(m + 1, n)
    cap = k0 * (k0 - 1) // 2 + (n - k0) * m
    eu = np.zeros(cap, dtype=np.int32)
    ev = np.zeros(cap, dtype=np.int32)
    ne = _L().gen_barabasi_albert(n, m, seed, _ptr(eu), _ptr(ev), cap)
    assert ne == cap
    w = np.random.default_rng(wseed).uniform(wlo, whi, ne)
    return csr_from_edges(n, eu.astype(np.int64), ev.astype(np.int64), w, name or f"ba_{n}_{m}")


def rhs(n: int, seed: int = 0) -> np.ndarray:
    """N(0,1) right-hand side with the constant projected out."""
    b = np.random.default_rng(seed).standard_normal(n)
    return b - b.mean()


# --------------------------------------------------------------------------
# small fixtures for tests
# --------------------------------------------------------------------------

def path(n: int, w=None) -> Graph:
    return csr_from_edges(n, np.arange(n - 1), np.arange(1, n), w, f"path{n}")


def cycle(n: int) -> Graph:
    return csr_from_edges(n, np.arange(n), (np.arange(n) + 1) % n, None, f"cycle{n}")


def star(n_leaves: int) -> Graph:
    return csr_from_edges(n_leaves + 1, np.zeros(n_leaves, dtype=np.int64),
                          np.arange(1, n_leaves + 1), None, f"star{n_leaves + 1}")


def complete(n: int) -> Graph:
    iu = np.triu_indices(n, 1)
    return csr_from_edges(n, iu[0], iu[1], None, f"K{n}")


def random_connected(n: int, extra: int, seed: int, weighted: bool = True, name: str = "") -> Graph:
    """Random spanning tree plus `extra` random edges; mixed degrees."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    parents = np.array([rng.integers(0, i) for i in range(1, n)], dtype=np.int64) if n > 1 else np.zeros(0, np.int64)
    u = perm[1:] if n > 1 else np.zeros(0, np.int64)
    v = perm[parents] if n > 1 else np.zeros(0, np.int64)
    if extra > 0 and n > 2:
        eu = rng.integers(0, n, extra)
        ev = rng.integers(0, n, extra)
        u = np.concatenate([u, eu])
        v = np.concatenate([v, ev])
    u, v = dedup_undirected(u, v)
    w = rng.uniform(0.1, 3.0, len(u)) if weighted else None
    return csr_from_edges(n, u, v, w, name or f"rand{n}_{seed}")


def config(k: int) -> Graph:
    """BASELINE.json configs[k-1] graph (cached on disk under LAPGEN_CACHE)."""
    makers = {
        1: lambda: grid2d(64, 64, "cfg1_grid2d_64"),
        2: lambda: grid3d(128, True, 1, "cfg2_grid3d_128"),
        3: lambda: rmat(20, 16, name="cfg3_rmat_s20"),
        4: lambda: barabasi_albert(4194304, 8, name="cfg4_ba_4M_8"),
        5: lambda: rmat_large(26, 16, name="cfg5_rmat_s26"),
    }
    cache = os.environ.get("LAPGEN_CACHE", os.path.join(os.path.expanduser("~"), ".cache", "lapgen"))
    tag = hashlib.sha256(f"{GEN_VERSION}-cfg{k}".encode()).hexdigest()[:12]
    fn = os.path.join(cache, f"cfg{k}_{tag}.npz")
    if k >= 2 and os.path.exists(fn):
        try:
            z = np.load(fn)
            w = z["w"] if z["w"].size else None  # cfg 5: unit weights are not materialised
            return Graph(int(z["n"]), z["row_ptr"], z["col"], w, str(z["name"]))
        except Exception:
            pass
    g = makers[k]()
    if k >= 2:
        try:
            os.makedirs(cache, exist_ok=True)
            tmp = fn + f".tmp{os.getpid()}.npz"
            np.savez(tmp, n=g.n, row_ptr=g.row_ptr, col=g.col, w=g.w if g.w is not None else np.zeros(0), name=g.name)
            os.replace(tmp, fn)
        except OSError:
            pass
    return g


CONFIG_NAMES = {
    1: "cfg1: 2D 5-pt grid 64x64, unit w",
    2: "cfg2: 3D 7-pt grid 128^3, log-uniform w in [1e-3,1]",
    3: "cfg3: R-MAT s20 ef16 LCC, unit w",
    4: "cfg4: Barabasi-Albert n=4194304 m=8, w~U[0.5,2]",
    5: "cfg5: R-MAT s26 ef16 LCC, unit w",
}
