"""GPU parity: liblap.so (through the C ABI) against the CPU oracle.

Contract (BASELINE.json north_star):
  - aggregates, F sets, every coarse operator (col, w, d) and S: bit-exact
  - SpMV: |dy_i| <= 1e-12 (d_i |x_i| + sum_j w_ij |x_j|)   (O-P2)
  - lambda-hat: bit-exact (canonical-sum Lanczos on both sides, DESIGN.md
    reading R-lambda; SURVEY's contract asks <= 1e-10 relative)
  - solve: true relative residual <= 1e-8, iterations within +-1 of the oracle
"""
import numpy as np
import pytest

import lapgen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    import paper_1705_06266_b200 as P
    from paper_1705_06266_b200 import build
    build.build()
    return P


def _bits(a):
    return np.asarray(a, np.float64).view(np.int64)


def compare_hierarchy(h, ho, check_S=False):
    assert h.nlev == ho.nlev
    for l in range(ho.nlev):
        a, o = h.level(l), ho.level(l)
        assert (a["kind"], a["n"], a["nnz"]) == (o.kind, o.n, o.nnz), f"level {l}"
        assert np.array_equal(a["row_ptr"], o.row_ptr), f"row_ptr level {l}"
        assert np.array_equal(a["col"], o.col), f"col level {l}"
        assert np.array_equal(_bits(a["w"]), _bits(o.w)), f"w level {l}"
        assert np.array_equal(_bits(a["d"]), _bits(o.d)), f"d level {l}"
        if o.kind == oracle.AGG:
            assert np.array_equal(a["agg"], o.agg), f"agg level {l}"
            # lambda-hat: every Lanczos sum is a CanonSum on both sides (reading R-lambda),
            # so the tridiagonal and its bisection are bit-identical
            assert _bits(a["lam"]) == _bits(o.lam), (l, a["lam"], o.lam)
            if check_S:
                assert np.array_equal(_bits(h.strength(l)), _bits(o.S)), f"S level {l}"
        elif o.kind == oracle.ELIM:
            assert np.array_equal(a["fmap"], o.fmap), f"fmap level {l}"
        else:
            assert np.allclose(a["pinv"], o.pinv, rtol=0, atol=1e-9 * max(1.0, np.abs(o.pinv).max()))


def spmv_bound(row_ptr, col, w, d, x):
    rows = np.repeat(np.arange(len(d)), np.diff(row_ptr))
    s = np.zeros(len(d))
    np.add.at(s, rows, np.abs(w) * np.abs(x[col]))
    return 1e-12 * (np.abs(d) * np.abs(x) + s)


SMALL = [
    lambda: lapgen.grid2d(64, 64, "cfg1"),
    lambda: lapgen.grid2d(37, 29),
    lambda: lapgen.grid3d(12),
    lambda: lapgen.rmat(12),
    lambda: lapgen.barabasi_albert(5000, 8),
    lambda: lapgen.random_connected(3000, 9000, 7),
    lambda: lapgen.path(777),
    lambda: lapgen.star(40000),          # hub row > 16384 entries: split-chunk SpMV path
    lambda: lapgen.complete(70),
    lambda: lapgen.complete(400),                     # avg degree >= 256, n small: k_spmv_smem (x in shared memory)
    lambda: lapgen.random_connected(6000, 900000, 11),  # dense-ish random level (avg degree ~300): k_spmv_smem
]


@pytest.mark.parametrize("mk", SMALL, ids=["cfg1", "grid37x29", "grid3d12", "rmat12", "ba5000", "rand3000",
                                           "path777", "star40000", "K70", "K400", "dense6000"])
def test_hierarchy_spmv_vcycle_solve_parity(P, mk):
    g = mk()
    h = P.Hierarchy(g, keep_strength=1)
    ho = oracle.Hierarchy(g)
    compare_hierarchy(h, ho, check_S=True)
    assert np.array_equal(h.perm(), ho.perm())
    rng = np.random.default_rng(0)
    # H1 on every level, device pointers through the C ABI
    for l in range(ho.nlev):
        o = ho.level(l)
        x = rng.standard_normal(o.n)
        y = h.spmv(l, torch.from_numpy(x).cuda()).cpu().numpy()
        yo = oracle.spmv(o.n, o.row_ptr, o.col, o.w, o.d, x)
        assert np.all(np.abs(y - yo) <= spmv_bound(o.row_ptr, o.col, o.w, o.d, x) + 1e-300), f"spmv level {l}"
    # one V-cycle (O-S7) in the internal numbering
    r = rng.standard_normal(g.n)
    r -= r.mean()
    z = h.vcycle(torch.from_numpy(r).cuda()).cpu().numpy()
    zo = ho.vcycle(0, r)
    assert np.abs(z - zo).max() <= 1e-9 * np.abs(zo).max()
    # full solve, host buffers (O-S8)
    b = lapgen.rhs(g.n, seed=3)
    x, it, rr, rc = h.solve(b)
    xo, ito, rro, rco = ho.solve(b)
    assert rc == rco == 0
    assert rr <= 1e-8 and abs(it - ito) <= 1, (it, ito, rr)
    assert np.abs(x - xo).max() <= 1e-6 * np.abs(xo).max()
    assert abs(x.mean()) <= 1e-10 * np.abs(x).max()


def test_degenerate_inputs(P):
    # n = 1: coarsest only, x = 0
    g1 = lapgen.Graph(1, np.array([0, 0], np.int64), np.zeros(0, np.int32), np.zeros(0))
    h = P.Hierarchy(g1)
    x, it, rr, rc = h.solve(np.array([5.0]))
    assert h.nlev == 1 and it == 0 and x.tolist() == [0.0]
    # constant RHS projects to zero
    g = lapgen.grid2d(20, 20)
    h = P.Hierarchy(g)
    x, it, rr, rc = h.solve(np.full(g.n, 2.0))
    assert it == 0 and np.all(x == 0)
    # single edge
    g2 = lapgen.path(2)
    x, it, rr, rc = P.Hierarchy(g2).solve(np.array([1.0, -1.0]))
    assert np.allclose(x, [0.5, -0.5])


@pytest.mark.parametrize("mode", ["hash", "sort", "search"])
def test_symmetry_check_modes(mode):
    """The three symmetry checks (LAP_SYMCHECK: the default multiset
    fingerprint computed by k_validate, the exact transposed sort, the exact
    per-entry search) accept symmetric graphs and reject asymmetric ones: a
    one-ulp weight change, a missing reverse entry, weights swapped between two
    edges (w_ij = w_kl = a, w_ji = w_lk = b), on a random weighted graph."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np, lapgen, paper_1705_06266_b200 as P\n"
            "g = lapgen.barabasi_albert(3000, 4)\n"
            "h = P.Hierarchy(g); assert h.nlev >= 2\n"
            "rp, col, w = g.row_ptr.copy(), g.col.copy(), g.w.copy()\n"
            "def rev(i, j):\n"
            "    return rp[j] + int(np.searchsorted(col[rp[j]:rp[j + 1]], i))\n"
            "def bad(rp2, col2, w2):\n"
            "    try:\n"
            "        P.Hierarchy(lapgen.Graph(len(rp2) - 1, rp2, col2, w2)); return False\n"
            "    except P.LapError as e:\n"
            "        return e.code == P.LAP_EGRAPH\n"
            "rng = np.random.default_rng(7)\n"
            "for t in range(5):\n"
            "    k = int(rng.integers(len(col))); w2 = w.copy(); w2[k] = np.nextafter(w2[k], 9.0)\n"
            "    assert bad(rp, col, w2), 'ulp'\n"
            "    i = int(np.searchsorted(rp, k, side='right') - 1); j = int(col[k]); k2 = rev(i, j)\n"
            "    assert k2 != k and col[k2] == i\n"
            "    w3 = w.copy(); w3[k], w3[k2] = 1.0, 2.0\n"
            "    k3 = int(rng.integers(len(col))); i3 = int(np.searchsorted(rp, k3, side='right') - 1); j3 = int(col[k3])\n"
            "    k4 = rev(i3, j3)\n"
            "    if len({k, k2, k3, k4}) == 4:\n"
            "        w3[k3], w3[k4] = 1.0, 2.0  # (i,j,1) (j,i,2) (i3,j3,1) (j3,i3,2): swapped, still asymmetric\n"
            "        assert bad(rp, col, w3), 'swap'\n"
            "    keep = np.ones(len(col), bool); keep[k2] = False\n"
            "    rp4 = rp.copy(); rp4[j + 1:] -= 1\n"
            "    assert bad(rp4, col[keep], w[keep]), 'missing'\n"
            "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ, LAP_SYMCHECK=mode)
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


def test_invalid_graphs_rejected(P):
    bad_sym = lapgen.Graph(2, np.array([0, 1, 1]), np.array([1], np.int32), np.array([1.0]))
    with pytest.raises(P.LapError) as e:
        P.Hierarchy(bad_sym)
    assert e.value.code == P.LAP_EGRAPH
    neg = lapgen.Graph(2, np.array([0, 1, 2]), np.array([1, 0], np.int32), np.array([-1.0, -1.0]))
    with pytest.raises(P.LapError) as e:
        P.Hierarchy(neg)
    assert e.value.code == P.LAP_EGRAPH
    loop = lapgen.Graph(2, np.array([0, 2, 3]), np.array([0, 1, 0], np.int32), np.ones(3))
    with pytest.raises(P.LapError) as e:
        P.Hierarchy(loop)
    assert e.value.code == P.LAP_EGRAPH
    # pattern symmetric, weights not bitwise equal (w_01 != w_10)
    asym_w = lapgen.Graph(3, np.array([0, 1, 3, 4]), np.array([1, 0, 2, 1], np.int32),
                          np.array([1.0, np.nextafter(1.0, 2.0), 2.0, 2.0]))
    with pytest.raises(P.LapError) as e:
        P.Hierarchy(asym_w)
    assert e.value.code == P.LAP_EGRAPH
    # unsorted columns / duplicate entry
    dup = lapgen.Graph(3, np.array([0, 2, 3, 4]), np.array([1, 1, 0, 0], np.int32), np.ones(4))
    with pytest.raises(P.LapError) as e:
        P.Hierarchy(dup)
    assert e.value.code == P.LAP_EGRAPH
    disc = lapgen.csr_from_edges(4, [0, 2], [1, 3])
    with pytest.raises(P.LapError) as e:
        P.Hierarchy(disc)
    assert e.value.code == P.LAP_EDISCONNECTED


def test_device_graph_and_determinism(P):
    g = lapgen.rmat(11)
    dev = lapgen.Graph(g.n, torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col).cuda(),
                       torch.from_numpy(g.w).cuda())
    h1 = P.Hierarchy(dev)
    h2 = P.Hierarchy(g)
    compare_hierarchy(h1, oracle.Hierarchy(g))
    b = lapgen.rhs(g.n)
    x1, i1, r1, _ = h1.solve(b)
    x2, i2, r2, _ = h2.solve(b)
    assert i1 == i2 and np.array_equal(_bits(x1), _bits(x2))   # bitwise run-to-run reproducible


@pytest.mark.parametrize("kw", [dict(random_order=0), dict(affinity_power=2), dict(seed=5),
                                dict(elim_enable=0), dict(cheby_degree=3), dict(use_graphs=0),
                                dict(elim_rounds=3)])
def test_parameter_variants(P, kw):
    g = lapgen.path(5000) if "elim_rounds" in kw else lapgen.rmat(11)  # path: consecutive elimination levels
    h = P.Hierarchy(g, **kw)
    okw = {k: v for k, v in kw.items() if k != "use_graphs"}
    ho = oracle.Hierarchy(g, **okw)
    compare_hierarchy(h, ho)
    b = lapgen.rhs(g.n)
    x, it, rr, rc = h.solve(b)
    xo, ito, _, _ = ho.solve(b)
    assert rr <= 1e-8 and abs(it - ito) <= 1


FULL = {2: "cfg2", 3: "cfg3", 4: "cfg4"}


@pytest.mark.slow
@pytest.mark.parametrize("k", [2, 3, 4])
def test_full_size_configs(P, k):
    """BASELINE.json configs at full size, default (bench) launch configuration:
    bit-exact hierarchy (lambda-hat included), per-entry SpMV check on every
    row of every level, solve residual and iterations."""
    g = lapgen.config(k)
    h = P.Hierarchy(g)
    ho = oracle.Hierarchy(g)
    compare_hierarchy(h, ho)
    rng = np.random.default_rng(k)
    # H1 per entry (O-P2 bound) on EVERY level and EVERY row, in the bench's launch configuration
    for l in range(ho.nlev):
        o = ho.level(l)
        x = rng.standard_normal(o.n)
        y = h.spmv(l, torch.from_numpy(x).cuda()).cpu().numpy()
        yo = oracle.spmv(o.n, o.row_ptr, o.col, o.w, o.d, x)
        bound = spmv_bound(o.row_ptr, o.col, o.w, o.d, x)
        bad = np.flatnonzero(np.abs(y - yo) > bound + 1e-300)
        assert bad.size == 0, (l, bad[:10])
    b = lapgen.rhs(g.n)
    bt = torch.from_numpy(b).cuda()
    xg, it, rr, rc = h.solve(bt)
    xo, ito, rro, _ = ho.solve(b)
    assert rc == 0 and rr <= 1e-8 and abs(it - ito) <= 1, (it, ito, rr)
    xg = xg.cpu().numpy()
    assert np.abs(xg - xo).max() <= 1e-6 * np.abs(xo).max()


def test_storage_layout_validated_in_debug_mode(P):
    """LAP_DEBUG_SYNC=1 turns on host-side validation of every level's storage
    layout (permutation, class ranges, SELL slices incl. ragged last slice) and
    a device sync after every launch."""
    import subprocess
    import sys
    code = ("import lapgen, paper_1705_06266_b200 as P\n"
            "for g in [lapgen.grid3d(23), lapgen.rmat(12), lapgen.barabasi_albert(3001, 5), lapgen.star(20000)]:\n"
            "    h = P.Hierarchy(g); x, it, rr, rc = h.solve(lapgen.rhs(g.n)); assert rr <= 1e-8, rr\n"
            "print('ok')\n")
    env = dict(__import__("os").environ, LAP_DEBUG_SYNC="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600,
                       cwd=__import__("os").path.dirname(__import__("os").path.dirname(__file__)))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("env", [{"LAP_DENSE_TAIL": "0"}, {"LAP_PDL": "0"}, {"LAP_FUSE_TRANSFERS": "0"},
                                 {"LAP_FUSE_ZSUMS": "0"}, {"LAP_SPMV_VEC": "0"}, {"LAP_SPMV_VEC": "16"},
                                 {"LAP_DENSE_TAIL": "0", "LAP_PDL": "0", "LAP_FUSE_TRANSFERS": "0", "LAP_FUSE_ZSUMS": "0"},
                                 {"LAP_XT": "force", "LAP_XT_W": "64"}, {"LAP_XT": "force", "LAP_XT_W": "1000", "LAP_XT_NB": "300"},
                                 {"LAP_XT": "1"}],
                         ids=["no-dense-tail", "no-pdl", "no-fused-transfers", "no-fused-zsums", "sell-only",
                              "vec16-everywhere", "none", "xt-forced-w64", "xt-forced-nb300", "xt-rule"])
def test_solve_path_switches(P, env):
    """The alternative solve paths (per-level kernels instead of the dense
    tail operator, launches without programmatic dependent launch) give the
    oracle's V-cycle and solution too (run in a subprocess: the switches are
    read once per process)."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np, lapgen, oracle, paper_1705_06266_b200 as P\n"
            "for g in [lapgen.grid2d(64, 64), lapgen.rmat(12), lapgen.grid3d(16)]:\n"
            "    h = P.Hierarchy(g); ho = oracle.Hierarchy(g)\n"
            "    r = np.random.default_rng(1).standard_normal(g.n); r -= r.mean()\n"
            "    z = h.vcycle(r); zo = ho.vcycle(0, r)\n"
            "    assert np.abs(z - zo).max() <= 1e-9 * np.abs(zo).max()\n"
            "    b = lapgen.rhs(g.n, seed=4); x, it, rr, rc = h.solve(b); xo, ito, _, _ = ho.solve(b)\n"
            "    assert rc == 0 and rr <= 1e-8 and abs(it - ito) <= 1, (it, ito, rr)\n"
            "print('ok')\n")
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_fused_transfers_bitwise(P, tmp_path):
    """Forming an aggregation level's pre-smoothing step 0 inside the
    restriction of the elimination level above it is the same arithmetic:
    V-cycle outputs are bit-identical with LAP_FUSE_TRANSFERS=0 (graphs with
    elimination levels above aggregation levels, per-level path so no level
    is folded into the dense tail)."""
    import os
    import subprocess
    import sys
    code = ("import sys, numpy as np, lapgen, paper_1705_06266_b200 as P\n"
            "out = []\n"
            "for g in [lapgen.rmat(13), lapgen.barabasi_albert(20000, 3), lapgen.grid2d(200, 150)]:\n"
            "    h = P.Hierarchy(g)\n"
            "    r = np.random.default_rng(2).standard_normal(g.n); r -= r.mean()\n"
            "    out.append(h.vcycle(r))\n"
            "np.save(sys.argv[1], np.concatenate(out))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for fuse in ["1", "0"]:
        f = str(tmp_path / f"z{fuse}.npy")
        e = dict(os.environ, LAP_FUSE_TRANSFERS=fuse, LAP_DENSE_TAIL="0")
        r = subprocess.run([sys.executable, "-c", code, f], env=e, capture_output=True, text=True, timeout=600, cwd=root)
        assert r.returncode == 0, r.stderr[-2000:]
        res.append(np.load(f))
    assert res[0].tobytes() == res[1].tobytes()


def test_memory_lean_paths_bit_exact(P):
    """The memory-lean and alternative setup paths give the oracle's hierarchy
    bit for bit: terms built in many small batches of output rows
    (LAP_TERM_BATCH; with the shared-memory Galerkin only its hub rows take
    that path), the global-sort Galerkin (LAP_GAL_FAST=0), the exact
    search- / sort-based symmetry checks (LAP_SYMCHECK), and released logical
    copies (keep_logical = 0) read back through lap_level_rows."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np, lapgen, oracle, paper_1705_06266_b200 as P\n"
            "for g in [lapgen.rmat(12), lapgen.barabasi_albert(6000, 8), lapgen.grid3d(14), lapgen.star(9000)]:\n"
            "    ho = oracle.Hierarchy(g)\n"
            "    h = P.Hierarchy(g)\n"
            "    assert h.nlev == ho.nlev\n"
            "    for l in range(ho.nlev):\n"
            "        a, o = h.level(l), ho.level(l)\n"
            "        assert (a['n'], a['nnz']) == (o.n, o.nnz)\n"
            "        assert np.array_equal(a['col'], o.col) and a['w'].tobytes() == o.w.tobytes() and a['d'].tobytes() == o.d.tobytes(), l\n"
            "        assert np.float64(a['lam']).tobytes() == np.float64(o.lam).tobytes()\n"
            "    hr = P.Hierarchy(g, keep_logical=0)\n"
            "    for l in range(ho.nlev):\n"
            "        o = ho.level(l)\n"
            "        rows = np.arange(o.n)\n"
            "        rp, col, w = hr.level_rows(l, rows)\n"
            "        assert np.array_equal(rp, o.row_ptr) and np.array_equal(col, o.col) and w.tobytes() == o.w.tobytes(), l\n"
            "    b = lapgen.rhs(g.n); x, it, rr, rc = hr.solve(b); xo, ito, _, _ = ho.solve(b)\n"
            "    assert rc == 0 and rr <= 1e-8 and abs(it - ito) <= 1\n"
            "bad = lapgen.Graph(3, np.array([0, 1, 3, 4]), np.array([1, 0, 2, 1], np.int32), np.array([1.0, np.nextafter(1.0, 2.0), 2.0, 2.0]))\n"
            "try:\n"
            "    P.Hierarchy(bad); raise SystemExit('accepted an asymmetric graph')\n"
            "except P.LapError as e:\n"
            "    assert e.code == P.LAP_EGRAPH\n"
            "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for env in [{"LAP_TERM_BATCH": "3000"}, {"LAP_SYMCHECK": "search"}, {"LAP_TERM_BATCH": "100000", "LAP_SYMCHECK": "search"},
                {"LAP_GAL_FAST": "0", "LAP_SYMCHECK": "sort"}, {"LAP_GAL_FAST": "0", "LAP_TERM_BATCH": "3000"},
                {"LAP_LANCZOS_ASYNC": "0", "LAP_SORT_LONG": "1", "LAP_L0_SORTED": "1"}]:
        e = dict(os.environ, **env)
        r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=900, cwd=root)
        assert r.returncode == 0 and "ok" in r.stdout, (env, r.stderr[-3000:])


@pytest.mark.parametrize("env", [{"LAP_XT": "force", "LAP_XT_W": "64"},
                                 {"LAP_XT": "force", "LAP_XT_W": "2", "LAP_XT_NB": "3"},
                                 {"LAP_XT": "force", "LAP_XT_W": "1000", "LAP_XT_NB": "300"},
                                 {"LAP_XT": "force", "LAP_XT_W": "777"}],
                         ids=["w64", "w2-nb3", "w1000-nb300", "w777-odd-tiles"])
def test_column_tiled_spmv_per_entry(P, env):
    """The column-tiled (x-stationary) SpMV (xt.cu), forced on every level with
    a few hundred rows, with tiny tiles (many tiles, odd tile lengths), few or
    many row blocks: every entry of L_l x within the O-P2 bound of the oracle,
    every epilogue through the V-cycle and solve."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np, lapgen, oracle, paper_1705_06266_b200 as P\n"
            "def spmv_bound(rp, col, w, d, x):\n"
            "    rows = np.repeat(np.arange(len(d)), np.diff(rp)); s = np.zeros(len(d))\n"
            "    np.add.at(s, rows, np.abs(w) * np.abs(x[col])); return 1e-12 * (np.abs(d) * np.abs(x) + s)\n"
            "for g in [lapgen.rmat(12), lapgen.barabasi_albert(6000, 8), lapgen.random_connected(3000, 60000, 3)]:\n"
            "    h = P.Hierarchy(g); ho = oracle.Hierarchy(g)\n"
            "    rng = np.random.default_rng(0)\n"
            "    for l in range(ho.nlev):\n"
            "        o = ho.level(l); x = rng.standard_normal(o.n)\n"
            "        y = h.spmv(l, x); yo = oracle.spmv(o.n, o.row_ptr, o.col, o.w, o.d, x)\n"
            "        assert np.all(np.abs(y - yo) <= spmv_bound(o.row_ptr, o.col, o.w, o.d, x) + 1e-300), l\n"
            "    r = rng.standard_normal(g.n); r -= r.mean()\n"
            "    z = h.vcycle(r); zo = ho.vcycle(0, r)\n"
            "    assert np.abs(z - zo).max() <= 1e-9 * np.abs(zo).max()\n"
            "    b = lapgen.rhs(g.n); x, it, rr, rc = h.solve(b); xo, ito, _, _ = ho.solve(b)\n"
            "    assert rc == 0 and rr <= 1e-8 and abs(it - ito) <= 1, (it, ito, rr)\n"
            "    x2, it2, _, _ = h.solve(b); assert it2 == it and x2.tobytes() == x.tobytes()\n"
            "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


@pytest.mark.parametrize("mk", [lambda: lapgen.rmat(16), lambda: lapgen.grid2d(420, 420),
                                lambda: lapgen.star(30000)], ids=["rmat16", "grid420", "star30000"])
def test_pattern_only_level0(P, mk, monkeypatch):
    """Unit-weight level 0: the solve SpMV reads the pattern
    only (4 B per entry, padding slots recognised by their own-row index).
    1.0 * x_j = x_j, so the SpMV, the V-cycle and the whole solve are
    bit-identical to the weighted kernel (LAP_UNIT=0), the SpMV is within the
    O-P2 bound of the oracle, and the library books 4 B per stored entry."""
    g = mk()
    g = lapgen.Graph(g.n, g.row_ptr, g.col, np.ones(g.nnz))
    monkeypatch.setenv("LAP_UNIT", "0")
    hw = P.Hierarchy(g)
    monkeypatch.delenv("LAP_UNIT")
    hu = P.Hierarchy(g)
    x = np.random.default_rng(3).standard_normal(g.n)
    yu, yw = hu.spmv(0, x), hw.spmv(0, x)
    assert yu.tobytes() == yw.tobytes()
    lv = hu.level(0)
    ref = oracle.spmv(lv["n"], lv["row_ptr"], lv["col"], lv["w"], lv["d"], x)
    assert np.all(np.abs(yu - ref) <= spmv_bound(lv["row_ptr"], lv["col"], lv["w"], lv["d"], x))
    b = lapgen.rhs(g.n)
    xu, itu, rru, _ = hu.solve(b)
    xw, itw, rrw, _ = hw.solve(b)
    assert itu == itw and xu.tobytes() == xw.tobytes() and rru <= 1e-8
    _, bu, eu = hu.bench_op(0, 0, 2)
    _, bw, ew = hw.bench_op(0, 0, 2)
    nnz = lv["nnz"]
    if lv["n"] > 131072 or np.diff(lv["row_ptr"]).max() > 64:  # big enough for k_spmv (not the small-level kernels)
        assert bw - bu == 8 * nnz, (bw, bu, nnz)


@pytest.mark.parametrize("mk", [lambda: lapgen.star(30000), lambda: lapgen.rmat(16),
                                lambda: lapgen.barabasi_albert(60000, 8)], ids=["star30000", "rmat16", "ba60000"])
def test_solves_bitwise_reproducible_with_hub_rows(P, mk):
    """Rows of several 1024-entry chunks are finished by whichever warp arrives
    last; their dot-epilogue terms (PCG p.q, the E_CHEBZ z-sums, FCG's two
    dots, the block solve's per-column p.q) are summed in slot order by the
    last block (dot_fixup), so repeated solves on one hierarchy give the same
    bits -- V-cycle + PCG, K-cycle + FCG, and the block solve."""
    g = mk()
    b = lapgen.rhs(g.n, seed=4)
    for kw in [dict(), dict(use_graphs=0), dict(cycle=1)]:
        h = P.Hierarchy(g, **kw)
        xs = {h.solve(b)[0].tobytes() for _ in range(5)}
        assert len(xs) == 1, kw
        h.close()
    h = P.Hierarchy(g)
    B = np.stack([lapgen.rhs(g.n, seed=j) for j in range(3)])
    Xs = {h.solve_block(B)[0].tobytes() for _ in range(4)}
    assert len(Xs) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["0", "1"], ids=["row-order", "active-list"])
@pytest.mark.parametrize("mk", [SMALL[0], SMALL[2], SMALL[3], SMALL[4], SMALL[7], SMALL[10]],
                         ids=["cfg1", "grid3d12", "rmat12", "ba5000", "star40000", "dense6000"])
def test_vote_round_modes_bit_exact(P, mk, mode, monkeypatch):
    """Alg. 3's vote rounds in both execution orders: every row of
    the level each round (LAP_VOTE_LIST=0, the default below 10 entries per row)
    or only the rows still Undecided, from a list compacted after every round
    (LAP_VOTE_LIST=1, the default above) -- the aggregates, and so every coarse
    operator, equal the oracle's bit for bit either way."""
    monkeypatch.setenv("LAP_VOTE_LIST", mode)
    g = mk()
    h, ho = P.Hierarchy(g), oracle.Hierarchy(g)
    assert h.nlev == ho.nlev
    for l in range(ho.nlev):
        a, o = h.level(l), ho.level(l)
        assert a["kind"] == o.kind and (a["n"], a["nnz"]) == (o.n, o.nnz), l
        assert np.array_equal(a["col"], o.col) and a["w"].tobytes() == o.w.tobytes(), l
        if o.kind == oracle.AGG:
            assert np.array_equal(a["agg"], o.agg), l
