"""K-cycle + FCG on the GPU against the oracle.

The hierarchy is bit-identical to the oracle's (test_gpu_parity.py), so the
K-cycle differs from orc_kcycle only in the summation order of its FCG dot
products (fixed two-pass reductions on the device, left-to-right loops in the
oracle): outputs agree to 1e-9 relative (the coefficients alpha, beta are
ratios of well-conditioned dots; the propagated relative error is ~1e-13 on
these fixtures).  Solves reach the true 1e-8 residual with outer iterations
within +-1 of the oracle's FCG.
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


GRAPHS = {
    "grid2d_64": lambda: lapgen.grid2d(64, 64),
    "path_10000": lambda: lapgen.path(10000),
    "grid3d_16": lambda: lapgen.grid3d(16),
    "rmat12": lambda: lapgen.rmat(12),
    "ba3000": lambda: lapgen.barabasi_albert(3000, 6),
    "rand2000": lambda: lapgen.random_connected(2000, 6000, 3),
    "star20000": lambda: lapgen.star(20000),
    "grid2d_300x200": lambda: lapgen.grid2d(300, 200),
}


def _close(a, b, rel):
    return np.abs(a - b).max() <= rel * max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("gname", list(GRAPHS))
def test_kcycle_matches_oracle(P, gname):
    g = GRAPHS[gname]()
    h = P.Hierarchy(g, cycle=1)
    ho = oracle.Hierarchy(g, cycle=1)
    r = np.random.default_rng(7).standard_normal(g.n)
    r -= r.mean()
    z = h.kcycle(0, r)
    zo = ho.kcycle(0, r)
    assert _close(z, zo, 1e-9), np.abs(z - zo).max() / np.abs(zo).max()
    # every aggregation level below the finest: the inner FCG iterations alone
    for l in range(1, ho.nlev):
        ld = ho.level(l)
        if ld.kind != oracle.AGG:
            continue
        b = np.random.default_rng(l).standard_normal(ld.n)
        b -= b.mean()
        x = h.kcycle(l, b, with_fcg=True)
        xo = ho.kcoarse(l, b)
        assert _close(x, xo, 1e-9), (l, np.abs(x - xo).max() / np.abs(xo).max())


@pytest.mark.parametrize("gname", list(GRAPHS))
def test_kcycle_solve_matches_oracle(P, gname):
    g = GRAPHS[gname]()
    b = lapgen.rhs(g.n, seed=3)
    x, it, rr, rc = P.Hierarchy(g, cycle=1).solve(b)
    xo, ito, rro, rco = oracle.Hierarchy(g, cycle=1).solve(b)
    assert rc == 0 and rco == 0
    assert rr <= 1e-8, rr
    assert abs(it - ito) <= 1, (it, ito)
    assert _close(x, xo, 1e-6)


def test_kcycle_eager_equals_graph(P):
    """use_graphs = 0 (host-driven launches) runs the same kernels as the
    resident FCG graph: identical iterations and bitwise-identical x."""
    g = lapgen.grid2d(300, 200)
    b = lapgen.rhs(g.n, seed=1)
    x1, it1, _, _ = P.Hierarchy(g, cycle=1).solve(b)
    x2, it2, _, _ = P.Hierarchy(g, cycle=1, use_graphs=0).solve(b)
    assert it1 == it2 and x1.tobytes() == x2.tobytes()


def test_kcycle_work_and_robustness(P):
    """S:562 #8: on a hierarchy with >= 4 aggregation levels the K-cycle does
    more SpMV work per outer iteration than the V-cycle, and needs no more
    outer iterations (P10000 and a 2D grid)."""
    for g in [lapgen.path(10000), lapgen.grid2d(300, 200)]:
        b = lapgen.rhs(g.n, seed=2)
        hv, hk = P.Hierarchy(g), P.Hierarchy(g, cycle=1)
        ho = oracle.Hierarchy(g)
        nagg = sum(1 for L in ho.levels() if L.kind == oracle.AGG)
        _, itv, _, _ = hv.solve(b)
        sv = hv.stats()
        _, itk, _, _ = hk.solve(b)
        sk = hk.stats()
        assert itk <= itv, (itk, itv)
        if nagg >= 4:
            assert sk["spmv_edges"] / itk > sv["spmv_edges"] / itv


def test_kcycle_rejected_when_sharded(P):
    comm = P.Comm(2, 2)
    with pytest.raises(P.LapError):
        P.Hierarchy(lapgen.grid2d(32, 32), comm=comm, cycle=1)
    comm.close()


def test_kcycle_launched_path_matches_oracle(P):
    """LAP_KTAIL=0: every level of the K-cycle as launched kernels (no
    single-CTA tail program) -- same oracle agreement (subprocess: the switch
    is read once per process)."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np, lapgen, oracle, paper_1705_06266_b200 as P\n"
            "for g in [lapgen.grid2d(64, 64), lapgen.rmat(12), lapgen.grid2d(300, 200)]:\n"
            "    h = P.Hierarchy(g, cycle=1); ho = oracle.Hierarchy(g, cycle=1)\n"
            "    r = np.random.default_rng(1).standard_normal(g.n); r -= r.mean()\n"
            "    z = h.kcycle(0, r); zo = ho.kcycle(0, r)\n"
            "    assert np.abs(z - zo).max() <= 1e-9 * np.abs(zo).max()\n"
            "    b = lapgen.rhs(g.n, seed=4); x, it, rr, rc = h.solve(b); xo, ito, _, _ = ho.solve(b)\n"
            "    assert rc == 0 and rr <= 1e-8 and abs(it - ito) <= 1, (it, ito, rr)\n"
            "print('ok')\n")
    e = dict(os.environ, LAP_KTAIL="0")
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_kcycle_tail_program_is_one_launch(P):
    """With the single-CTA tail program the whole coarse K-cycle of a small
    graph is one launch per outer iteration (cfg 1: every level <= 4096 rows)."""
    g = lapgen.grid2d(64, 64)
    b = lapgen.rhs(g.n, seed=1)
    h = P.Hierarchy(g, cycle=1)
    _, it, rr, rc = h.solve(b)
    st = h.stats()
    assert rc == 0 and rr <= 1e-8
    # per outer iteration: level-0 cycle (elimination: restrict + tail + prolong) + FCG vector ops
    assert st["kernel_launches"] <= 20 * (it + 2), (st["kernel_launches"], it)


@pytest.mark.parametrize("kw", [dict(kcycle_inner=1), dict(kcycle_inner=3), dict(elim_enable=0),
                                dict(cheby_degree=3)], ids=["inner1", "inner3", "no-elim", "cheb3"])
def test_kcycle_parameters_match_oracle(P, kw):
    """The K-cycle under other parameter choices (inner FCG iterations,
    no elimination levels, degree-3 smoothing) against the oracle with the
    same parameters."""
    for g in [lapgen.grid2d(120, 90), lapgen.rmat(12)]:
        h = P.Hierarchy(g, cycle=1, **kw)
        ho = oracle.Hierarchy(g, cycle=1, **kw)
        r = np.random.default_rng(3).standard_normal(g.n)
        r -= r.mean()
        z, zo = h.kcycle(0, r), ho.kcycle(0, r)
        assert _close(z, zo, 1e-9), np.abs(z - zo).max() / np.abs(zo).max()
        b = lapgen.rhs(g.n, seed=6)
        x, it, rr, rc = h.solve(b)
        xo, ito, _, rco = ho.solve(b)
        assert rc == 0 and rco == 0 and rr <= 1e-8 and abs(it - ito) <= 1, (it, ito, rr)
