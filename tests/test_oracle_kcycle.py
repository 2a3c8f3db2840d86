"""Pins for the K-cycle + FCG oracle (
S:524-532).

The oracle's orc_kcoarse runs kcycle_inner FCG(1) iterations; these tests pin
it to what FCG is, independently of its recurrence: after one iteration x is
the L-energy minimiser on span{c1}, after two on span{c1, c2} (c1 = K b,
c2 = K (b - L x1)), both evaluated here by a direct Gram solve on a scipy
matrix built from the exported level.  Where no aggregation level lies below
the finest, the K-cycle IS the V-cycle (bit for bit) and outer FCG reproduces
PCG; the robustness direction of S:562 (K-cycle outer iterations <= V-cycle's
on P10000) is checked on the SPEC fixtures.
"""
import numpy as np
import pytest
import scipy.sparse as sp

import lapgen
import oracle


def _lmat(ld):
    """L_l = diag(d) - W from the exported level."""
    n = ld.n
    W = sp.csr_matrix((ld.w, ld.col, ld.row_ptr), shape=(n, n))
    return sp.diags(ld.d) - W


def _agg_levels_below_finest(h):
    return [l for l, L in enumerate(h.levels()) if l > 0 and L.kind == oracle.AGG]


FIXTURES = {
    "grid2d_64": lambda: lapgen.grid2d(64, 64),
    "path_10000": lambda: lapgen.path(10000),
    "grid3d_16": lambda: lapgen.grid3d(16),
    "rmat12": lambda: lapgen.rmat(12),
    "ba3000": lambda: lapgen.barabasi_albert(3000, 6),
}


@pytest.mark.parametrize("name", ["grid2d_64", "grid3d_16", "ba3000", "rmat12"])
@pytest.mark.parametrize("inner", [1, 2])
def test_kcoarse_is_energy_minimiser(name, inner):
    """FCG(1) from x = 0: x_1 = argmin_{x in span c1} ||x* - x||_L with
    c1 = K_l b; x_2 = argmin over span{c1, c2}, c2 = K_l (b - L x_1) --
    the Galerkin conditions c_i.(b - L x) = 0 solved as a Gram system."""
    g = FIXTURES[name]()
    h = oracle.Hierarchy(g, cycle=1, kcycle_inner=inner)
    levels = _agg_levels_below_finest(h)
    assert levels, "fixture must have an aggregation level below the finest"
    for l in levels:
        ld = h.level(l)
        L = _lmat(ld)
        b = np.random.default_rng(l).standard_normal(ld.n)
        b -= b.mean()
        x = h.kcoarse(l, b)
        c1 = h.kcycle(l, b)
        x1 = (c1 @ b) / (c1 @ (L @ c1)) * c1
        if inner == 1:
            want = x1
        else:
            c2 = h.kcycle(l, b - L @ x1)
            C = np.stack([c1, c2], axis=1)
            G = C.T @ (L @ C)
            want = C @ np.linalg.solve(G, C.T @ b)
        assert np.abs(x - want).max() <= 1e-9 * np.abs(want).max(), (l, np.abs(x - want).max())


def test_kcoarse_degenerate_cases():
    """Zero right-hand side -> x = 0 (the p.q = 0 guard, DESIGN reading
    R-K2); homogeneity K(2b) = 2 K(b) holds exactly (scaling by 2 is exact
    and FCG's coefficients are scale-free)."""
    g = lapgen.grid2d(64, 64)
    h = oracle.Hierarchy(g, cycle=1)
    l = _agg_levels_below_finest(h)[0]
    n = h.level(l).n
    assert np.all(h.kcoarse(l, np.zeros(n)) == 0.0)
    b = np.random.default_rng(3).standard_normal(n)
    b -= b.mean()
    assert (h.kcoarse(l, 2.0 * b) == 2.0 * h.kcoarse(l, b)).all()
    assert (h.kcycle(0, 2.0 * np.resize(b, h.level(0).n)) == 2.0 * h.kcycle(0, np.resize(b, h.level(0).n))).all()


def _no_inner_agg_graphs():
    """Hierarchies whose aggregation levels are all at the finest level."""
    out = []
    for g in [lapgen.grid2d(12, 12), lapgen.random_connected(120, 200, 1), lapgen.complete(30),
              lapgen.star(200), lapgen.barabasi_albert(150, 3)]:
        h = oracle.Hierarchy(g, cycle=1)
        if not _agg_levels_below_finest(h):
            out.append((g, h))
    return out


def test_kcycle_is_vcycle_without_inner_aggregation():
    """with no aggregation level below the finest the K-cycle is the
    V-cycle -- the same arithmetic, bit for bit; outer FCG with a fixed SPD
    preconditioner is PCG (equal iterations, solutions within rounding)."""
    cases = _no_inner_agg_graphs()
    assert len(cases) >= 2
    for g, hk in cases:
        hv = oracle.Hierarchy(g)
        r = np.random.default_rng(0).standard_normal(g.n)
        r -= r.mean()
        assert (hk.kcycle(0, r) == hv.vcycle(0, r)).all()
        b = lapgen.rhs(g.n, seed=2)
        xk, itk, rrk, rck = hk.solve(b)
        xv, itv, rrv, rcv = hv.solve(b)
        assert rck == 0 and rcv == 0 and itk == itv, (itk, itv)
        assert np.abs(xk - xv).max() <= 1e-9 * np.abs(xv).max()


@pytest.mark.parametrize("name", list(FIXTURES))
def test_kcycle_solve_converges_and_is_no_worse(name):
    """Convergence to 1e-8 (true residual) on the SPEC fixtures and the
    robustness direction of S:562: K-cycle outer iterations <= V-cycle's;
    solutions agree to the tolerance."""
    g = FIXTURES[name]()
    b = lapgen.rhs(g.n, seed=1)
    xv, itv, rrv, rcv = oracle.Hierarchy(g).solve(b)
    xk, itk, rrk, rck = oracle.Hierarchy(g, cycle=1).solve(b)
    assert rck == 0 and rrk <= 1e-8
    assert itk <= itv, (itk, itv)
    assert np.abs(xk - xv).max() <= 1e-4 * np.abs(xv).max()
    # the K-cycle's answer solves the caller's system (caller numbering)
    A = sp.csr_matrix((g.w, g.col, g.row_ptr), shape=(g.n, g.n))
    Lg = sp.diags(np.asarray(A.sum(axis=1)).ravel()) - A
    bb = b - b.mean()
    assert np.linalg.norm(bb - Lg @ xk) <= 1.01e-8 * np.linalg.norm(bb)


def test_kcycle_path_graph_much_better():
    """High-diameter graph ("iterate recombination ... helps
    improve performance on high diameter graphs"): on P10000 the K-cycle
    needs at most half the V-cycle's outer iterations."""
    g = lapgen.path(10000)
    b = lapgen.rhs(g.n, seed=4)
    _, itv, _, _ = oracle.Hierarchy(g).solve(b)
    _, itk, _, rc = oracle.Hierarchy(g, cycle=1).solve(b)
    assert rc == 0 and 2 * itk <= itv, (itk, itv)
