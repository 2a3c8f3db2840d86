"""Pins for the smoother, lambda-hat, coarsest solve, V-cycle and PCG
(O-P9..O-P13) and hierarchy invariants (O-S9)."""
import numpy as np
import pytest

import lapgen
import oracle
from _dense import cheb_T, csr_to_dense_L, dense_L


def _d(g):
    return oracle.row_sums(g.n, g.row_ptr, g.w)


@pytest.mark.parametrize("K", [1, 2, 3])
@pytest.mark.parametrize("k", [1, 5, 16, 31])
def test_chebyshev_error_polynomial_on_cycle(K, k):
    """C_n (D = 2I), b = 0, x0 = cos(2 pi k i / n): x_K = T_K((theta - t)/delta)/T_K(sigma) x0
    with t = 1 - cos(2 pi k/n) the D^-1 L eigenvalue (O-S6, O-P9)."""
    n = 64
    g = lapgen.cycle(n)
    lam = 2.0
    x0 = np.cos(2 * np.pi * k * np.arange(n) / n)
    x = oracle.chebyshev(n, g.row_ptr, g.col, g.w, _d(g), lam, np.zeros(n), x0, degree=K)
    a, b = 0.3 * lam, 1.1 * lam
    theta, delta = (a + b) / 2, (b - a) / 2
    t = 1 - np.cos(2 * np.pi * k / n)
    fac = cheb_T(K, (theta - t) / delta) / cheb_T(K, theta / delta)
    assert np.abs(x - fac * x0).max() <= 4e-14  # K steps of O(eps) rounding


def test_degree1_chebyshev_is_richardson():
    """Degree 1 = one Jacobi-Richardson step x + D^-1 (b - L x)/theta."""
    for seed in range(10):
        g = lapgen.random_connected(50, 60, seed)
        d = _d(g)
        rng = np.random.default_rng(seed)
        b, x0 = rng.standard_normal(g.n), rng.standard_normal(g.n)
        lam = 1.7
        x = oracle.chebyshev(g.n, g.row_ptr, g.col, g.w, d, lam, b, x0, degree=1)
        want = x0 + (b - dense_L(g) @ x0) / d / (0.7 * lam)
        assert np.allclose(x, want, atol=1e-13)


def test_lambda_hat_pins():
    # P3: D^-1 L spectrum {0, 1, 2}; Lanczos is exact for n <= steps  (O-P10)
    g = lapgen.path(3)
    lam, _, _ = oracle.lanczos(3, g.row_ptr, g.col, g.w, _d(g))
    assert abs(lam - 2.0) <= 1e-13
    # K_n: D^-1 L = (n I - J)/(n-1) -> lambda_max = n/(n-1)
    for n in [4, 7, 12]:
        g = lapgen.complete(n)
        lam, _, _ = oracle.lanczos(n, g.row_ptr, g.col, g.w, _d(g))
        assert abs(lam - n / (n - 1)) <= 1e-12
    # random graphs n <= 200: 0.9 lambda_max <= lam_hat <= lambda_max (S:640 acceptance 7)
    for seed in range(8):
        g = lapgen.random_connected(120 + 10 * seed, 150, seed)
        d = _d(g)
        lam, _, _ = oracle.lanczos(g.n, g.row_ptr, g.col, g.w, d, seed=seed)
        ev = np.linalg.eigvalsh(dense_L(g) / np.sqrt(np.outer(d, d)))
        assert 0.9 * ev[-1] <= lam <= ev[-1] * (1 + 1e-12)
    # bipartite grid: lambda_max(D^-1 L) = 2
    g = lapgen.grid2d(20, 20)
    lam, _, _ = oracle.lanczos(g.n, g.row_ptr, g.col, g.w, _d(g))
    assert 1.9 <= lam <= 2.0 + 1e-12


def test_tridiag_bisection_matches_eigvalsh():
    rng = np.random.default_rng(0)
    for k in range(1, 11):
        a = rng.standard_normal(k)
        b = rng.uniform(0.01, 1, max(k - 1, 0))
        T = np.diag(a) + np.diag(b, 1) + np.diag(b, -1)
        assert abs(oracle.tridiag_max_eig(a, b) - np.linalg.eigvalsh(T)[-1]) <= 1e-13 * max(1, abs(a).max())


def test_coarse_pinv_matches_numpy():
    for seed in range(6):
        g = lapgen.random_connected(5 + 20 * seed, 10, seed)
        d = _d(g)
        rc, Pi = oracle.coarse_pinv(g.n, g.row_ptr, g.col, g.w, d)
        assert rc == 0
        assert np.allclose(Pi, np.linalg.pinv(dense_L(g)), atol=1e-10)
    rc, Pi = oracle.coarse_pinv(1, np.array([0, 0]), np.zeros(0, np.int32), np.zeros(0), np.zeros(1))
    assert rc == 0 and Pi.tolist() == [[0.0]]


def _vcycle_M(h):
    n = h.level(0).n
    return np.column_stack([h.vcycle(0, e) for e in np.eye(n)])


@pytest.mark.parametrize("g", [lapgen.grid2d(12, 12), lapgen.random_connected(150, 300, 3),
                               lapgen.rmat(8), lapgen.barabasi_albert(300, 4)], ids=lambda g: g.name)
def test_vcycle_symmetric_and_preserves_nullspace(g):
    h = oracle.Hierarchy(g, coarse_nnz=60)
    M = _vcycle_M(h)
    kinds = [h.level(l).kind for l in range(h.nlev)]
    assert kinds[-1] == oracle.COARSEST and len(kinds) >= 3
    assert np.abs(M - M.T).max() <= 1e-12 * np.abs(M).max()              # S:535, O-P12
    L0 = h.level(0)
    L = csr_to_dense_L(L0.n, L0.row_ptr, L0.col, L0.w, L0.d)
    # M is positive definite on 1-perp (a valid CG preconditioner)
    Pj = np.eye(L0.n) - 1.0 / L0.n
    ev = np.linalg.eigvalsh(Pj @ M @ Pj)
    assert ev[1] > 0
    # energy does not increase: || I - M L ||_L <= 1 on 1-perp
    E = np.eye(L0.n) - M @ L
    rng = np.random.default_rng(0)
    for _ in range(10):
        e = Pj @ rng.standard_normal(L0.n)
        e2 = E @ e
        assert e2 @ L @ e2 <= e @ L @ e * (1 + 1e-12)


def test_elimination_only_hierarchy_is_exact():
    """STAR6: eliminate the 5 leaves, coarsest 1x1 -> one V-cycle is exact."""
    g = lapgen.star(5)
    h = oracle.Hierarchy(g, coarse_nnz=1)
    assert [h.level(l).kind for l in range(h.nlev)] == [oracle.ELIM, oracle.COARSEST]
    assert h.level(1).n == 1
    b = np.random.default_rng(0).standard_normal(6)
    b -= b.mean()
    x, it, rr, rc = h.solve(b)
    assert rc == 0 and it == 1 and rr <= 1e-14


def test_pcg_path_closed_form():
    """Unit resistor chain, b = e_0 - e_{n-1}: x_i = (n-1)/2 - i (O-P13)."""
    n = 200
    g = lapgen.path(n)
    h = oracle.Hierarchy(g)
    b = np.zeros(n)
    b[0], b[-1] = 1.0, -1.0
    x, it, rr, rc = h.solve(b)
    assert rc == 0 and rr <= 1e-8
    assert np.abs(x - ((n - 1) / 2 - np.arange(n))).max() <= 1e-6


def test_pcg_grid_eigenvector_closed_form():
    """cfg-1 grid, b = v_jk -> x = v_jk / lambda_jk (O-P13)."""
    g = lapgen.config(1)
    h = oracle.Hierarchy(g)
    xs = np.arange(64)
    j, k = 3, 5
    v = np.outer(np.cos(np.pi * k * (xs + 0.5) / 64), np.cos(np.pi * j * (xs + 0.5) / 64)).ravel()
    lam = 4 * np.sin(np.pi * j / 128) ** 2 + 4 * np.sin(np.pi * k / 128) ** 2
    x, it, rr, rc = h.solve(v)
    assert rc == 0 and rr <= 1e-8
    assert np.abs(x - v / lam).max() <= 1e-6 * np.abs(v / lam).max()


@pytest.mark.parametrize("seed", range(8))
def test_pcg_matches_dense_pinv(seed):
    g = lapgen.random_connected(100 + 40 * seed, 200, seed)
    h = oracle.Hierarchy(g, coarse_nnz=100, seed=seed)
    b = np.random.default_rng(seed).standard_normal(g.n)
    x, it, rr, rc = h.solve(b)
    assert rc == 0 and rr <= 1e-8
    xs = np.linalg.pinv(dense_L(g)) @ (b - b.mean())
    assert np.abs(x - xs).max() <= 1e-6 * np.abs(xs).max()
    assert abs(x.mean()) <= 1e-12


def test_zero_rhs_and_single_vertex():
    g = lapgen.grid2d(8, 8)
    h = oracle.Hierarchy(g)
    x, it, rr, rc = h.solve(np.ones(g.n) * 3.0)  # constant projects to zero
    assert it == 0 and np.all(x == 0) and rc == 0
    g1 = lapgen.Graph(1, np.array([0, 0]), np.zeros(0, np.int32), np.zeros(0))
    h1 = oracle.Hierarchy(g1)
    assert h1.nlev == 1 and h1.level(0).kind == oracle.COARSEST
    x, it, rr, rc = h1.solve(np.array([2.0]))
    assert it == 0 and x.tolist() == [0.0]


@pytest.mark.parametrize("k", [1])
def test_hierarchy_invariants_cfg(k):
    g = lapgen.config(k)
    h = oracle.Hierarchy(g)
    levels = h.levels()
    assert len(levels) <= 40 and levels[-1].kind == oracle.COARSEST
    assert levels[-1].n + levels[-1].nnz <= 1000
    prev = None
    for l, L in enumerate(levels):
        # Laplacian closure at every level
        rows = np.repeat(np.arange(L.n), np.diff(L.row_ptr))
        assert np.all(L.w > 0) and np.all(L.col != rows)
        Ld = csr_to_dense_L(L.n, L.row_ptr, L.col, L.w, L.d) if L.n <= 5000 else None
        if Ld is not None:
            assert np.array_equal(Ld, Ld.T)
            assert np.abs(Ld.sum(1)).max() <= 1e-12 * L.d.max()
        if L.kind == oracle.ELIM:
            assert prev != oracle.ELIM and 20 * L.nF > L.n                  # O-R20, O-R21
            assert levels[l + 1].n == L.n - L.nF
        if L.kind == oracle.AGG:
            assert levels[l + 1].n == L.m < L.n and 1.0 < L.lam <= 2.0 + 1e-12
        prev = L.kind
    b = lapgen.rhs(g.n)
    x, it, rr, rc = h.solve(b)
    assert rc == 0 and rr <= 1e-8 and it <= 60
    # operator complexity (S acceptance 9)
    oc = sum(L.n + L.nnz for L in levels) / (levels[0].n + levels[0].nnz)
    assert oc <= 3.0


def test_random_order_off_gives_same_solution():
    g = lapgen.grid2d(24, 24)
    b = lapgen.rhs(g.n)
    x1, it1, _, _ = oracle.Hierarchy(g).solve(b)
    x0, it0, _, _ = oracle.Hierarchy(g, random_order=0).solve(b)
    assert np.abs(x1 - x0).max() <= 1e-6 * np.abs(x0).max()
