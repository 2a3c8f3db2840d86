"""Many right-hand sides at once.

The oracle for column j is orc_solve on column j alone (the definition: k
independent solves).  The block path runs the k PCG solves in lockstep with
SpMM passes and freezes converged columns, so each column must agree with
its own oracle solve exactly as lap_solve does: true relative residual <=
1e-8, iterations within +-1, solution within 1e-6 relative.
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
    "rmat12": lambda: lapgen.rmat(12),
    "ba3000": lambda: lapgen.barabasi_albert(3000, 6),
    "grid3d_16": lambda: lapgen.grid3d(16),
    "star20000": lambda: lapgen.star(20000),
    "rand2000": lambda: lapgen.random_connected(2000, 6000, 3),
}


def _rhs(n, k, seed=0):
    return np.stack([lapgen.rhs(n, seed=seed + j) for j in range(k)])


@pytest.mark.parametrize("gname", list(GRAPHS))
@pytest.mark.parametrize("k", [1, 3, 4, 8])
def test_block_matches_per_column_oracle(P, gname, k):
    g = GRAPHS[gname]()
    B = _rhs(g.n, k, seed=10)
    X, it, rr, rc = P.Hierarchy(g).solve_block(B)
    assert rc == 0
    ho = oracle.Hierarchy(g)
    for j in range(k):
        xo, ito, _, rco = ho.solve(B[j])
        assert rco == 0
        assert rr[j] <= 1e-8, (j, rr[j])
        assert abs(int(it[j]) - ito) <= 1, (j, it[j], ito)
        assert np.abs(X[j] - xo).max() <= 1e-6 * np.abs(xo).max(), j
        assert abs(X[j].mean()) <= 1e-10 * np.abs(X[j]).max()


@pytest.mark.parametrize("gname", ["grid2d_64", "rmat12", "star20000", "ba3000"])
@pytest.mark.parametrize("k", [12, 16, 25, 32])
def test_wide_block_matches_per_column_oracle(P, gname, k, monkeypatch):
    """k = 9..32 columns on the lane-per-column SpMM (K = 16 / 32, forced by
    LAP_BLOCK_WIDE=1) and the per-element vector kernels; each column is
    still its own O-S8 solve."""
    monkeypatch.setenv("LAP_BLOCK_WIDE", "1")
    g = GRAPHS[gname]()
    B = _rhs(g.n, k, seed=40)
    X, it, rr, rc = P.Hierarchy(g).solve_block(B)
    assert rc == 0
    ho = oracle.Hierarchy(g)
    for j in range(k):
        xo, ito, _, rco = ho.solve(B[j])
        assert rco == 0
        assert rr[j] <= 1e-8, (j, rr[j])
        assert abs(int(it[j]) - ito) <= 1, (j, it[j], ito)
        assert np.abs(X[j] - xo).max() <= 1e-6 * np.abs(xo).max(), j


@pytest.mark.parametrize("gname", ["grid2d_64", "grid3d_16", "rmat12", "rand2000"])
@pytest.mark.parametrize("k", [9, 16, 21, 32])
def test_grouped_block_matches_per_column_oracle(P, gname, k):
    """Default routing past 8 columns: groups of <= 8 columns on the
    thread-per-row SpMM one after the other (k <= 16, or any k on a level 0
    with < 10 entries per row), else K = 32; each column is its own O-S8
    solve whichever way, and the grouped columns equal the same columns
    solved alone as a block (bitwise: the same K = 8 program)."""
    g = GRAPHS[gname]()
    B = _rhs(g.n, k, seed=70)
    h = P.Hierarchy(g)
    X, it, rr, rc = h.solve_block(B)
    assert rc == 0
    ho = oracle.Hierarchy(g)
    for j in range(k):
        xo, ito, _, rco = ho.solve(B[j])
        assert rco == 0
        assert rr[j] <= 1e-8, (j, rr[j])
        assert abs(int(it[j]) - ito) <= 1, (j, it[j], ito)
        assert np.abs(X[j] - xo).max() <= 1e-6 * np.abs(xo).max(), j
    if k <= 16 or 10 * g.n > len(g.col):
        c0 = 8 * ((k - 1) // 8)
        Xg, itg, _, _ = h.solve_block(B[c0:])
        assert np.array_equal(itg, it[c0:])
        assert Xg.tobytes() == X[c0:].tobytes()


def test_wide_block_agrees_with_narrow(P, monkeypatch):
    """The first 8 columns of a 32-column block solve on the lane-per-column
    SpMM agree with the same 8 columns solved at K = 8 (same iterations, x to
    1e-10 relative)."""
    monkeypatch.setenv("LAP_BLOCK_WIDE", "1")
    g = lapgen.rmat(12)
    B = _rhs(g.n, 32, seed=5)
    h = P.Hierarchy(g)
    X32, it32, _, rc32 = h.solve_block(B)
    X8, it8, _, rc8 = h.solve_block(B[:8])
    assert rc32 == 0 and rc8 == 0
    assert np.array_equal(it32[:8], it8)
    assert np.abs(X32[:8] - X8).max() <= 1e-10 * np.abs(X8).max()


def test_block_columns_do_not_interact(P):
    """Identical columns give bit-identical answers and iteration counts,
    whatever the other columns hold (zero, constant, different rhs); a zero
    or constant column returns x = 0 after 0 iterations."""
    g = lapgen.grid2d(60, 50)
    b = lapgen.rhs(g.n, seed=3)
    B = np.stack([b, np.zeros(g.n), b, lapgen.rhs(g.n, seed=4), np.full(g.n, 2.5), b])
    X, it, rr, rc = P.Hierarchy(g).solve_block(B)
    assert rc == 0
    assert X[0].tobytes() == X[2].tobytes() == X[5].tobytes()
    assert it[0] == it[2] == it[5]
    for j in (1, 4):
        assert it[j] == 0 and rr[j] == 0.0 and np.all(X[j] == 0.0)
    x1, it1, rr1, _ = P.Hierarchy(g).solve(b)
    assert abs(int(it[0]) - it1) <= 1 and np.abs(X[0] - x1).max() <= 1e-6 * np.abs(x1).max()


def test_block_device_buffers(P):
    g = lapgen.rmat(12)
    B = _rhs(g.n, 4, seed=1)
    Bt = torch.from_numpy(B).cuda()
    X, it, rr, rc = P.Hierarchy(g).solve_block(Bt)
    assert rc == 0 and X.is_cuda and np.all(rr <= 1e-8)
    Xh, ith, _, _ = P.Hierarchy(g).solve_block(B)
    assert np.array_equal(it, ith)
    assert np.abs(X.cpu().numpy() - Xh).max() <= 1e-12 * np.abs(Xh).max()


def test_block_invalid(P):
    g = lapgen.grid2d(16, 16)
    h = P.Hierarchy(g)
    with pytest.raises(P.LapError):
        h.solve_block(np.zeros((33, g.n)))


def test_block_max_iters_and_tolerance(P):
    """max_iters reached -> LAP_ENOCONV with every column's iteration count at
    the cap and its residual above tol (as lap_solve reports it); a looser
    tolerance stops each column at the oracle's iteration count for it."""
    g = lapgen.grid2d(64, 64)
    B = _rhs(g.n, 3, seed=21)
    X, it, rr, rc = P.Hierarchy(g, max_iters=4).solve_block(B)
    assert rc == P.LAP_ENOCONV and np.all(it == 4) and np.all(rr > 1e-8)
    ho = oracle.Hierarchy(g)
    X, it, rr, rc = P.Hierarchy(g).solve_block(B, tol=1e-5)
    assert rc == 0 and np.all(rr <= 1e-5)
    for j in range(3):
        _, ito, _, _ = ho.solve(B[j], tol=1e-5)
        assert abs(int(it[j]) - ito) <= 1, (j, it[j], ito)
