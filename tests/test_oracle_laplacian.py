"""Pins for validation, the Laplacian/diagonal and the fp64 SpMV (O-P1, O-P2)."""
import json
import os

import numpy as np
import pytest

import lapgen
import oracle
from _dense import dense_L

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_p3_laplacian_and_ones():
    g = lapgen.path(3)
    d = oracle.row_sums(g.n, g.row_ptr, g.w)
    L = np.diag(d)
    for i in range(3):
        for k in range(g.row_ptr[i], g.row_ptr[i + 1]):
            L[i, g.col[k]] = -g.w[k]
    assert L.tolist() == GOLD["laplacian_p3"]["L"]
    y = oracle.spmv(3, g.row_ptr, g.col, g.w, d, np.ones(3))
    assert y.tolist() == GOLD["spmv_p3_ones"]["y"]


@pytest.mark.parametrize("seed", range(10))
def test_spmv_matches_dense_matvec(seed):
    g = lapgen.random_connected(40 + seed, 60, seed)
    d = oracle.row_sums(g.n, g.row_ptr, g.w)
    x = np.random.default_rng(seed).standard_normal(g.n)
    y = oracle.spmv(g.n, g.row_ptr, g.col, g.w, d, x)
    Ld = dense_L(g)
    assert np.allclose(y, Ld @ x, rtol=0, atol=1e-12 * np.abs(Ld).sum(axis=1).max())
    # diagonal is the row sum to within 1/2 ulp (CanonSum, O-R23)
    assert np.all(np.abs(d - Ld.diagonal()) <= np.spacing(d) * 2)
    # x^T L x = sum_{i<j} w_ij (x_i - x_j)^2 (O-P1)
    rows = np.repeat(np.arange(g.n), np.diff(g.row_ptr))
    q = 0.5 * np.sum(g.w * (x[rows] - x[g.col]) ** 2)
    assert abs(x @ y - q) <= 1e-12 * q


def test_unit_weight_L_times_ones_is_bitwise_zero():
    for g in [lapgen.grid2d(16, 16), lapgen.star(9), lapgen.complete(7), lapgen.random_connected(50, 80, 3, weighted=False)]:
        d = oracle.row_sums(g.n, g.row_ptr, g.w)
        assert np.all(oracle.spmv(g.n, g.row_ptr, g.col, g.w, d, np.ones(g.n)) == 0.0)


def test_grid_closed_form_eigenvectors():
    """On the 64x64 unit grid, v_jk(x,y) = cos(pi j (x+1/2)/64) cos(pi k (y+1/2)/64)
    satisfies L v = (4 sin^2(pi j/128) + 4 sin^2(pi k/128)) v  (O-P2)."""
    g = lapgen.grid2d(64, 64)
    d = oracle.row_sums(g.n, g.row_ptr, g.w)
    xs = np.arange(64)
    for j, k in [(0, 1), (1, 0), (3, 7), (63, 63), (20, 41)]:
        v = np.outer(np.cos(np.pi * k * (xs + 0.5) / 64), np.cos(np.pi * j * (xs + 0.5) / 64)).ravel()
        lam = 4 * np.sin(np.pi * j / 128) ** 2 + 4 * np.sin(np.pi * k / 128) ** 2
        y = oracle.spmv(g.n, g.row_ptr, g.col, g.w, d, v)
        assert np.abs(y - lam * v).max() <= 1e-13


def _mk(n, rp, col, w):
    return lapgen.Graph(n, np.array(rp, dtype=np.int64), np.array(col, dtype=np.int32), np.array(w, dtype=np.float64))


def test_validate_rejects_bad_graphs():
    ok = lapgen.path(3)
    assert oracle.validate(ok) == oracle.ORC_OK
    assert oracle.validate(_mk(1, [0, 0], [], [])) == oracle.ORC_OK             # n = 1
    assert oracle.validate(_mk(2, [0, 1, 1], [1], [1.0])) == oracle.ORC_EGRAPH  # asymmetric pattern
    assert oracle.validate(_mk(2, [0, 1, 2], [1, 0], [1.0, 2.0])) == oracle.ORC_EGRAPH  # asymmetric w
    assert oracle.validate(_mk(2, [0, 1, 2], [1, 0], [-1.0, -1.0])) == oracle.ORC_EGRAPH  # w <= 0
    assert oracle.validate(_mk(2, [0, 1, 2], [1, 0], [np.nan, np.nan])) == oracle.ORC_EGRAPH
    assert oracle.validate(_mk(2, [0, 2, 3], [0, 1, 0], [1.0, 1.0, 1.0])) == oracle.ORC_EGRAPH  # self loop
    assert oracle.validate(_mk(3, [0, 2, 3, 4], [2, 1, 0, 0], [1.0] * 4)) == oracle.ORC_EGRAPH  # unsorted
    two = lapgen.csr_from_edges(4, [0, 2], [1, 3])
    assert oracle.validate(two) == oracle.ORC_EDISCONNECTED


def test_graph_generators_are_valid_laplacians():
    for g in [lapgen.config(1), lapgen.grid3d(8), lapgen.rmat(10), lapgen.barabasi_albert(2000, 8)]:
        assert oracle.validate(g) == oracle.ORC_OK, g.name


def test_relabel_hand_example():
    """O-S1: level 0 = Pi L Pi^T with perm[old] = new.  Path
    0 -1.5- 1 -2.5- 2 under perm = [2, 0, 1]: new vertex 0 = old 1 (neighbours
    old 2 -> new 1 with 2.5, old 0 -> new 2 with 1.5), new 1 = old 2, new 2 = old 0
    (worked by hand; a swapped perm / inverse gives new row 0 one neighbour)."""
    g = lapgen.path(3, w=[1.5, 2.5])
    rp, col, w = oracle.relabel(g, np.array([2, 0, 1], np.int64))
    assert rp.tolist() == [0, 2, 3, 4]
    assert col.tolist() == [1, 2, 0, 0]
    assert w.tolist() == [2.5, 1.5, 2.5, 1.5]


@pytest.mark.parametrize("seed", range(6))
def test_relabel_is_permutation_similarity(seed):
    """Pi L Pi^T against scipy's sparse product with the permutation matrix
    Pi[perm[i], i] = 1 (exact: every product is 1 * w * 1, every sum has one
    term), rows in ascending column order; unit weights for w = None; and the
    relabelled Laplacian applied to the permuted vector is the permuted L x."""
    import scipy.sparse as sp
    g = lapgen.random_connected(30 + 7 * seed, 50, seed, weighted=(seed % 2 == 0))
    n = g.n
    perm = np.random.default_rng(100 + seed).permutation(n).astype(np.int64)
    rp, col, w = oracle.relabel(g, perm)
    gw = np.ones(g.nnz) if g.w is None else g.w
    A = sp.csr_matrix((gw, g.col, g.row_ptr), shape=(n, n))
    Pi = sp.csr_matrix((np.ones(n), (perm, np.arange(n))), shape=(n, n))
    B = (Pi @ A @ Pi.T).tocsr()
    B.sort_indices()
    assert rp.tolist() == B.indptr.tolist()
    assert col.tolist() == B.indices.tolist()
    assert w.tolist() == B.data.tolist()
    x = np.random.default_rng(seed).standard_normal(n)
    d = oracle.row_sums(n, g.row_ptr, gw)
    y = oracle.spmv(n, g.row_ptr, g.col, gw, d, x)
    d2 = oracle.row_sums(n, rp, w)
    xp = np.empty(n); xp[perm] = x
    y2 = oracle.spmv(n, rp, col, w, d2, xp)
    assert np.allclose(y2[perm], y, rtol=0, atol=1e-12 * np.abs(y).max())
