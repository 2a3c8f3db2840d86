"""Pins for low-degree elimination: Alg. 2 selection and the Schur level (O-P4, O-P5)."""
import json
import os

import numpy as np
import pytest

import lapgen
import oracle
from _dense import brute_elim, csr_to_dense_L, dense_L, dense_schur

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _g(ex):
    e = np.array(ex["edges"])
    return lapgen.csr_from_edges(ex["n"], e[:, 0], e[:, 1])


@pytest.mark.parametrize("key", ["elim_p3_identity_hash", "elim_p4_identity_hash",
                                 "elim_p4_hash_0517", "elim_star6_identity_hash"])
def test_spec_selection_examples(key):
    ex = GOLD[key]
    g = _g(ex)
    F, nF = oracle.elim_select(g.n, g.row_ptr, g.col, 4, 0, np.array(ex["hash"], dtype=np.uint64))
    assert np.flatnonzero(F).tolist() == ex["F"]
    assert nF == len(ex["F"])


@pytest.mark.parametrize("seed", range(50))
def test_selection_matches_brute_force_and_properties(seed):
    """S:635 corpus: 50 seeded random graphs, n <= 60, mixed degrees."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 61))
    g = lapgen.random_connected(n, int(rng.integers(0, 2 * n)), seed)
    F, nF = oracle.elim_select(g.n, g.row_ptr, g.col, 4, seed)
    s2 = oracle.salt(seed, 2)
    hashes = [oracle.mix64(i ^ s2) for i in range(n)]
    assert np.flatnonzero(F).tolist() == brute_elim(dense_L(g), hashes)
    deg = np.diff(g.row_ptr)
    for f in np.flatnonzero(F):
        nb = g.col[g.row_ptr[f]:g.row_ptr[f + 1]]
        assert deg[f] <= 4
        assert not F[nb].any()                                           # independent
        assert all(hashes[f] < hashes[j] for j in nb if deg[j] <= 4)      # minimal


def _elim_level(g, F):
    d = oracle.row_sums(g.n, g.row_ptr, g.w)
    fmap, nrp, ncol, nw, nd = oracle.schur(g.n, g.row_ptr, g.col, g.w, d, F.astype(np.uint8))
    return d, fmap, csr_to_dense_L(len(nd), nrp, ncol, nw, nd), (nrp, ncol, nw, nd)


def test_spec_schur_examples():
    g = lapgen.path(3)
    _, fmap, Lc, _ = _elim_level(g, np.array([1, 0, 0], bool))
    assert Lc.tolist() == GOLD["schur_p3_F0"]["L_next"]
    assert fmap.tolist() == [-1, 0, 1]
    g = lapgen.star(5)
    _, _, Lc, _ = _elim_level(g, np.array([0, 1, 1, 1, 1, 1], bool))
    assert Lc.tolist() == GOLD["schur_star6_leaves"]["L_next"]


@pytest.mark.parametrize("seed", range(30))
def test_schur_matches_dense_schur_and_is_laplacian(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 60))
    g = lapgen.random_connected(n, int(rng.integers(0, n)), seed)
    F, nF = oracle.elim_select(g.n, g.row_ptr, g.col, 4, seed)
    d, fmap, Lc, (nrp, ncol, nw, nd) = _elim_level(g, F)
    want, C = dense_schur(dense_L(g), np.flatnonzero(F).tolist())
    assert np.allclose(Lc, want, rtol=0, atol=1e-13 * np.abs(want).max())
    # coarse numbering is order preserving (O-R22)
    assert [fmap[c] for c in C] == list(range(len(C)))
    # Laplacian closure: W' > 0, bitwise symmetric, d' = row sum
    assert np.all(nw > 0)
    assert np.array_equal(Lc, Lc.T)
    assert np.all(np.abs(Lc.sum(axis=1)) <= 4 * np.spacing(np.abs(Lc).max()) * (1 + np.diff(nrp)))


def test_two_level_elimination_is_exact():
    """Elimination + exact coarse solve = dense minimum-norm solve."""
    for seed in range(10):
        g = lapgen.random_connected(40, 10, seed)
        F, _ = oracle.elim_select(g.n, g.row_ptr, g.col, 4, seed)
        d, fmap, Lc, _ = _elim_level(g, F)
        b = np.random.default_rng(seed).standard_normal(g.n)
        b -= b.mean()
        # P^T b: b'_idx(c) = b_c + sum_{f~c} (w_fc/d_f) b_f
        L = dense_L(g)
        Fi = np.flatnonzero(F)
        Ci = np.flatnonzero(~F)
        P = np.zeros((g.n, len(Ci)))
        P[Ci, np.arange(len(Ci))] = 1
        P[np.ix_(Fi, np.arange(len(Ci)))] = -np.linalg.inv(L[np.ix_(Fi, Fi)]) @ L[np.ix_(Fi, Ci)]
        xc = np.linalg.pinv(Lc) @ (P.T @ b)
        x = P @ xc
        x[Fi] += b[Fi] / d[Fi]
        xs = np.linalg.pinv(L) @ b
        assert np.allclose(x - x.mean(), xs, atol=1e-10 * np.abs(xs).max())
        assert np.allclose(P @ np.ones(len(Ci)), 1.0)                    # P 1 = 1 (O-P5)


def test_spec_restriction_example_p3():
    """with F = {0} on P3, P^T b = [-1, 1] for b = [1,-2,1] (dense P of P:458-461)."""
    ex = GOLD["elim_restrict_p3"]
    L = dense_L(lapgen.path(3))
    P = np.zeros((3, 2))
    P[1:, :] = np.eye(2)
    P[0, :] = -L[0, 1:] / L[0, 0]
    assert (P.T @ np.array(ex["b"], float)).tolist() == ex["b_next"]


def test_elimination_vcycle_is_exact_on_p3():
    """Elimination level + exact coarsest: one V-cycle is the exact solve.
    With seed 0, h(1) < h(2) < h(0) (golden hashes), so F = {1} (middle vertex)."""
    b = np.array([1.0, -2.0, 1.0])
    h = oracle.Hierarchy(lapgen.path(3), random_order=0, coarse_nnz=0, max_levels=2)
    L0 = h.level(0)
    assert L0.kind == oracle.ELIM and L0.fmap.tolist() == [0, -1, 1]
    assert h.level(1).kind == oracle.COARSEST
    x = h.vcycle(0, b)
    xs = np.linalg.pinv(dense_L(lapgen.path(3))) @ b
    assert np.allclose(x - x.mean(), xs, atol=1e-14)


def test_elim_rounds_consecutive_levels():
    """"we can run low-degree elimination multiple times in a row";
    elim_rounds = r allows up to r elimination levels in a row (default 1)."""
    g = lapgen.path(3000)
    for r in (1, 2, 4):
        h = oracle.Hierarchy(g, elim_rounds=r)
        kinds = [L.kind for L in h.levels()]
        run = best = 0
        for k in kinds:
            run = run + 1 if k == oracle.ELIM else 0
            best = max(best, run)
        assert best <= r
        if r > 1:
            assert best >= 2, kinds          # a path keeps passing the 5% gate
        x, it, rr, rc = h.solve(lapgen.rhs(g.n))
        assert rc == 0 and rr <= 1e-8
    # an elimination-only hierarchy down to the coarsest is an exact solver: one iteration
    h = oracle.Hierarchy(lapgen.path(200), elim_rounds=40)
    assert all(L.kind != oracle.AGG for L in h.levels())
    x, it, rr, rc = h.solve(lapgen.rhs(200))
    assert it == 1 and rr <= 1e-12
