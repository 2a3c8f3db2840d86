"""Pins for strength of connection, voting and Galerkin coarsening (O-P6..O-P8)."""
import json
import os

import numpy as np
import pytest

import lapgen
import oracle
from _dense import brute_vote, csr_to_dense_L, dense_A, dense_L

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _d(g):
    return oracle.row_sums(g.n, g.row_ptr, g.w)


# ------------------------------------------------------------------ strength

def test_spec_jacobi_sweep_p3():
    ex = GOLD["jacobi_sweep_p3"]
    g = lapgen.path(3)
    X0 = np.zeros((3, 4))
    X0[:, 0] = ex["x0"]
    X = oracle.test_vectors_from(3, g.row_ptr, g.col, g.w, _d(g), X0, sweeps=1, omega=ex["omega"])
    assert X[:, 0].tolist() == ex["x1"]


def test_constant_vector_is_fixed_point_of_sweeps():
    for g in [lapgen.grid2d(8, 8), lapgen.random_connected(50, 50, 1), lapgen.grid3d(5)]:
        X0 = np.full((g.n, 4), 0.5)  # power of two: every product w*c is exact (O-P6)
        X = oracle.test_vectors_from(g.n, g.row_ptr, g.col, g.w, _d(g), X0, sweeps=3)
        assert np.array_equal(X, X0)


def test_sweep_matches_damped_jacobi_definition():
    """x <- x - omega D^-1 L x on each column (O-R6), to rounding."""
    g = lapgen.random_connected(60, 80, 5)
    d = _d(g)
    X0 = np.random.default_rng(0).uniform(-1, 1, (g.n, 4))
    X = oracle.test_vectors_from(g.n, g.row_ptr, g.col, g.w, d, X0, sweeps=2)
    L = dense_L(g)
    Y = X0.copy()
    for _ in range(2):
        Y = Y - (2.0 / 3.0) * (L @ Y) / d[:, None]
    assert np.allclose(X, Y, atol=1e-14)


def test_initial_test_vectors_uniform_and_seeded():
    g = lapgen.grid2d(32, 32)
    X = oracle.test_vectors(g.n, g.row_ptr, g.col, g.w, _d(g), seed=0, level=0, attempt=0, sweeps=0)
    assert X.min() >= -1 and X.max() < 1 and abs(X.mean()) < 0.05
    X2 = oracle.test_vectors(g.n, g.row_ptr, g.col, g.w, _d(g), seed=0, level=0, attempt=1, sweeps=0)
    assert not np.array_equal(X, X2)
    X3 = oracle.test_vectors(g.n, g.row_ptr, g.col, g.w, _d(g), seed=0, level=1, attempt=0, sweeps=0)
    assert not np.array_equal(X, X3) and not np.array_equal(X2, X3)


def test_spec_affinity_example():
    ex = GOLD["affinity_p3"]
    g = lapgen.path(3)
    X = np.zeros((3, 4))
    X[:, :2] = ex["X"]
    C = oracle.affinity(3, g.row_ptr, g.col, X)
    # stored entries: row0:(1) row1:(0,2) row2:(1)
    assert C[0] == ex["C01"] and C[1] == ex["C01"] and C[2] == ex["C12"] and C[3] == ex["C12"]


def test_spec_normalize_example_k3():
    ex = GOLD["normalize_k3"]
    g = lapgen.complete(3)
    pair = {(0, 1): "01", (1, 0): "01", (1, 2): "12", (2, 1): "12", (0, 2): "02", (2, 0): "02"}
    C = np.zeros(g.nnz)
    for i in range(3):
        for k in range(g.row_ptr[i], g.row_ptr[i + 1]):
            C[k] = ex["C"][pair[(i, int(g.col[k]))]]
    S = oracle.normalize_strength(3, g.row_ptr, g.col, C)
    for i in range(3):
        for k in range(g.row_ptr[i], g.row_ptr[i + 1]):
            assert S[k] == ex["S"][pair[(i, int(g.col[k]))]]


@pytest.mark.parametrize("power", [1, 2])
def test_affinity_properties(power):
    g = lapgen.random_connected(60, 120, 2)
    X = oracle.test_vectors(g.n, g.row_ptr, g.col, g.w, _d(g), sweeps=3)
    C = oracle.affinity(g.n, g.row_ptr, g.col, X, power)
    A = dense_A(lapgen.Graph(g.n, g.row_ptr, g.col, C))
    assert np.array_equal(A, A.T)                                    # bitwise symmetric
    if power == 1:
        assert C.min() >= 0 and C.max() <= 1 + 1e-15                 # Cauchy-Schwarz
        # closed form: cos^2 of the angle between rows
        rows = np.repeat(np.arange(g.n), np.diff(g.row_ptr))
        xi, xj = X[rows], X[g.col]
        want = np.sum(xi * xj, 1) ** 2 / (np.sum(xi * xi, 1) * np.sum(xj * xj, 1))
        assert np.allclose(C, want, rtol=1e-14, atol=0)
    for k in [-3, 5]:                                                # C(2^k X) = C(X) exactly (power 1)
        Ck = oracle.affinity(g.n, g.row_ptr, g.col, X * 2.0 ** k, power)
        if power == 1:
            assert np.array_equal(Ck, C)
    S = oracle.normalize_strength(g.n, g.row_ptr, g.col, C)
    assert S.min() >= 0 and S.max() == 1.0
    # S_ij = 1 iff C_ij is the max of both its row and its column (corrected S:248)
    M = np.array([C[g.row_ptr[i]:g.row_ptr[i + 1]].max() for i in range(g.n)])
    rows = np.repeat(np.arange(g.n), np.diff(g.row_ptr))
    mutual = (C == M[rows]) & (C == M[g.col])
    assert np.array_equal(S == 1.0, mutual)


# ------------------------------------------------------------------ voting

def test_spec_vote_k3():
    g = lapgen.complete(3)
    S = np.ones(g.nnz)
    _, _, st, votes = oracle.aggregate(3, g.row_ptr, g.col, S, rounds=1)
    assert votes.tolist() == GOLD["vote_k3_round1_votes"]["votes"]
    ex = GOLD["vote_k3_seed_round"]
    _, _, st3, _ = oracle.aggregate(3, g.row_ptr, g.col, S, rounds=ex["seed_round"] - 1)
    _, _, st4, _ = oracle.aggregate(3, g.row_ptr, g.col, S, rounds=ex["seed_round"])
    _, _, st5, _ = oracle.aggregate(3, g.row_ptr, g.col, S, rounds=ex["decided_round"])
    assert st3[ex["seed"]] == 1 and st4[ex["seed"]] == 2
    assert st5.tolist() == [2, 0, 0]
    agg, m, _, _ = oracle.aggregate(3, g.row_ptr, g.col, S)
    assert m == 1 and agg.tolist() == [0, 0, 0]


def test_spec_vote_p3():
    ex = GOLD["vote_p3_seed_round"]
    g = lapgen.path(3)
    S = np.ones(g.nnz)
    _, _, st3, _ = oracle.aggregate(3, g.row_ptr, g.col, S, rounds=ex["seed_round"] - 1)
    _, _, st4, _ = oracle.aggregate(3, g.row_ptr, g.col, S, rounds=ex["seed_round"])
    assert st3[ex["seed"]] == 1 and st4[ex["seed"]] == 2
    agg, m, _, _ = oracle.aggregate(3, g.row_ptr, g.col, S)
    assert m == 1


def test_empty_strength_gives_singletons():
    g = lapgen.random_connected(30, 20, 0)
    agg, m, st, votes = oracle.aggregate(g.n, g.row_ptr, g.col, np.zeros(g.nnz))
    assert m == g.n and agg.tolist() == list(range(g.n)) and votes.sum() == 0


@pytest.mark.parametrize("seed", range(25))
def test_vote_matches_brute_force(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 50))
    g = lapgen.random_connected(n, int(rng.integers(0, 3 * n)), seed)
    if seed % 2:
        X = oracle.test_vectors(g.n, g.row_ptr, g.col, g.w, _d(g), seed=seed, sweeps=3)
        S = oracle.normalize_strength(g.n, g.row_ptr, g.col, oracle.affinity(g.n, g.row_ptr, g.col, X))
    else:  # coarse values with many exact ties to exercise the index tie-break
        S = rng.choice([0.0, 0.25, 0.5, 1.0], g.nnz)
        Sd = dense_A(lapgen.Graph(g.n, g.row_ptr, g.col, S))
        Sd = np.maximum(Sd, Sd.T)
        S = Sd[np.repeat(np.arange(g.n), np.diff(g.row_ptr)), g.col]
    thr = int(rng.integers(1, 9))
    agg, m, st, votes = oracle.aggregate(g.n, g.row_ptr, g.col, S, 10, thr)
    Sd = dense_A(lapgen.Graph(g.n, g.row_ptr, g.col, S))
    bagg, bm, bst, bvotes = brute_vote(Sd, 10, thr)
    assert agg.tolist() == bagg and m == bm and st.tolist() == bst and votes.tolist() == bvotes
    # totality: each aggregate has exactly one root (Seed/Undecided), ids 0..m-1 ascending by root
    roots = np.flatnonzero(st != 0)
    assert agg[roots].tolist() == list(range(m))
    assert set(agg.tolist()) == set(range(m))


# ------------------------------------------------------------------ Galerkin

def test_spec_galerkin_p3():
    ex = GOLD["galerkin_p3"]
    g = lapgen.path(3)
    crp, ccol, cw, cd = oracle.galerkin(3, g.row_ptr, g.col, g.w, np.array(ex["agg"]), 2)
    assert csr_to_dense_L(2, crp, ccol, cw, cd).tolist() == ex["L_next"]


def test_galerkin_identity_and_single_aggregate():
    g = lapgen.random_connected(25, 30, 4)
    d = _d(g)
    crp, ccol, cw, cd = oracle.galerkin(g.n, g.row_ptr, g.col, g.w, np.arange(g.n), g.n)
    assert np.array_equal(crp, g.row_ptr) and np.array_equal(ccol, g.col) and np.array_equal(cw, g.w)
    assert np.array_equal(cd, d)
    crp, ccol, cw, cd = oracle.galerkin(g.n, g.row_ptr, g.col, g.w, np.zeros(g.n), 1)
    assert crp.tolist() == [0, 0] and cd.tolist() == [0.0]


@pytest.mark.parametrize("seed", range(15))
def test_galerkin_matches_dense_RLP(seed):
    rng = np.random.default_rng(seed)
    g = lapgen.random_connected(int(rng.integers(5, 60)), 40, seed)
    m = int(rng.integers(1, g.n + 1))
    agg = np.concatenate([np.arange(m), rng.integers(0, m, g.n - m)])
    rng.shuffle(agg)
    crp, ccol, cw, cd = oracle.galerkin(g.n, g.row_ptr, g.col, g.w, agg, m)
    R = np.zeros((m, g.n))
    R[agg, np.arange(g.n)] = 1
    want = R @ dense_L(g) @ R.T
    Lc = csr_to_dense_L(m, crp, ccol, cw, cd)
    assert np.allclose(Lc, want, atol=1e-13 * max(1, np.abs(want).max()))
    assert np.array_equal(Lc, Lc.T) and np.all(cw > 0)
