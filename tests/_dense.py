"""Dense / brute-force helpers for pinning the oracle (test-only, numpy).

Each helper evaluates a definition from PAPER.md directly on dense matrices
(tiny n), independently of oracle/lap_oracle.c.
"""
import numpy as np


def dense_A(g):
    A = np.zeros((g.n, g.n))
    for i in range(g.n):
        for k in range(g.row_ptr[i], g.row_ptr[i + 1]):
            A[i, g.col[k]] = g.w[k]
    return A


def dense_L(g):
    """L = D - A."""
    A = dense_A(g)
    return np.diag(A.sum(axis=1)) - A


def csr_to_dense_L(n, row_ptr, col, w, d):
    L = np.zeros((n, n))
    for i in range(n):
        L[i, i] = d[i]
        for k in range(row_ptr[i], row_ptr[i + 1]):
            L[i, col[k]] = -w[k]
    return L


def brute_elim(L, hashes, max_degree=4):
    """Alg. 2 evaluated from its definitions on a dense L:
    candidates_i = i if degree <= 4 else empty; z_i = oplus over the stored
    entries of row i (the diagonal included) of candidates, choosing
    the smallest hash (ties: smaller index); eliminate i iff z_i = i."""
    n = L.shape[0]
    deg = [(np.count_nonzero(L[i]) - (1 if L[i, i] != 0 else 0)) for i in range(n)]
    cand = [i if deg[i] <= max_degree else None for i in range(n)]
    F = []
    for i in range(n):
        best = None
        for j in range(n):
            if L[i, j] == 0 and i != j:
                continue
            c = cand[j]
            if c is None:
                continue
            if best is None or (hashes[c], c) < (hashes[best], best):
                best = c
        if best == i:
            F.append(i)
    return F


def dense_schur(L, F):
    C = [i for i in range(L.shape[0]) if i not in set(F)]
    LFF = L[np.ix_(F, F)]
    LFC = L[np.ix_(F, C)]
    LCC = L[np.ix_(C, C)]
    if len(F) == 0:
        return LCC, C
    return LCC - LFC.T @ np.linalg.inv(LFF) @ LFC, C


SEED, UND, DEC = 2, 1, 0


def brute_vote(S, rounds=10, threshold=8, trace=False):
    """Alg. 3 on a dense S: synchronous rounds, frozen
    Seed/Decided (O-R9), oplus_agg = max of (state, w, -index) (P:597-612 +
    O-R10), votes >= threshold."""
    n = S.shape[0]
    st = [UND] * n
    idx = list(range(n))
    votes = [0] * n
    hist = []
    for t in range(1, rounds + 1):
        f = 0.5 ** t
        nst, nidx = st[:], idx[:]
        for i in range(n):
            if st[i] != UND:
                continue
            best = None
            for j in range(n):
                s = S[i, j]
                if j == i or s == 0 or s < f or st[j] == DEC:
                    continue
                key = (st[j], s, -j)
                if best is None or key > best:
                    best = key
            if best is None:
                continue
            j = -best[2]
            if best[0] == SEED:
                nst[i], nidx[i] = DEC, j
            else:
                votes[j] += 1
        for i in range(n):
            if nst[i] == UND and votes[i] >= threshold:
                nst[i] = SEED
        st, idx = nst, nidx
        hist.append((st[:], idx[:], votes[:]))
    roots = [i for i in range(n) if st[i] != DEC]
    rid = {r: k for k, r in enumerate(roots)}
    agg = [rid[i] if st[i] != DEC else rid[idx[i]] for i in range(n)]
    if trace:
        return agg, len(roots), st, votes, hist
    return agg, len(roots), st, votes


def cheb_T(k, x):
    return np.cos(k * np.arccos(x)) if abs(x) <= 1 else np.cosh(k * np.arccosh(abs(x))) * (np.sign(x) ** k)
