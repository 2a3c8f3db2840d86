"""Host-side accounting for the benchmark (no part of the method's arithmetic).

Work units and WDA as the paper defines them (§2.3.1):

    WDA = -work / log10(dr),  dr = ||r_final|| / ||r_initial||,
    work = FLOPs / FLOPs of one residual on the finest level,

approximated, as the paper allows ("typically approximated in terms of the
number of nonzeros in the sparse operators"), by nonzero counts:
one application of L_l costs nnz(L_l)/nnz(L_0) units with nnz(L) = n + nnz_off
(P:672-673); a restriction or prolongation (n_l + m_l)/nnz(L_0); an
elimination transfer (restriction or prolongation) (n_l + nnz(L_FC))/nnz(L_0);
a vector operation n_0/nnz(L_0); the coarsest solve n_c^2/nnz(L_0).
TDA = -time / log10(dr).
"""
from __future__ import annotations

import math

AGG, ELIM, COARSEST = 0, 1, 2


def vcycle_work(levels, cheby_degree: int = 2) -> float:
    """Work units of one V-cycle (O-S7) over `levels`: list of dicts with
    kind, n, nnz (off-diagonal), m (aggregation: next level size) and
    nnz_fc (elimination: stored entries of the eliminated rows)."""
    nnz0 = levels[0]["n"] + levels[0]["nnz"]
    w = 0.0
    for i, L in enumerate(levels):
        nl = L["n"] + L["nnz"]
        if L["kind"] == COARSEST:
            w += L["n"] ** 2 / nnz0
            break
        if L["kind"] == ELIM:
            w += 2.0 * (L["n"] + L.get("nnz_fc", 0)) / nnz0
            continue
        m = L.get("m", levels[i + 1]["n"] if i + 1 < len(levels) else 0)
        # pre: step 0 (elementwise) + (K-1) SpMV steps; residual; post: K SpMV steps
        w += (2 * cheby_degree) * nl / nnz0 + L["n"] / nnz0
        w += 2.0 * (L["n"] + m) / nnz0        # R and P
    return w


def solve_work(levels, iters: int, vcycles: int, cheby_degree: int = 2, vec_ops_per_iter: int = 8) -> float:
    """Work units of one PCG solve (O-S8): per iteration one fine SpMV,
    `vec_ops_per_iter` vector operations and one V-cycle; plus the final
    true-residual SpMV."""
    n0 = levels[0]["n"]
    nnz0 = n0 + levels[0]["nnz"]
    per_it = 1.0 + vec_ops_per_iter * n0 / nnz0
    return iters * per_it + vcycles * vcycle_work(levels, cheby_degree) + 1.0


def wda(work: float, dr: float) -> float:
    """-work / log10(dr); raises ValueError when no digit was gained."""
    if not (dr > 0.0) or dr >= 1.0:
        raise ValueError("no residual reduction: WDA undefined")
    return -work / math.log10(dr)


def tda(time_s: float, dr: float) -> float:
    if not (dr > 0.0) or dr >= 1.0:
        raise ValueError("no residual reduction: TDA undefined")
    return -time_s / math.log10(dr)


def vcycle_spmv_edges(levels, cheby_degree: int = 2) -> int:
    """SpMV edges of one V-cycle = sum over aggregation levels of
    2K nnz_off(L_l) ((K-1) pre + 1 residual + K post smoother SpMVs; 4 nnz
    for the paper's degree K = 2)."""
    return sum(2 * cheby_degree * L["nnz"] for L in levels if L["kind"] == AGG)


def solve_spmv_edges(levels, iters: int, vcycles: int, cheby_degree: int = 2) -> int:
    """SpMV edges of one PCG solve (O-S8): `vcycles` V-cycles, `iters` fine
    products q = L p, the true-residual confirmation and the final residual."""
    return vcycles * vcycle_spmv_edges(levels, cheby_degree) + (iters + 2) * levels[0]["nnz"]
