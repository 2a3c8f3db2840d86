// tail.cu -- the V-cycle below a small level as ONE dense operator.
//
// V(l, b) (Alg. 1 with gamma = 1; O-S7) is linear in b: zero
// initial guess, fixed Chebyshev polynomials, exact elimination transfers and
// the dense L_c^+ at the bottom.  Below the first level t with n_t <=
// DTAIL_MAX_N the cycle is a chain of ~15-20 tiny kernels whose cost is pure
// dependent-load latency (4-7 us each on B200 inside a CUDA graph, DESIGN.md
// §7).  At setup we therefore apply the sub-cycle V(t, .) to the n_t unit
// vectors at once -- a batched (column-major, n_l x n_t) replay of exactly the
// same recursion and formulas as solve.cu vcycle_rec -- and keep
//     M_t = [V(t, e_0) ... V(t, e_{n_t-1})]        (n_t x n_t, column-major)
// so that in the solve V(t, b) = M_t b is one GEMV (<= 75 MB, one launch).
// The operator is the method's own (linearity), only the rounding differs:
// solve-phase parity is by tolerance (O-P2 / O-S8), and tests compare the
// cycle against the oracle's V-cycle.  LAP_DENSE_TAIL=0 disables it.
#include <algorithm>
#include <vector>

#include "lap_internal.cuh"

namespace lap {

#define FOR_ELEM(e, total) \
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (total); e += (int64_t)gridDim.x * blockDim.x)

__global__ void k_b_identity(int64_t n, double *X) {
    FOR_ELEM(e, n * n) X[e] = (e % n == e / n) ? 1.0 : 0.0;
}
__global__ void k_b_cheb_first(int64_t n, int64_t k, const double *__restrict__ B, const double *__restrict__ d,
                               double inv_theta, double *__restrict__ X, double *__restrict__ DV) {
    FOR_ELEM(e, n * k) {
        int64_t i = e % n;
        double v = (B[e] / d[i]) * inv_theta;
        DV[e] = v;
        X[e] = v;
    }
}
// the SpMV epilogues of solve.cu (E_CHEB = 3, E_RESID = 2, E_CHEB0 = 5), column by column
// A thread owns row i of BC consecutive columns: each matrix entry is loaded
// once for BC gathers (the matrix was re-read once per column: ~1 GB of L2
// traffic per pass on cfg 2's 2486-column tail); per column, the row sum and
// the epilogue are the single-column ones.
constexpr int BC = 4;
template <int EPI>
__global__ void k_b_spmv(int64_t n, int64_t k, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                         const double *__restrict__ w, const double *__restrict__ d, const double *__restrict__ X,
                         double *__restrict__ Y, const double *__restrict__ B, double *__restrict__ DV, double c1,
                         double c2) {
    const int64_t ngrp = (k + BC - 1) / BC;
    FOR_ELEM(e0, n * ngrp) {
        const int64_t i = e0 % n, cb = (e0 / n) * BC;
        const int nc = (int)min((int64_t)BC, k - cb);
        double ax[BC] = {0.0, 0.0, 0.0, 0.0};
        for (int64_t q = rp[i]; q < rp[i + 1]; q++) {
            const double wq = w[q];
            const int64_t j = col[q];
#pragma unroll
            for (int u = 0; u < BC; u++)
                if (u < nc) ax[u] += wq * X[(cb + u) * n + j];
        }
#pragma unroll
        for (int u = 0; u < BC; u++) {
            if (u >= nc) break;
            const int64_t e = (cb + u) * n + i;
            const double xi = X[e], lx = d[i] * xi - ax[u];
            if (EPI == 2) {
                Y[e] = B[e] - lx;
            } else if (EPI == 3) {
                double dv = c1 * DV[e] + c2 * ((B[e] - lx) / d[i]);
                DV[e] = dv;
                Y[e] = xi + dv;
            } else {
                double dv = c2 * ((B[e] - lx) / d[i]);
                DV[e] = dv;
                Y[e] = xi + dv;
            }
        }
    }
}
__global__ void k_b_restrict(int64_t m, int64_t n, int64_t k, const int64_t *__restrict__ mp,
                             const int32_t *__restrict__ mem, const double *__restrict__ R, double *__restrict__ RC) {
    FOR_ELEM(e, m * k) {
        const int64_t a = e % m, c = e / m;
        double s = 0.0;
        for (int64_t q = mp[a]; q < mp[a + 1]; q++) s += R[c * n + mem[q]];
        RC[e] = s;
    }
}
__global__ void k_b_prolong(int64_t n, int64_t m, int64_t k, const int32_t *__restrict__ agg,
                            const double *__restrict__ XC, double *__restrict__ X) {
    FOR_ELEM(e, n * k) {
        const int64_t i = e % n, c = e / n;
        X[e] += XC[c * m + agg[i]];
    }
}
__global__ void k_b_elim_restrict(int64_t nc, int64_t n, int64_t k, const int32_t *__restrict__ cid,
                                  const int64_t *__restrict__ ctp, const int32_t *__restrict__ ctf,
                                  const double *__restrict__ ctc, const double *__restrict__ B,
                                  double *__restrict__ BC) {
    FOR_ELEM(e, nc * k) {
        const int64_t kk = e % nc, c0 = (e / nc) * n;
        double s = B[c0 + cid[kk]];
        for (int64_t q = ctp[kk]; q < ctp[kk + 1]; q++) s += ctc[q] * B[c0 + ctf[q]];
        BC[e] = s;
    }
}
__global__ void k_b_elim_prolong(int64_t nc, int64_t nf, int64_t n, int64_t k, const int32_t *__restrict__ cid,
                                 const int32_t *__restrict__ flist, const int32_t *__restrict__ fmap,
                                 const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                                 const double *__restrict__ w, const double *__restrict__ d,
                                 const double *__restrict__ B, const double *__restrict__ XC, double *__restrict__ X) {
    FOR_ELEM(e, (nc + nf) * k) {
        const int64_t t = e % (nc + nf), c = e / (nc + nf);
        if (t < nc) {
            X[c * n + cid[t]] = XC[c * nc + t];
        } else {
            const int64_t f = flist[t - nc];
            double s = B[c * n + f];
            for (int64_t q = rp[f]; q < rp[f + 1]; q++) s += w[q] * XC[c * nc + fmap[col[q]]];
            X[c * n + f] = s / d[f];
        }
    }
}
__global__ void k_b_coarse(int64_t n, int64_t k, const double *__restrict__ P, const double *__restrict__ B,
                           double *__restrict__ X) {
    FOR_ELEM(e, n * k) {
        const int64_t i = e % n, c0 = e - i;
        double acc = 0.0;
        for (int64_t j = 0; j < n; j++) acc += P[i * n + j] * B[c0 + j];
        X[e] = acc;
    }
}

// x = M b with M column-major n x n (the 49 MB operator of cfg 2's tail is
// streamed from HBM every V-cycle).  Grid = (row tiles of 32) x (DG_SPLIT
// column ranges): a block's 8 warps stride over its column range (lane = row,
// coalesced 256-byte reads, 4 columns in flight per warp), the warp partials
// are summed in warp order in shared memory, the split partial goes to
// part[split][row], and the LAST block of a row tile to arrive (per-tile
// counter) sums the DG_SPLIT partials in split order: deterministic, and
// ~600 blocks over all SMs instead of one 1024-thread block per 32 rows
// (78 blocks on cfg 2: 1.9 TB/s).
template <int NW>  // warps per block: 32 for unsplit small operators, 8 for the split ones
__global__ void __launch_bounds__(NW * 32) k_dense_gemv(int64_t n, const double *__restrict__ M,
                                                        const double *__restrict__ b, double *__restrict__ x,
                                                        double *__restrict__ part, int *__restrict__ cnt) {
    pdl_begin();
    __shared__ double wp[NW][33];
    __shared__ int last;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int nw = NW;
    const int64_t i = (int64_t)blockIdx.x * 32 + lane;
    const int nsplit = gridDim.y, sp = blockIdx.y;
    const int64_t cb = n * sp / nsplit, ce = n * (sp + 1) / nsplit;
    double acc = 0.0;
    if (i < n) {
        int64_t c = cb + wid;
        for (; c + 7 * nw < ce; c += 8 * nw) {  // 8 columns in flight per warp
            double m[8];
#pragma unroll
            for (int u = 0; u < 8; u++) m[u] = __ldg(&M[(c + u * nw) * n + i]);
#pragma unroll
            for (int u = 0; u < 8; u++) acc += m[u] * b[c + u * nw];
        }
        for (; c < ce; c += nw) acc += __ldg(&M[c * n + i]) * b[c];
    }
    wp[wid][lane] = acc;
    __syncthreads();
    if (nsplit == 1) {  // small operators: no split, no combine
        if (wid == 0) {
            double s = 0.0;
            for (int q = 0; q < nw; q++) s += wp[q][lane];
            if (i < n) x[i] = s;
        }
        return;
    }
    if (wid == 0) {
        double s = 0.0;
        for (int q = 0; q < nw; q++) s += wp[q][lane];
        if (i < n) part[(int64_t)sp * n + i] = s;
        __threadfence();
    }
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&cnt[blockIdx.x], 1) == nsplit - 1;
    __syncthreads();
    if (!last) return;
    if (wid == 0) {
        __threadfence();
        double s = 0.0;
        for (int q = 0; q < nsplit; q++) s += (i < n) ? __ldcg(&part[(int64_t)q * n + i]) : 0.0;
        if (i < n) x[i] = s;
        if (lane == 0) cnt[blockIdx.x] = 0;
    }
}

static unsigned dense_splits(int64_t n) {  // ~4 blocks of 256 per SM in total, >= 256 columns per split
    if (n < 1536) return 1;  // latency-bound: the split combine costs more than it saves
    const int64_t tiles = (n + 31) / 32;
    int64_t sp = (4 * 148 + tiles - 1) / tiles;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(sp, n / 256));
}

static inline unsigned bg(int64_t total) { return grid_for(total, 256, 148 * 16); }

// batched replay of solve.cu vcycle_rec on k column vectors (column-major)
struct BWork {
    double *b = nullptr, *x = nullptr, *x2 = nullptr, *t = nullptr, *r = nullptr, *dv = nullptr;
};
static void vcycle_batched(lap_hierarchy *h, int l, int64_t k, std::vector<BWork> &W, const double *B, double *Xout,
                           cudaStream_t s) {
    Level &L = h->lev[l];
    const int64_t n = L.n;
    if (L.kind == KIND_COARSEST) {
        k_b_coarse<<<bg(n * k), 256, 0, s>>>(n, k, L.pinv_s, B, Xout);
        LAP_CHECK_LAUNCH();
        return;
    }
    Level &C = h->lev[l + 1];
    BWork &WC = W[l + 1];
    if (L.kind == KIND_ELIM) {
        const int64_t nc = C.n;
        k_b_elim_restrict<<<bg(nc * k), 256, 0, s>>>(nc, n, k, L.cid_s, L.ct_ptr_s, L.ct_f_s, L.ct_coef_s, B, WC.b);
        vcycle_batched(h, l + 1, k, W, WC.b, WC.x, s);
        k_b_elim_prolong<<<bg((nc + L.nF) * k), 256, 0, s>>>(nc, L.nF, n, k, L.cid_s, L.flist, L.fmap_s, L.srp, L.scol,
                                                              L.sw, L.sd, B, WC.x, Xout);
        LAP_CHECK_LAUNCH();
        return;
    }
    BWork &w = W[l];
    const int K = h->p.cheby_degree;
    const double theta = L.cheb_theta, delta = L.cheb_delta, sigma = L.cheb_sigma;
    double *cur = w.x2, *alt = w.t;
    k_b_cheb_first<<<bg(n * k), 256, 0, s>>>(n, k, B, L.sd, 1.0 / theta, cur, w.dv);
    double rho_old = 1.0 / sigma;
    for (int q = 1; q < K; q++) {
        double rho = 1.0 / (2.0 * sigma - rho_old);
        k_b_spmv<3><<<bg(n * ((k + BC - 1) / BC)), 256, 0, s>>>(n, k, L.srp, L.scol, L.sw, L.sd, cur, alt, B, w.dv, rho * rho_old,
                                                2.0 * rho / delta);
        std::swap(cur, alt);
        rho_old = rho;
    }
    k_b_spmv<2><<<bg(n * ((k + BC - 1) / BC)), 256, 0, s>>>(n, k, L.srp, L.scol, L.sw, L.sd, cur, w.r, B, w.dv, 0.0, 0.0);
    k_b_restrict<<<bg(L.m * k), 256, 0, s>>>(L.m, n, k, L.mem_ptr, L.members, w.r, WC.b);
    vcycle_batched(h, l + 1, k, W, WC.b, WC.x, s);
    k_b_prolong<<<bg(n * k), 256, 0, s>>>(n, L.m, k, L.agg_s, WC.x, cur);
    rho_old = 1.0 / sigma;
    for (int q = 0; q < K; q++) {
        double *dst = (q == K - 1) ? Xout : alt;
        if (q == 0) {
            k_b_spmv<5><<<bg(n * ((k + BC - 1) / BC)), 256, 0, s>>>(n, k, L.srp, L.scol, L.sw, L.sd, cur, dst, B, w.dv, 0.0, 1.0 / theta);
        } else {
            double rho = 1.0 / (2.0 * sigma - rho_old);
            k_b_spmv<3><<<bg(n * ((k + BC - 1) / BC)), 256, 0, s>>>(n, k, L.srp, L.scol, L.sw, L.sd, cur, dst, B, w.dv, rho * rho_old,
                                                    2.0 * rho / delta);
            rho_old = rho;
        }
        if (q < K - 1) std::swap(cur, alt);
    }
    LAP_CHECK_LAUNCH();
}

void build_dense_tail(lap_hierarchy *h, cudaStream_t s) {
    const char *e = getenv("LAP_DENSE_TAIL");
    if (e && e[0] == '0') return;
    const int nl = (int)h->lev.size();
    int t = -1;
    for (int l = 1; l < nl - 1; l++)
        if (h->lev[l].n <= DTAIL_MAX_N) {
            t = l;
            break;
        }
    if (t < 0) return;
    const int64_t k = h->lev[t].n;
    std::vector<BWork> W(nl);
    std::vector<void *> tmp;
    auto al = [&](int64_t cnt) {
        double *p = (double *)dalloc(sizeof(double) * (size_t)(cnt > 0 ? cnt : 1), s);
        tmp.push_back(p);
        return p;
    };
    for (int l = t; l < nl; l++) {
        const int64_t sz = h->lev[l].n * k;
        W[l].b = al(sz);
        W[l].x = al(sz);
        if (h->lev[l].kind == KIND_AGG) {
            W[l].x2 = al(sz);
            W[l].t = al(sz);
            W[l].r = al(sz);
            W[l].dv = al(sz);
        }
    }
    Level &T = h->lev[t];
    T.dense = (double *)dalloc(sizeof(double) * (size_t)(k * k), s);
    T.dense_part = (double *)dalloc(sizeof(double) * (size_t)k * dense_splits(k), s);
    T.dense_cnt = (int *)dalloc(sizeof(int) * (size_t)((k + 31) / 32), s);
    LAP_CUDA(cudaMemsetAsync(T.dense_cnt, 0, sizeof(int) * (size_t)((k + 31) / 32), s));
    try {
        k_b_identity<<<bg(k * k), 256, 0, s>>>(k, W[t].b);
        vcycle_batched(h, t, k, W, W[t].b, T.dense, s);
        LAP_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
        for (void *p : tmp) dfree(p, s);
        throw;
    }
    for (void *p : tmp) dfree(p, s);
    h->dtail_level = t;
}

void launch_dense_gemv(const Level &L, const double *b, double *x, cudaStream_t s) {
    const unsigned tiles = (unsigned)((L.n + 31) / 32);
    cudaLaunchConfig_t cfg = {};
    const unsigned sp = dense_splits(L.n);
    cfg.gridDim = dim3(tiles, sp);
    cfg.blockDim = dim3(sp == 1 ? 1024 : 256);  // unsplit small operators: 32 warps share a tile's columns
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    if (sp == 1)
        LAP_CUDA(cudaLaunchKernelEx(&cfg, k_dense_gemv<32>, L.n, (const double *)L.dense, b, x, L.dense_part,
                                    L.dense_cnt));
    else
        LAP_CUDA(cudaLaunchKernelEx(&cfg, k_dense_gemv<8>, L.n, (const double *)L.dense, b, x, L.dense_part,
                                    L.dense_cnt));
}

}  // namespace lap
