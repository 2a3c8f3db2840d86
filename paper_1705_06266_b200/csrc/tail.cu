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
template <int EPI>
__global__ void k_b_spmv(int64_t n, int64_t k, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                         const double *__restrict__ w, const double *__restrict__ d, const double *__restrict__ X,
                         double *__restrict__ Y, const double *__restrict__ B, double *__restrict__ DV, double c1,
                         double c2) {
    FOR_ELEM(e, n * k) {
        const int64_t i = e % n, c0 = e - i;
        double ax = 0.0;
        for (int64_t q = rp[i]; q < rp[i + 1]; q++) ax += w[q] * X[c0 + col[q]];
        const double xi = X[e], lx = d[i] * xi - ax;
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

// x = M b with M column-major n x n: a block owns 32 consecutive rows (lane =
// row, coalesced 256-byte reads of each column), its 32 warps split the
// columns, and the warp partials are summed in a fixed order in shared memory.
__global__ void __launch_bounds__(1024) k_dense_gemv(int64_t n, const double *__restrict__ M,
                                                     const double *__restrict__ b, double *__restrict__ x) {
    pdl_begin();
    __shared__ double part[32][33];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * 32 + lane;
    double acc = 0.0;
    if (i < n) {
        int64_t c = wid;
        for (; c + 96 < n; c += 128) {
            double m0 = M[c * n + i], m1 = M[(c + 32) * n + i], m2 = M[(c + 64) * n + i], m3 = M[(c + 96) * n + i];
            acc += m0 * b[c] + m1 * b[c + 32] + m2 * b[c + 64] + m3 * b[c + 96];
        }
        for (; c < n; c += 32) acc += M[c * n + i] * b[c];
    }
    part[wid][lane] = acc;
    __syncthreads();
    if (wid == 0) {
        double s = 0.0;
        for (int q = 0; q < 32; q++) s += part[q][lane];
        if (i < n) x[i] = s;
    }
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
        k_b_spmv<3><<<bg(n * k), 256, 0, s>>>(n, k, L.srp, L.scol, L.sw, L.sd, cur, alt, B, w.dv, rho * rho_old,
                                                2.0 * rho / delta);
        std::swap(cur, alt);
        rho_old = rho;
    }
    k_b_spmv<2><<<bg(n * k), 256, 0, s>>>(n, k, L.srp, L.scol, L.sw, L.sd, cur, w.r, B, w.dv, 0.0, 0.0);
    k_b_restrict<<<bg(L.m * k), 256, 0, s>>>(L.m, n, k, L.mem_ptr, L.members, w.r, WC.b);
    vcycle_batched(h, l + 1, k, W, WC.b, WC.x, s);
    k_b_prolong<<<bg(n * k), 256, 0, s>>>(n, L.m, k, L.agg_s, WC.x, cur);
    rho_old = 1.0 / sigma;
    for (int q = 0; q < K; q++) {
        double *dst = (q == K - 1) ? Xout : alt;
        if (q == 0) {
            k_b_spmv<5><<<bg(n * k), 256, 0, s>>>(n, k, L.srp, L.scol, L.sw, L.sd, cur, dst, B, w.dv, 0.0, 1.0 / theta);
        } else {
            double rho = 1.0 / (2.0 * sigma - rho_old);
            k_b_spmv<3><<<bg(n * k), 256, 0, s>>>(n, k, L.srp, L.scol, L.sw, L.sd, cur, dst, B, w.dv, rho * rho_old,
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
    launch_pdl(k_dense_gemv, (unsigned)((L.n + 31) / 32), 1024, s, L.n, (const double *)L.dense, b, x);
}

}  // namespace lap
