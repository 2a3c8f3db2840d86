// solve.cu -- solve-phase kernels (sm_100a): degree-binned fp64 Laplacian
// SpMV with fused epilogues (H0/H1/H2/H3), aggregate restriction and
// prolongation (H3/H4), exact elimination transfers (H5), coarsest GEMV (H6),
// deterministic PCG reductions (H7), V-cycle (H16, Alg. 1 with gamma = 1,
// P:209-233) and PCG.
//
// HBM-bound by construction (2 flops per 12-20 bytes): the kernels stream
// col/w with coalesced loads through the read-only path, keep the gathered x
// vector L2-resident, and fuse every elementwise step of the smoother into
// the SpMV that produces its input.  All reductions are two-pass with a fixed
// launch geometry, so every run is bitwise reproducible.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "lap_internal.cuh"

namespace lap {

struct Csr {
    const int64_t *__restrict__ rp;
    const int32_t *__restrict__ col;
    const double *__restrict__ w;
    const double *__restrict__ d;
};

// ------------------------------------------------------------------ epilogues
// Ax = sum_j w_ij x_j ; (L x)_i = d_i x_i - Ax  (L = D - A)
enum { E_SPMV = EPI_SPMV, E_DOT = EPI_SPMV_DOT, E_RESID = EPI_RESID, E_CHEB = EPI_CHEB, E_CHEB0 = 5 };

template <int EPI>
__device__ __forceinline__ void apply_epi(int64_t i, double ax, const Csr &A, const EpiArgs &a, double &dacc) {
    double xi = a.x[i];
    double lx = A.d[i] * xi - ax;
    if (EPI == E_SPMV) {
        a.y[i] = lx;
    } else if (EPI == E_DOT) {
        a.y[i] = lx;
        dacc += xi * lx;
    } else if (EPI == E_RESID) {
        a.y[i] = a.b[i] - lx;
    } else if (EPI == E_CHEB) {  // dv = c1 dv + c2 D^-1 (b - L x); x_out = x + dv   (O-S6)
        double r = a.b[i] - lx;
        double dv = a.c1 * a.dv[i] + a.c2 * (r / A.d[i]);
        a.dv[i] = dv;
        a.y[i] = xi + dv;
    } else if (EPI == E_CHEB0) {  // first step from a nonzero x: dv = D^-1 r / theta
        double r = a.b[i] - lx;
        double dv = a.c2 * (r / A.d[i]);
        a.dv[i] = dv;
        a.y[i] = xi + dv;
    }
}

__device__ __forceinline__ double block_sum(double v, double *sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double r = 0.0;
    if (wid == 0) {
        int nw = blockDim.x >> 5;
        r = lane < nw ? sh[lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    }
    return r;  // valid in thread 0
}

// class 0: SELL-32 (rows of <= SHORT_MAX entries).  A warp owns a 32-row
// slice, a thread owns a row; the slice is stored column-major and padded to
// its widest row, so every col/w load instruction is one fully coalesced
// 128/256-byte access.  Epilogue operands are loaded before the gather loop
// so their latency overlaps it.  No shared memory, no barriers.
template <int EPI>
__global__ void __launch_bounds__(256, 6) k_spmv_sell(int64_t nslices, int64_t nrows, const int64_t *__restrict__ sp,
                                                   const int32_t *__restrict__ ec, const double *__restrict__ ew,
                                                   Csr A, EpiArgs a, double *__restrict__ partials) {
    __shared__ double sh[8];
    const int lane = threadIdx.x & 31;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double dacc = 0.0;
    for (int64_t sl = warp; sl < nslices; sl += nwarps) {
        const int64_t i = sl * 32 + lane;
        const int64_t beg = sp[sl], end = sp[sl + 1];
        double xi = 0.0, di = 0.0, bi = 0.0, dvi = 0.0;
        const bool live = i < nrows;
        if (live) {
            xi = a.x[i];
            di = A.d[i];
            if (EPI == E_RESID || EPI == E_CHEB || EPI == E_CHEB0) bi = a.b[i];
            if (EPI == E_CHEB) dvi = a.dv[i];
        }
        double acc0 = 0.0, acc1 = 0.0;
        int64_t k = beg + lane;
        for (; k + 32 < end; k += 64) {
            int c0 = __ldg(&ec[k]), c1 = __ldg(&ec[k + 32]);
            double w0 = __ldg(&ew[k]), w1 = __ldg(&ew[k + 32]);
            acc0 += w0 * a.x[c0];
            acc1 += w1 * a.x[c1];
        }
        if (k < end) acc0 += __ldg(&ew[k]) * a.x[__ldg(&ec[k])];
        if (live) {
            double ax = acc0 + acc1;
            double lx = di * xi - ax;
            if (EPI == E_SPMV) {
                a.y[i] = lx;
            } else if (EPI == E_DOT) {
                a.y[i] = lx;
                dacc += xi * lx;
            } else if (EPI == E_RESID) {
                a.y[i] = bi - lx;
            } else if (EPI == E_CHEB) {
                double dv = a.c1 * dvi + a.c2 * ((bi - lx) / di);
                a.dv[i] = dv;
                a.y[i] = xi + dv;
            } else if (EPI == E_CHEB0) {
                double dv = a.c2 * ((bi - lx) / di);
                a.dv[i] = dv;
                a.y[i] = xi + dv;
            }
        }
    }
    if (EPI == E_DOT) {
        double r = block_sum(dacc, sh);
        if (threadIdx.x == 0) partials[blockIdx.x] = r;
    }
}

// class 1: warp per row, rows [row0, row0 + cnt)
template <int EPI>
__global__ void __launch_bounds__(256) k_spmv_warp(int64_t cnt, int64_t row0, Csr A, EpiArgs a,
                                                   double *__restrict__ partials) {
    __shared__ double sh[8];
    const int lane = threadIdx.x & 31;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double dacc = 0.0;
    for (int64_t t = warp; t < cnt; t += nwarps) {
        int64_t i = row0 + t;
        int64_t s = A.rp[i], e = A.rp[i + 1];
        double a0 = 0.0, a1 = 0.0;
        int64_t k = s + lane;
        for (; k + 32 < e; k += 64) {
            int c0 = __ldg(&A.col[k]), c1 = __ldg(&A.col[k + 32]);
            double w0 = __ldg(&A.w[k]), w1 = __ldg(&A.w[k + 32]);
            a0 += w0 * a.x[c0];
            a1 += w1 * a.x[c1];
        }
        if (k < e) a0 += __ldg(&A.w[k]) * a.x[__ldg(&A.col[k])];
        double acc = a0 + a1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) apply_epi<EPI>(i, acc, A, a, dacc);
    }
    if (EPI == E_DOT) {
        double r = block_sum(dacc, sh);
        if (threadIdx.x == 0) partials[blockIdx.x] = r;
    }
}

// class 2: one 256-thread block per row
template <int EPI>
__global__ void __launch_bounds__(256) k_spmv_block(int64_t cnt, int64_t row0, Csr A, EpiArgs a,
                                                    double *__restrict__ partials) {
    __shared__ double sh[8];
    double dacc = 0.0;
    for (int64_t t = blockIdx.x; t < cnt; t += gridDim.x) {
        int64_t i = row0 + t;
        int64_t s = A.rp[i], e = A.rp[i + 1];
        double acc = 0.0;
#pragma unroll 4
        for (int64_t k = s + threadIdx.x; k < e; k += blockDim.x) acc += __ldg(&A.w[k]) * a.x[__ldg(&A.col[k])];
        double r = block_sum(acc, sh);
        if (threadIdx.x == 0) apply_epi<EPI>(i, r, A, a, dacc);
    }
    if (EPI == E_DOT) {
        __syncthreads();
        double r = block_sum(threadIdx.x == 0 ? dacc : 0.0, sh);
        if (threadIdx.x == 0) partials[blockIdx.x] = r;
    }
}

// class 3: block per HUB_CHUNK-entry chunk -> ordered partial sums, then epilogue
__global__ void __launch_bounds__(256) k_spmv_hub_chunks(int64_t nchunks, int64_t nhub, int64_t row0,
                                                         const int64_t *__restrict__ cfirst, Csr A,
                                                         const double *__restrict__ x, double *__restrict__ cpart) {
    __shared__ double sh[8];
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        int64_t lo = 0, hi = nhub;  // last h with cfirst[h] <= c
        while (hi - lo > 1) {
            int64_t mid = (lo + hi) >> 1;
            if (cfirst[mid] <= c) lo = mid;
            else hi = mid;
        }
        int64_t i = row0 + lo;
        int64_t s = A.rp[i] + (c - cfirst[lo]) * HUB_CHUNK;
        int64_t e = min(A.rp[i + 1], s + HUB_CHUNK);
        double acc = 0.0;
#pragma unroll 4
        for (int64_t k = s + threadIdx.x; k < e; k += blockDim.x) acc += __ldg(&A.w[k]) * x[__ldg(&A.col[k])];
        double r = block_sum(acc, sh);
        if (threadIdx.x == 0) cpart[c] = r;
    }
}
template <int EPI>
__global__ void k_spmv_hub_epi(int64_t nhub, int64_t row0, const int64_t *__restrict__ cfirst,
                               const double *__restrict__ cpart, Csr A, EpiArgs a, double *__restrict__ partials) {
    __shared__ double sh[8];
    double dacc = 0.0;
    for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < nhub; h += (int64_t)gridDim.x * blockDim.x) {
        double ax = 0.0;
        for (int64_t c = cfirst[h]; c < cfirst[h + 1]; c++) ax += cpart[c];
        apply_epi<EPI>(row0 + h, ax, A, a, dacc);
    }
    if (EPI == E_DOT) {
        double r = block_sum(dacc, sh);
        if (threadIdx.x == 0) partials[blockIdx.x] = r;
    }
}

// launch geometry per class (fixed for a level -> deterministic partial slots)
static unsigned class_grid(const Level &L, int c) {
    int64_t lo = c == 0 ? 0 : L.c_end[c - 1];
    int64_t cnt = L.c_end[c] - lo;
    if (cnt <= 0) return 0;
    switch (c) {
        case 0: return grid_for(L.nslices * 32, 256, 148 * 16);
        case 1: return grid_for(cnt * 32, 256, 148 * 8);
        case 2: return (unsigned)std::min<int64_t>(cnt, 148 * 8);
        default: return grid_for(cnt, 256, 148);
    }
}

int64_t spmv_partial_slots(const Level &L) {
    int64_t t = 0;
    for (int c = 0; c < NCLASS; c++) t += class_grid(L, c);
    return t;
}

template <int EPI>
static void spmv_dispatch(lap_hierarchy *h, const Level &L, const EpiArgs &a, cudaStream_t s) {
    Csr A{L.srp, L.scol, L.sw, L.sd};
    double *part = a.partials;
    int64_t slot = 0;
    for (int c = 0; c < NCLASS; c++) {
        int64_t row0 = c == 0 ? 0 : L.c_end[c - 1];
        int64_t cnt = L.c_end[c] - row0;
        if (cnt <= 0) continue;
        unsigned g = class_grid(L, c);
        double *pp = part ? part + slot : nullptr;
        switch (c) {
            case 0: k_spmv_sell<EPI><<<g, 256, 0, s>>>(L.nslices, cnt, L.slice_ptr, L.ell_col, L.ell_w, A, a, pp); break;
            case 1: k_spmv_warp<EPI><<<g, 256, 0, s>>>(cnt, row0, A, a, pp); break;
            case 2: k_spmv_block<EPI><<<g, 256, 0, s>>>(cnt, row0, A, a, pp); break;
            default: {
                unsigned gc = (unsigned)std::min<int64_t>(L.nchunks, 148 * 8);
                k_spmv_hub_chunks<<<gc, 256, 0, s>>>(L.nchunks, cnt, row0, L.chunk_first, A, a.x, L.chunk_part);
                k_spmv_hub_epi<EPI><<<g, 256, 0, s>>>(cnt, row0, L.chunk_first, L.chunk_part, A, a, pp);
                h->cur.launches++;
                break;
            }
        }
        h->cur.launches++;
        slot += g;
    }
    LAP_CHECK_LAUNCH();
}

void spmv_level(lap_hierarchy *h, const Level &L, EpiKind kind, const EpiArgs &a, cudaStream_t s) {
    switch ((int)kind) {
        case E_SPMV: spmv_dispatch<E_SPMV>(h, L, a, s); break;
        case E_DOT: spmv_dispatch<E_DOT>(h, L, a, s); break;
        case E_RESID: spmv_dispatch<E_RESID>(h, L, a, s); break;
        case E_CHEB: spmv_dispatch<E_CHEB>(h, L, a, s); break;
        case E_CHEB0: spmv_dispatch<E_CHEB0>(h, L, a, s); break;
        default: throw Error{LAP_EINVAL, "bad epilogue"};
    }
    int64_t extra = (kind == EPI_RESID) ? 8 : (kind == EPI_CHEB) ? 24 : (kind == (EpiKind)E_CHEB0) ? 16 : 0;
    h->cur.edges += L.nnz;
    h->cur.bytes += 12 * L.nnz + (32 + extra) * L.n;
}

// ------------------------------------------------------------------ reductions
constexpr int RED_BLOCKS = 296;  // fixed: deterministic two-pass reductions

__global__ void __launch_bounds__(256) k_dot_partial(int64_t n, const double *__restrict__ a,
                                                     const double *__restrict__ b, double *__restrict__ part) {
    __shared__ double sh[8];
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += a[i] * (b ? b[i] : 1.0);
    double r = block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = r;
}
__global__ void __launch_bounds__(256) k_reduce_final(const double *__restrict__ part, int64_t np,
                                                      double *__restrict__ out) {
    __shared__ double sh[8];
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < np; i += blockDim.x) acc += part[i];
    double r = block_sum(acc, sh);
    if (threadIdx.x == 0) *out = r;
}

void reduce_partials(lap_hierarchy *h, const double *partials, int64_t np, double *out, cudaStream_t s) {
    k_reduce_final<<<1, 256, 0, s>>>(partials, np, out);
    h->cur.launches++;
    LAP_CHECK_LAUNCH();
}

void dot(lap_hierarchy *h, const double *a, const double *b, int64_t n, double *out, cudaStream_t s) {
    k_dot_partial<<<RED_BLOCKS, 256, 0, s>>>(n, a, b, h->partials);
    h->cur.launches++;
    reduce_partials(h, h->partials, RED_BLOCKS, out, s);
}

// ------------------------------------------------------------------ V-cycle kernels
__global__ void k_cheb_first(int64_t n, const double *__restrict__ b, const double *__restrict__ d, double inv_theta,
                             double *__restrict__ x, double *__restrict__ dv) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double v = (b[i] / d[i]) * inv_theta;
        dv[i] = v;
        x[i] = v;
    }
}
// r_c[a] = sum over members of a (ascending) of r_i; 8 lanes per aggregate
__global__ void __launch_bounds__(256) k_restrict(int64_t m, const int64_t *__restrict__ mp,
                                                  const int32_t *__restrict__ mem, const double *__restrict__ r,
                                                  double *__restrict__ rc) {
    const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = warp * 4; base < m; base += nwarps * 4) {
        int64_t a = base + grp;
        double acc = 0.0;
        if (a < m)
            for (int64_t k = mp[a] + sub; k < mp[a + 1]; k += 8) acc += r[mem[k]];
        for (int o = 4; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (sub == 0 && a < m) rc[a] = acc;
    }
}
__global__ void k_prolong(int64_t n, const int32_t *__restrict__ agg, const double *__restrict__ xc,
                          double *__restrict__ x) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] += xc[agg[i]];
}
// P^T b on an elimination level: b'_k = b_{cid[k]} + sum_{f ~ cid[k]} (w_fc/d_f) b_f
__global__ void k_elim_restrict(int64_t nc, const int32_t *__restrict__ cid, const int64_t *__restrict__ ctp,
                                const int32_t *__restrict__ ctf, const double *__restrict__ ctc,
                                const double *__restrict__ b, double *__restrict__ bc) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nc; k += (int64_t)gridDim.x * blockDim.x) {
        double s = b[cid[k]];
        for (int64_t q = ctp[k]; q < ctp[k + 1]; q++) s += ctc[q] * b[ctf[q]];
        bc[k] = s;
    }
}
// x = P x' + Fsmooth(b): x_c = x'_idx(c); x_f = (b_f + sum_c w_fc x'_idx(c)) / d_f
// (storage order: cid_s maps coarse -> fine row, flist lists F rows, fmap_s maps C rows -> coarse)
__global__ void k_elim_prolong(int64_t nc, int64_t nf, const int32_t *__restrict__ cid, const int32_t *__restrict__ flist,
                               const int32_t *__restrict__ fmap, Csr A, const double *__restrict__ b,
                               const double *__restrict__ xc, double *__restrict__ x) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nc + nf; t += (int64_t)gridDim.x * blockDim.x) {
        if (t < nc) {
            x[cid[t]] = xc[t];
        } else {
            int64_t f = flist[t - nc];
            double s = b[f];
            for (int64_t q = A.rp[f]; q < A.rp[f + 1]; q++) s += A.w[q] * xc[fmap[A.col[q]]];
            x[f] = s / A.d[f];
        }
    }
}
// x = L_c^+ b (warp per row)
__global__ void k_coarse_gemv(int64_t n, const double *__restrict__ P, const double *__restrict__ b,
                              double *__restrict__ x) {
    int lane = threadIdx.x & 31;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < n; i += nwarps) {
        double acc = 0.0;
        for (int64_t j = lane; j < n; j += 32) acc += P[i * n + j] * b[j];
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) x[i] = acc;
    }
}

static inline unsigned eg(int64_t n) { return grid_for(n, 256, 148 * 8); }

// x_out = V(l, b)   (Alg. 1, gamma = 1; elimination levels exact, O-S7)
static void vcycle_rec(lap_hierarchy *h, int l, const double *b, double *xout, cudaStream_t s) {
    Level &L = h->lev[l];
    int64_t n = L.n;
    if (L.kind == KIND_COARSEST) {
        k_coarse_gemv<<<grid_for(n * 32, 256, 148), 256, 0, s>>>(n, L.pinv_s, b, xout);
        h->cur.launches++;
        LAP_CHECK_LAUNCH();
        return;
    }
    Level &C = h->lev[l + 1];
    if (L.kind == KIND_ELIM) {
        int64_t nc = C.n;
        k_elim_restrict<<<eg(nc), 256, 0, s>>>(nc, L.cid_s, L.ct_ptr_s, L.ct_f_s, L.ct_coef_s, b, C.b);
        h->cur.launches++;
        vcycle_rec(h, l + 1, C.b, C.x, s);
        Csr A{L.srp, L.scol, L.sw, L.sd};
        k_elim_prolong<<<eg(nc + L.nF), 256, 0, s>>>(nc, L.nF, L.cid_s, L.flist, L.fmap_s, A, b, C.x, xout);
        h->cur.launches++;
        h->cur.bytes += 16 * n + 24 * (n - nc) * 4;
        LAP_CHECK_LAUNCH();
        return;
    }
    // aggregation level: degree-K Chebyshev in D^-1 L on [lo, hi] * lambda (O-S6)
    const int K = h->p.cheby_degree;
    const double theta = L.cheb_theta, delta = L.cheb_delta, sigma = L.cheb_sigma;
    double *cur = L.x2, *alt = L.t;  // ping-pong pair, distinct from xout and r
    // pre-smoothing from x = 0
    k_cheb_first<<<eg(n), 256, 0, s>>>(n, b, L.sd, 1.0 / theta, cur, L.dv);
    h->cur.launches++;
    h->cur.bytes += 32 * n;
    double rho_old = 1.0 / sigma;
    EpiArgs a;
    a.b = b;
    a.dv = L.dv;
    for (int k = 1; k < K; k++) {
        double rho = 1.0 / (2.0 * sigma - rho_old);
        a.c1 = rho * rho_old;
        a.c2 = 2.0 * rho / delta;
        a.x = cur;
        a.y = alt;
        spmv_level(h, L, EPI_CHEB, a, s);
        std::swap(cur, alt);
        rho_old = rho;
    }
    // residual + restriction (H3)
    a.x = cur;
    a.y = L.r;
    spmv_level(h, L, EPI_RESID, a, s);
    k_restrict<<<grid_for(L.m * 8, 256, 148 * 8), 256, 0, s>>>(L.m, L.mem_ptr, L.members, L.r, C.b);
    h->cur.launches++;
    h->cur.bytes += 16 * n + 8 * L.m;
    vcycle_rec(h, l + 1, C.b, C.x, s);
    // prolongation x += P x_c (H4)
    k_prolong<<<eg(n), 256, 0, s>>>(n, L.agg_s, C.x, cur);
    h->cur.launches++;
    h->cur.bytes += 20 * n + 8 * L.m;
    // post-smoothing from the corrected x
    rho_old = 1.0 / sigma;
    for (int k = 0; k < K; k++) {
        double *dst = (k == K - 1) ? xout : alt;
        a.x = cur;
        a.y = dst;
        if (k == 0) {
            a.c1 = 0.0;
            a.c2 = 1.0 / theta;
            spmv_level(h, L, (EpiKind)E_CHEB0, a, s);
        } else {
            double rho = 1.0 / (2.0 * sigma - rho_old);
            a.c1 = rho * rho_old;
            a.c2 = 2.0 * rho / delta;
            spmv_level(h, L, EPI_CHEB, a, s);
            rho_old = rho;
        }
        if (k < K - 1) std::swap(cur, alt);
    }
}

void vcycle(lap_hierarchy *h, int l, cudaStream_t s) {
    Level &L = h->lev[l];
    vcycle_rec(h, l, L.b, L.x, s);
}

// exposed for lap_vcycle / PCG: z = V(0, r)
void vcycle_apply(lap_hierarchy *h, const double *r, double *z, cudaStream_t s) { vcycle_rec(h, 0, r, z, s); }

// ------------------------------------------------------------------ PCG kernels
// scal layout: 0 rho, 1 pq, 2 rr, 3 sum(z), 4 rho_new, 5 bnorm2, 6 tmp
__global__ void __launch_bounds__(256) k_pcg_xr(int64_t n, const double *__restrict__ p, const double *__restrict__ q,
                                                double *__restrict__ x, double *__restrict__ r,
                                                const double *__restrict__ sc, double *__restrict__ part) {
    __shared__ double sh[8];
    double alpha = sc[0] / sc[1];
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        x[i] += alpha * p[i];
        double ri = r[i] - alpha * q[i];
        r[i] = ri;
        acc += ri * ri;
    }
    double t = block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}
// z -= mean(z) ; partial r.z
__global__ void __launch_bounds__(256) k_pcg_proj_dot(int64_t n, double *__restrict__ z, const double *__restrict__ r,
                                                      const double *__restrict__ sc, double *__restrict__ part) {
    __shared__ double sh[8];
    double mean = sc[3] / (double)n;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double zi = z[i] - mean;
        z[i] = zi;
        acc += r[i] * zi;
    }
    double t = block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}
// p = z + (rho_new/rho) p ; rho = rho_new  (last block updates the scalar after all read it: done by k_pcg_rho)
__global__ void k_pcg_p(int64_t n, const double *__restrict__ z, double *__restrict__ p, const double *__restrict__ sc,
                        int first) {
    double beta = first ? 0.0 : sc[4] / sc[0];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = first ? z[i] : z[i] + beta * p[i];  // first: p is uninitialised (0*NaN must not leak)
}
__global__ void k_copy_scalar(double *sc, int dst, int src) { sc[dst] = sc[src]; }
__global__ void k_sub_mean(int64_t n, double *__restrict__ v, const double *__restrict__ sum) {
    double mean = *sum / (double)n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] -= mean;
}

static double read_scalar(lap_hierarchy *h, const double *dptr, cudaStream_t s) {
    LAP_CUDA(cudaMemcpyAsync(h->host_scal, dptr, sizeof(double), cudaMemcpyDeviceToHost, s));
    LAP_CUDA(cudaStreamSynchronize(s));
    return h->host_scal[0];
}

void launch_vcycle(lap_hierarchy *h, cudaStream_t s);

// PCG on the internal numbering: h->pb holds b' (projected); result in h->px  (O-S8)
void run_pcg(lap_hierarchy *h, double tol, int32_t *iters, double *relres, int *conv, cudaStream_t s) {
    Level &L0 = h->lev[0];
    int64_t n = L0.n;
    double *sc = h->scal;
    unsigned g = RED_BLOCKS;
    *conv = 0;
    h->stats.vcycles = 0;
    dot(h, h->pb, h->pb, n, sc + 5, s);
    double bn = std::sqrt(read_scalar(h, sc + 5, s));
    LAP_CUDA(cudaMemsetAsync(h->px, 0, sizeof(double) * n, s));
    if (bn == 0.0) {
        *iters = 0;
        *relres = 0.0;
        *conv = 1;
        return;
    }
    LAP_CUDA(cudaMemcpyAsync(h->pr, h->pb, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    // z = V(r); project; rho = r.z; p = z
    launch_vcycle(h, s);
    h->stats.vcycles++;
    dot(h, h->pz, nullptr, n, sc + 3, s);
    k_pcg_proj_dot<<<g, 256, 0, s>>>(n, h->pz, h->pr, sc, h->partials);
    reduce_partials(h, h->partials, g, sc + 0, s);
    k_pcg_p<<<eg(n), 256, 0, s>>>(n, h->pz, h->pp, sc, 1);
    h->cur.launches += 2;
    int64_t slots = spmv_partial_slots(L0);
    int k;
    for (k = 1; k <= h->p.max_iters; k++) {
        // q = L p ; pq = p.q   (H1 fused with H7)
        EpiArgs a;
        a.x = h->pp;
        a.y = h->pq;
        a.partials = h->partials;
        spmv_level(h, L0, EPI_SPMV_DOT, a, s);
        reduce_partials(h, h->partials, slots, sc + 1, s);
        // x += alpha p ; r -= alpha q ; rr = r.r
        k_pcg_xr<<<g, 256, 0, s>>>(n, h->pp, h->pq, h->px, h->pr, sc, h->partials);
        h->cur.launches++;
        reduce_partials(h, h->partials, g, sc + 2, s);
        double rr = read_scalar(h, sc + 2, s);
        if (std::sqrt(rr) / bn <= tol) {  // O-R30: confirm with the true residual
            EpiArgs t;
            t.x = h->px;
            t.b = h->pb;
            t.y = h->pq;
            spmv_level(h, L0, EPI_RESID, t, s);
            dot(h, h->pq, h->pq, n, sc + 6, s);
            double tr = read_scalar(h, sc + 6, s);
            if (std::sqrt(tr) / bn <= tol) {
                *conv = 1;
                break;
            }
            LAP_CUDA(cudaMemcpyAsync(h->pr, h->pq, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
        }
        // z = V(r) ; z -= mean z ; rho' = r.z ; p = z + (rho'/rho) p
        launch_vcycle(h, s);
        h->stats.vcycles++;
        dot(h, h->pz, nullptr, n, sc + 3, s);
        k_pcg_proj_dot<<<g, 256, 0, s>>>(n, h->pz, h->pr, sc, h->partials);
        reduce_partials(h, h->partials, g, sc + 4, s);
        k_pcg_p<<<eg(n), 256, 0, s>>>(n, h->pz, h->pp, sc, 0);
        k_copy_scalar<<<1, 1, 0, s>>>(sc, 0, 4);
        h->cur.launches += 3;
        LAP_CHECK_LAUNCH();
    }
    if (!*conv) k = h->p.max_iters;
    *iters = k;
    // x -= mean(x) ; true relative residual
    dot(h, h->px, nullptr, n, sc + 3, s);
    k_sub_mean<<<eg(n), 256, 0, s>>>(n, h->px, sc + 3);
    h->cur.launches++;
    EpiArgs t;
    t.x = h->px;
    t.b = h->pb;
    t.y = h->pq;
    spmv_level(h, L0, EPI_RESID, t, s);
    dot(h, h->pq, h->pq, n, sc + 6, s);
    *relres = std::sqrt(read_scalar(h, sc + 6, s)) / bn;
}

}  // namespace lap
