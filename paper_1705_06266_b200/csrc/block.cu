// block.cu -- many right-hand sides at once.
//
// k independent PCG solves (O-S8 per column: same projection, stopping rule,
// iteration count per column) advanced in lockstep so every pass over a
// level's matrix serves all k vectors: the SpMV becomes an SpMM with the k
// values of a row stored contiguously (row-major n x K block vectors, K the
// compile-time width >= k, unused columns zero).  A gather of x_j then reads
// K*8 contiguous bytes -- for K = 4 one 32-byte sector, the same sector count
// as the single-vector gather -- so the matrix and index bytes (12 per
// stored entry) and the gather sectors are amortised over K solves:
//   bytes per nnz * rhs ~ 12/K + 8 (vs 12 + 8 per nnz for one vector).
// The V-cycle is the single-vector one (solve.cu cycle_rec, V mode, per-level
// path) with every kernel widened to K columns; the Chebyshev coefficients
// are level constants, so all columns share them.  Columns that have
// converged are frozen (alpha = beta = 0 for them) so each column's x and
// iteration count are those of its own solve.  The V-cycle of the block is
// captured once per (hierarchy, K) as a CUDA graph.
#include "lap_internal.cuh"

#include <cmath>
#include <vector>

namespace lap {

constexpr int BLK_RED = 296;  // fixed reduction geometry (deterministic)

__device__ __forceinline__ double blk_block_sum(double v, double *sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double r = 0.0;
    if (wid == 0) {
        r = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    }
    return r;  // thread 0
}

template <int K>
struct Vk {
    double v[K];
};
template <int K>
__device__ __forceinline__ Vk<K> ldk(const double *p) {  // K contiguous doubles (8K-byte aligned rows)
    Vk<K> r;
    if (K % 4 == 0) {  // 256-bit loads (LDG.E.ENL2.256 on sm_100): one request per 32 bytes
#pragma unroll
        for (int c = 0; c < K; c += 4)
            asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                : "=d"(r.v[c]), "=d"(r.v[c + 1]), "=d"(r.v[c + 2]), "=d"(r.v[c + 3])
                : "l"(p + c));
    } else if (K % 2 == 0) {
#pragma unroll
        for (int c = 0; c < K; c += 2) {
            double2 t = __ldg((const double2 *)(p + c));
            r.v[c] = t.x;
            r.v[c + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int c = 0; c < K; c++) r.v[c] = __ldg(p + c);
    }
    return r;
}

template <int K>
__device__ __forceinline__ void stk(double *p, const Vk<K> &v) {
    if (K % 2 == 0) {
#pragma unroll
        for (int c = 0; c < K; c += 2) *(double2 *)(p + c) = make_double2(v.v[c], v.v[c + 1]);
    } else {
#pragma unroll
        for (int c = 0; c < K; c++) p[c] = v.v[c];
    }
}

enum { BE_DOT = 0, BE_RESID = 1, BE_CHEB = 2, BE_CHEB0 = 3 };
struct BArgs {
    const double *x;
    double *y;
    const double *b;
    double *dv;
    double c1, c2;
    double *partials;  // BE_DOT: [K][grid]
};

struct BChunks {  // the level's LCHUNK chunks of its long rows (storage.cu), K partials per chunk
    int64_t nchunks;
    const int32_t *crow, *cidx, *cslot;
    int32_t *ccnt;
    double *cpart;  // [nchunks][K]
    int64_t nmulti;  // rows of several chunks: their BE_DOT terms [nmulti][K] in mdot (see blk_dot_fixup)
    double *mdot;
    int *mdone;
};
// the last block to finish adds the multi-chunk rows' dot terms (slot order) to
// the last block's partial of every column: bitwise reproducible (solve.cu dot_fixup)
template <int K>
__device__ __forceinline__ void blk_dot_fixup(const BChunks &R, double *__restrict__ partials, double *sh) {
    if (R.nmulti == 0) return;
    __shared__ int last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(R.mdone, 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int c = 0; c < K; c++) {
        double acc = 0.0;
        for (int64_t q = threadIdx.x; q < R.nmulti; q += blockDim.x) acc += __ldcg(&R.mdot[q * K + c]);
        const double r = blk_block_sum(acc, sh);
        if (threadIdx.x == 0) {
            double *p = partials + (int64_t)c * gridDim.x + gridDim.x - 1;
            *p = __ldcg(p) + r;
        }
    }
    if (threadIdx.x == 0) *R.mdone = 0;
}

// y = epilogue(L X) for a block of K columns, ONE launch: SELL-32 slices of
// the short rows (coalesced index/weight loads, a thread per row), then the
// LCHUNK-entry warp chunks of the long rows (lane-strided, shuffle tree, K
// chunk partials, the last-arriving chunk of a row sums them in chunk order
// -- the single-vector kernel's scheme, solve.cu chunk_reduce).
template <int EPI, int K>
__global__ void __launch_bounds__(256) k_blk_spmv(int64_t nslices, int64_t nshort, int64_t n,
                                                  const int64_t *__restrict__ sp, const int32_t *__restrict__ ec,
                                                  const double *__restrict__ ew, const int64_t *__restrict__ rp,
                                                  const int32_t *__restrict__ col, const double *__restrict__ w,
                                                  const double *__restrict__ d, BChunks R, BArgs a) {
    pdl_begin();
    __shared__ double sh[8];
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double dacc[K];
#pragma unroll
    for (int c = 0; c < K; c++) dacc[c] = 0.0;
    // row epilogue: the K values of a row are contiguous -> 16-byte vector loads / stores
    auto epi = [&](int64_t i, const double *ax, int slot = -1) {
        const double di = d[i];
        const Vk<K> xi = ldk<K>(a.x + i * K);
        Vk<K> bi, dvi, yo, dvo;
        if (EPI != BE_DOT) bi = ldk<K>(a.b + i * K);
        if (EPI == BE_CHEB) dvi = ldk<K>(a.dv + i * K);
#pragma unroll
        for (int c = 0; c < K; c++) {
            const double lx = di * xi.v[c] - ax[c];
            if (EPI == BE_DOT) {
                yo.v[c] = lx;
                if (slot >= 0) R.mdot[(int64_t)slot * K + c] = xi.v[c] * lx;
                else dacc[c] += xi.v[c] * lx;
            } else if (EPI == BE_RESID) {
                yo.v[c] = bi.v[c] - lx;
            } else if (EPI == BE_CHEB) {
                dvo.v[c] = a.c1 * dvi.v[c] + a.c2 * ((bi.v[c] - lx) / di);
                yo.v[c] = xi.v[c] + dvo.v[c];
            } else {  // BE_CHEB0
                dvo.v[c] = a.c2 * ((bi.v[c] - lx) / di);
                yo.v[c] = xi.v[c] + dvo.v[c];
            }
        }
        stk<K>(a.y + i * K, yo);
        if (EPI == BE_CHEB || EPI == BE_CHEB0) stk<K>(a.dv + i * K, dvo);
    };
    for (int64_t t = warp; t < nslices + R.nchunks; t += nwarps) {
        if (t < nslices) {
            const int64_t i = t * 32 + lane, beg = sp[t], end = sp[t + 1];
            const int width = (int)((end - beg) >> 5);
            double ax[K];
#pragma unroll
            for (int c = 0; c < K; c++) ax[c] = 0.0;
            constexpr int NB = 4;  // padded columns per batch: indices first, then the gathers
            for (int q = 0; q < width; q += NB) {
                int32_t j[NB];
                double wv[NB];
#pragma unroll
                for (int u = 0; u < NB; u++) {
                    j[u] = 0;
                    wv[u] = 0.0;
                    if (q + u < width) {
                        j[u] = __ldg(&ec[beg + (int64_t)(q + u) * 32 + lane]);
                        wv[u] = __ldg(&ew[beg + (int64_t)(q + u) * 32 + lane]);
                    }
                }
#pragma unroll
                for (int u = 0; u < NB; u++) {
                    if (q + u < width) {
                        const Vk<K> xj = ldk<K>(a.x + (int64_t)j[u] * K);
#pragma unroll
                        for (int c = 0; c < K; c++) ax[c] += wv[u] * xj.v[c];
                    }
                }
            }
            if (i < nshort) epi(i, ax);
        } else {
            const int64_t ch = t - nslices;
            const int64_t i = R.crow[ch], j = R.cidx[ch];
            const int64_t rb = rp[i], re = rp[i + 1], b0 = rb + j * LCHUNK, e0 = min(re, b0 + LCHUNK);
            double ax[K];
#pragma unroll
            for (int c = 0; c < K; c++) ax[c] = 0.0;
            for (int64_t q = b0 + lane; q < e0; q += 32) {
                const double wv = __ldg(&w[q]);
                const Vk<K> xj = ldk<K>(a.x + (int64_t)__ldg(&col[q]) * K);
#pragma unroll
                for (int c = 0; c < K; c++) ax[c] += wv * xj.v[c];
            }
#pragma unroll
            for (int c = 0; c < K; c++)
                for (int o = 16; o > 0; o >>= 1) ax[c] += __shfl_xor_sync(0xffffffffu, ax[c], o);
            const int slot = R.cslot[ch];
            if (slot < 0) {  // the whole row in one chunk
                if (lane == 0) epi(i, ax);
                continue;
            }
            const int nch = (int)((re - rb + LCHUNK - 1) / LCHUNK);
            int last = 0;
            if (lane == 0) {
#pragma unroll
                for (int c = 0; c < K; c++) R.cpart[ch * K + c] = ax[c];
                __threadfence();
                last = atomicAdd(&R.ccnt[slot], 1) == nch - 1;
            }
            last = __shfl_sync(0xffffffffu, last, 0);
            if (!last) continue;
            __threadfence();
            if (lane == 0) {  // chunk order, per column
                const int64_t c0 = ch - j;
                double s2[K];
#pragma unroll
                for (int c = 0; c < K; c++) s2[c] = 0.0;
                for (int q = 0; q < nch; q++)
#pragma unroll
                    for (int c = 0; c < K; c++) s2[c] += __ldcg(&R.cpart[(c0 + q) * K + c]);
                R.ccnt[slot] = 0;
                epi(i, s2, slot);
            }
        }
    }
    if (EPI == BE_DOT) {
#pragma unroll
        for (int c = 0; c < K; c++) {
            double r = blk_block_sum(dacc[c], sh);
            if (threadIdx.x == 0) a.partials[c * gridDim.x + blockIdx.x] = r;
        }
        blk_dot_fixup<K>(R, a.partials, sh);
    }
}

// The same SpMM for K = 16 / 32 columns with the LANES owning the columns
// (K lanes per row, 32 / K rows of a slice at a time): a register array of K
// accumulators per thread and K-wide vector gathers would spill, while here
// every x_j gather is ONE coalesced K*8-byte warp access (4 / 8 sectors, all
// bytes used) and each thread keeps one accumulator.  A row's index and
// weight loads are warp-uniform (broadcast; the slice's 128-byte col line
// serves its 32 rows from L1); padded SELL slots (w = 0) skip their gather.
// Per column the products are added in the row's slot order, as in the
// narrow kernel; chunk partials are combined in chunk order.
template <int EPI, int K>
__global__ void __launch_bounds__(256) k_blk_spmv_wide(int64_t nslices, int64_t nshort, int64_t n,
                                                       const int64_t *__restrict__ sp, const int32_t *__restrict__ ec,
                                                       const double *__restrict__ ew, const int64_t *__restrict__ rp,
                                                       const int32_t *__restrict__ col, const double *__restrict__ w,
                                                       const double *__restrict__ d, BChunks R, BArgs a) {
    static_assert(K == 16 || K == 32, "wide SpMM: K = 16 or 32");
    constexpr int RPW = 32 / K;  // rows of a slice per warp pass
    pdl_begin();
    __shared__ double shd[8][32];
    const int lane = threadIdx.x & 31, c = lane & (K - 1), sub = lane / K;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double dacc = 0.0;
    auto epi = [&](int64_t i, double ax, int slot = -1) {  // column c of row i
        const double di = d[i], xi = a.x[i * K + c];
        const double lx = di * xi - ax;
        if (EPI == BE_DOT) {
            a.y[i * K + c] = lx;
            if (slot >= 0) R.mdot[(int64_t)slot * K + c] = xi * lx;
            else dacc += xi * lx;
        } else if (EPI == BE_RESID) {
            a.y[i * K + c] = a.b[i * K + c] - lx;
        } else {
            const double r = (a.b[i * K + c] - lx) / di;
            const double dvo = EPI == BE_CHEB ? a.c1 * a.dv[i * K + c] + a.c2 * r : a.c2 * r;
            a.dv[i * K + c] = dvo;
            a.y[i * K + c] = xi + dvo;
        }
    };
    for (int64_t t = warp; t < nslices + R.nchunks; t += nwarps) {
        if (t < nslices) {
            const int64_t beg = sp[t];
            const int width = (int)((sp[t + 1] - beg) >> 5);
            for (int r0 = 0; r0 < 32; r0 += RPW) {
                const int r = r0 + sub;
                const int64_t i = t * 32 + r;
                double ax = 0.0;
                for (int q = 0; q < width; q += 8) {
                    int32_t jj[8];
                    double wv[8];
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        jj[u] = 0;
                        wv[u] = 0.0;
                        if (q + u < width) {
                            jj[u] = __ldg(&ec[beg + (int64_t)(q + u) * 32 + r]);
                            wv[u] = __ldg(&ew[beg + (int64_t)(q + u) * 32 + r]);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 8; u++)
                        if (wv[u] != 0.0) ax += wv[u] * __ldg(a.x + (int64_t)jj[u] * K + c);
                }
                if (i < nshort) epi(i, ax);
            }
        } else {
            const int64_t ch = t - nslices;
            const int64_t i = R.crow[ch], j = R.cidx[ch];
            const int64_t rb = rp[i], re = rp[i + 1], b0 = rb + j * LCHUNK, e0 = min(re, b0 + LCHUNK);
            double ax = 0.0;
            for (int64_t q0 = b0; q0 < e0; q0 += 32) {
                const int cnt = (int)min((int64_t)32, e0 - q0);
                const int32_t cl = lane < cnt ? __ldg(&col[q0 + lane]) : 0;
                const double wl = lane < cnt ? __ldg(&w[q0 + lane]) : 0.0;
#pragma unroll
                for (int v = 0; v < 32 / RPW; v++) {  // entry v * RPW + sub of this batch
                    const int u = v * RPW + sub;
                    const int32_t jj = __shfl_sync(0xffffffffu, cl, u);
                    const double ww = __shfl_sync(0xffffffffu, wl, u);
                    if (u < cnt) ax += ww * __ldg(a.x + (int64_t)jj * K + c);
                }
            }
            if (RPW == 2) ax += __shfl_xor_sync(0xffffffffu, ax, 16);
            const int slot = R.cslot[ch];
            if (slot < 0) {  // the whole row in one chunk
                if (lane < K) epi(i, ax);
                continue;
            }
            const int nch = (int)((re - rb + LCHUNK - 1) / LCHUNK);
            if (lane < K) R.cpart[ch * K + c] = ax;
            __threadfence();
            __syncwarp();
            int last = 0;
            if (lane == 0) last = atomicAdd(&R.ccnt[slot], 1) == nch - 1;
            last = __shfl_sync(0xffffffffu, last, 0);
            if (!last) continue;
            __threadfence();
            if (lane < K) {  // chunk order, per column
                const int64_t c0 = ch - j;
                double s2 = 0.0;
                for (int q = 0; q < nch; q++) s2 += __ldcg(&R.cpart[(c0 + q) * K + c]);
                epi(i, s2, slot);
            }
            __syncwarp();
            if (lane == 0) R.ccnt[slot] = 0;
        }
    }
    if (EPI == BE_DOT) {
        if (RPW == 2) dacc += __shfl_xor_sync(0xffffffffu, dacc, 16);
        const int wid = threadIdx.x >> 5;
        if (lane < K) shd[wid][c] = dacc;
        __syncthreads();
        if (threadIdx.x < K) {
            double r = 0.0;
            for (int q = 0; q < (int)(blockDim.x >> 5); q++) r += shd[q][threadIdx.x];
            a.partials[threadIdx.x * gridDim.x + blockIdx.x] = r;
        }
        __shared__ double shf[8];
        blk_dot_fixup<K>(R, a.partials, shf);
    }
}

template <int K>
__global__ void k_blk_cheb_first(int64_t n, const double *__restrict__ b, const double *__restrict__ d,
                                 double inv_theta, double *__restrict__ x, double *__restrict__ dv) {
    pdl_begin();
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * K; t += (int64_t)gridDim.x * blockDim.x) {
        double v = (b[t] / d[t / K]) * inv_theta;
        dv[t] = v;
        x[t] = v;
    }
}
// a thread per (aggregate, column); aggregates of more than RESTRICT_SHORT
// members (hubs) are left to k_blk_restrict_big
template <int K>
__global__ void k_blk_restrict(int64_t m, const int64_t *__restrict__ mp, const int32_t *__restrict__ mem,
                               const double *__restrict__ r, double *__restrict__ rc) {
    pdl_begin();
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m * K; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = t / K;
        const int c = (int)(t - a * K);
        if (mp[a + 1] - mp[a] > RESTRICT_SHORT) continue;
        double acc = 0.0;
        for (int64_t q = mp[a]; q < mp[a + 1]; q++) acc += r[(int64_t)mem[q] * K + c];
        rc[t] = acc;
    }
}
// hub aggregates: a block per aggregate (the first chunk of each in the level's
// restriction chunk list), threads strided over its members, column sums by a
// fixed-order block reduction
template <int K>
__global__ void __launch_bounds__(256) k_blk_restrict_big(int64_t nchunks, const int32_t *__restrict__ crow,
                                                          const int32_t *__restrict__ cidx,
                                                          const int64_t *__restrict__ mp,
                                                          const int32_t *__restrict__ mem,
                                                          const double *__restrict__ r, double *__restrict__ rc) {
    pdl_begin();
    __shared__ double sh[8][K];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        if (cidx[ch] != 0) continue;  // uniform over the block
        const int64_t a = crow[ch];
        double acc[K];
#pragma unroll
        for (int c = 0; c < K; c++) acc[c] = 0.0;
        for (int64_t q = mp[a] + threadIdx.x; q < mp[a + 1]; q += blockDim.x) {
            const double *rr = r + (int64_t)mem[q] * K;
#pragma unroll
            for (int c = 0; c < K; c++) acc[c] += rr[c];
        }
#pragma unroll
        for (int c = 0; c < K; c++) {
            double v = acc[c];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) sh[wid][c] = v;
        }
        __syncthreads();
        if (threadIdx.x < K) {
            double v = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); w++) v += sh[w][threadIdx.x];
            rc[a * K + threadIdx.x] = v;
        }
        __syncthreads();
    }
}
template <int K>
__global__ void k_blk_prolong(int64_t n, const int32_t *__restrict__ agg, const double *__restrict__ xc,
                              double *__restrict__ x) {
    pdl_begin();
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * K; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / K;
        x[t] += xc[(int64_t)agg[i] * K + (t - i * K)];
    }
}
template <int K>
__global__ void k_blk_elim_restrict(int64_t nc, const int32_t *__restrict__ cid, const int64_t *__restrict__ ctp,
                                    const int32_t *__restrict__ ctf, const double *__restrict__ ctc,
                                    const double *__restrict__ b, double *__restrict__ bc) {
    pdl_begin();
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nc * K; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t / K;
        const int c = (int)(t - k * K);
        double s = b[(int64_t)cid[k] * K + c];
        for (int64_t q = ctp[k]; q < ctp[k + 1]; q++) s += ctc[q] * b[(int64_t)ctf[q] * K + c];
        bc[t] = s;
    }
}
template <int K>
__global__ void k_blk_elim_prolong(int64_t nc, int64_t nf, const int32_t *__restrict__ cid,
                                   const int32_t *__restrict__ flist, const int32_t *__restrict__ fmap,
                                   const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                                   const double *__restrict__ w, const double *__restrict__ d,
                                   const double *__restrict__ b, const double *__restrict__ xc,
                                   double *__restrict__ x) {
    pdl_begin();
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (nc + nf) * K;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = t / K;
        const int c = (int)(t - u * K);
        if (u < nc) {
            x[(int64_t)cid[u] * K + c] = xc[t];
        } else {
            const int64_t f = flist[u - nc];
            double s = b[f * K + c];
            for (int64_t q = rp[f]; q < rp[f + 1]; q++) s += w[q] * xc[(int64_t)fmap[col[q]] * K + c];
            x[f * K + c] = s / d[f];
        }
    }
}
template <int K>
__global__ void k_blk_coarse(int64_t n, const double *__restrict__ P, const double *__restrict__ b,
                             double *__restrict__ x) {
    pdl_begin();
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < n; i += nwarps) {
        double acc[K];
#pragma unroll
        for (int c = 0; c < K; c++) acc[c] = 0.0;
        for (int64_t j = lane; j < n; j += 32) {
            const double p = P[i * n + j];
#pragma unroll
            for (int c = 0; c < K; c++) acc[c] += p * b[j * K + c];
        }
#pragma unroll
        for (int c = 0; c < K; c++) {
            for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
            if (lane == 0) x[i * K + c] = acc[c];
        }
    }
}

// ---- per-column PCG vector operations (scalars: sc[16 * c + slot])
//   slots: 0 rho, 1 pq, 2 rr, 3 sum z, 4 active (1/0), 5 ||b||^2, 6 sum r, 7 beta
template <int K, int NS>
__global__ void __launch_bounds__(256) k_blk_sums(int64_t n, const double *__restrict__ a0, const double *__restrict__ a1,
                                                  const double *__restrict__ a2, double *__restrict__ part) {
    // NS = 1: sum a0*a1 ; NS = 3: sum a0, sum a0*a1, sum a1 (z, r) ; per column
    pdl_begin();
    __shared__ double sh[8];
    double s0[K], s1[K], s2[K];
#pragma unroll
    for (int c = 0; c < K; c++) s0[c] = s1[c] = s2[c] = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int c = 0; c < K; c++) {
            const double x0 = a0[i * K + c], x1 = a1 ? a1[i * K + c] : 1.0;
            if (NS == 1) {
                s0[c] += x0 * x1;
            } else {
                s0[c] += x0;
                s1[c] += x0 * x1;
                s2[c] += x1;
            }
        }
    }
#pragma unroll
    for (int c = 0; c < K; c++) {
        double t0 = blk_block_sum(s0[c], sh);
        if (threadIdx.x == 0) part[(NS * c) * gridDim.x + blockIdx.x] = t0;
        if (NS == 3) {
            double t1 = blk_block_sum(s1[c], sh), t2 = blk_block_sum(s2[c], sh);
            if (threadIdx.x == 0) {
                part[(NS * c + 1) * gridDim.x + blockIdx.x] = t1;
                part[(NS * c + 2) * gridDim.x + blockIdx.x] = t2;
            }
        }
    }
}
// reduce nv groups of np partials each; group g -> column g / per, slot sl[g % per]
__global__ void k_blk_reduce(const double *__restrict__ part, int np, int nv, int per, double *__restrict__ sc, int s0,
                             int s1, int s2) {
    pdl_begin();
    __shared__ double sh[8];
    for (int g = 0; g < nv; g++) {
        double acc = 0.0;
        for (int i = threadIdx.x; i < np; i += blockDim.x) acc += part[(int64_t)g * np + i];
        double r = blk_block_sum(acc, sh);
        const int j = g % per;
        if (threadIdx.x == 0) sc[16 * (g / per) + (j == 0 ? s0 : j == 1 ? s1 : s2)] = r;
    }
}
// per column: rho' = r.(z - mean z) = r.z - mean(z) sum r ; beta = rho'/rho (0 first / frozen)
template <int K>
__global__ void k_blk_zfinish(int64_t n, double *__restrict__ sc, int first) {
    pdl_begin();
    const int c = threadIdx.x;
    if (c >= K) return;
    double *s = sc + 16 * c;
    const double rho_new = s[8] - (s[3] / (double)n) * s[6];
    s[7] = (first || s[4] == 0.0) ? 0.0 : rho_new / s[0];
    s[0] = rho_new;
}
template <int K>
__global__ void k_blk_p(int64_t n, const double *__restrict__ z, double *__restrict__ p, const double *__restrict__ sc,
                        int first) {
    pdl_begin();
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * K; t += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(t % K);
        const double *s = sc + 16 * c;
        const double zm = z[t] - s[3] / (double)n;
        p[t] = first ? zm : zm + s[7] * p[t];
    }
}
// x += alpha p ; r -= alpha q (active columns) ; partial r.r
template <int K>
__global__ void __launch_bounds__(256) k_blk_xr(int64_t n, const double *__restrict__ p, const double *__restrict__ q,
                                                double *__restrict__ x, double *__restrict__ r,
                                                const double *__restrict__ sc, double *__restrict__ part) {
    pdl_begin();
    __shared__ double sh[8];
    double alpha[K], acc[K];
#pragma unroll
    for (int c = 0; c < K; c++) {
        const double *s = sc + 16 * c;
        alpha[c] = (s[4] != 0.0 && s[1] != 0.0) ? s[0] / s[1] : 0.0;
        acc[c] = 0.0;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int c = 0; c < K; c++) {
            x[i * K + c] += alpha[c] * p[i * K + c];
            const double ri = r[i * K + c] - alpha[c] * q[i * K + c];
            r[i * K + c] = ri;
            acc[c] += ri * ri;
        }
    }
#pragma unroll
    for (int c = 0; c < K; c++) {
        double t = blk_block_sum(acc[c], sh);
        if (threadIdx.x == 0) part[c * gridDim.x + blockIdx.x] = t;
    }
}
// K >= 16: the same sums and update with a thread per ELEMENT of the n x K
// block (coalesced; the grid stride is a multiple of K, so a thread always
// serves column threadIdx.x % K) and a fixed-order per-column combine of the
// block's 256 / K threads -- a register array of K (or 3K) partials per thread
// would hold 100-250 registers
template <int K>
__device__ __forceinline__ double blk_col_sum(double v, double *sh) {  // -> threads 0..K-1: column sums
    __syncthreads();
    sh[threadIdx.x] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x < K)
        for (int q = threadIdx.x; q < (int)blockDim.x; q += K) r += sh[q];
    return r;
}
template <int K, int NS>
__global__ void __launch_bounds__(256) k_blk_sums_w(int64_t n, const double *__restrict__ a0,
                                                    const double *__restrict__ a1, const double *__restrict__ a2,
                                                    double *__restrict__ part) {
    pdl_begin();
    __shared__ double sh[256];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * K; t += (int64_t)gridDim.x * blockDim.x) {
        const double x0 = a0[t], x1 = a1 ? a1[t] : 1.0;
        if (NS == 1) {
            s0 += x0 * x1;
        } else {
            s0 += x0;
            s1 += x0 * x1;
            s2 += x1;
        }
    }
    const int c = threadIdx.x;
    double r = blk_col_sum<K>(s0, sh);
    if (c < K) part[(NS * c) * gridDim.x + blockIdx.x] = r;
    if (NS == 3) {
        r = blk_col_sum<K>(s1, sh);
        if (c < K) part[(NS * c + 1) * gridDim.x + blockIdx.x] = r;
        r = blk_col_sum<K>(s2, sh);
        if (c < K) part[(NS * c + 2) * gridDim.x + blockIdx.x] = r;
    }
}
template <int K>
__global__ void __launch_bounds__(256) k_blk_xr_w(int64_t n, const double *__restrict__ p,
                                                  const double *__restrict__ q, double *__restrict__ x,
                                                  double *__restrict__ r, const double *__restrict__ sc,
                                                  double *__restrict__ part) {
    pdl_begin();
    __shared__ double sh[256];
    const double *s = sc + 16 * (threadIdx.x % K);
    const double alpha = (s[4] != 0.0 && s[1] != 0.0) ? s[0] / s[1] : 0.0;
    double acc = 0.0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * K; t += (int64_t)gridDim.x * blockDim.x) {
        x[t] += alpha * p[t];
        const double ri = r[t] - alpha * q[t];
        r[t] = ri;
        acc += ri * ri;
    }
    const double v = blk_col_sum<K>(acc, sh);
    if (threadIdx.x < K) part[threadIdx.x * gridDim.x + blockIdx.x] = v;
}
// caller layout (n x k column-major, caller numbering) <-> block layout (storage order, row-major n x K)
template <int K>
__global__ void k_blk_in(int64_t n, int k, const int64_t *__restrict__ cmap, const double *__restrict__ B,
                         double *__restrict__ out) {
    pdl_begin();
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * K; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / K;
        const int c = (int)(t - i * K);
        out[cmap[i] * K + c] = c < k ? B[(int64_t)c * n + i] : 0.0;
    }
}
template <int K>
__global__ void k_blk_out(int64_t n, int k, const int64_t *__restrict__ cmap, const double *__restrict__ in,
                          const double *__restrict__ sc, double *__restrict__ X) {
    pdl_begin();
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * k; t += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(t / n);
        const int64_t i = t - (int64_t)c * n;
        X[t] = in[cmap[i] * K + c] - sc[16 * c + 3] / (double)n;  // x -= mean x (per column)
    }
}
template <int K>
__global__ void k_blk_sub_mean(int64_t n, double *__restrict__ v, const double *__restrict__ sc, int slot) {
    pdl_begin();
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * K; t += (int64_t)gridDim.x * blockDim.x)
        v[t] -= sc[16 * (t % K) + slot] / (double)n;
}

// ------------------------------------------------------------------ host
struct BlockWork {  // per (hierarchy, K)
    int K = 0;
    std::vector<double *> lb, lx, lx2, lt, lr, ldv;  // per level, n_l x K
    std::vector<double *> lcpart;                     // per level, K partials per long-row chunk
    std::vector<double *> lmdot;                      // per level, K dot terms per multi-chunk row
    int *mdone = nullptr;                             // blk_dot_fixup arrival counter (kept at 0)
    double *b = nullptr, *x = nullptr, *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr;
    double *sc = nullptr, *part = nullptr;
    double *hsc = nullptr;  // pinned host copy of the scalars
    cudaGraphExec_t vgraph = nullptr;
    Stats vcounts;
};

static inline unsigned beg(int64_t n) { return grid_for(n, 256, 148 * 8); }

template <int K>
static void blk_spmv(lap_hierarchy *h, const Level &L, double *cpart, double *mdot, int *mdone, int epi,
                     const BArgs &a, cudaStream_t s, unsigned grid) {
    BChunks R{L.nchunks, L.chunk_row, L.chunk_idx, L.chunk_slot, L.chunk_cnt, cpart, L.nmulti, mdot, mdone};
#define BLK_LAUNCH(E)                                                                                             \
    launch_pdl(K >= 16 ? k_blk_spmv_wide<E, (K >= 16 ? K : 16)> : k_blk_spmv<E, K>, grid, 256, s, L.nslices,      \
               L.c_end[0], L.n, (const int64_t *)L.slice_ptr,                                                     \
               (const int32_t *)L.ell_col, (const double *)L.ell_w, (const int64_t *)L.srp,                       \
               (const int32_t *)L.scol, (const double *)L.sw, (const double *)L.sd, R, a)
    switch (epi) {
        case BE_DOT: BLK_LAUNCH(BE_DOT); break;
        case BE_RESID: BLK_LAUNCH(BE_RESID); break;
        case BE_CHEB: BLK_LAUNCH(BE_CHEB); break;
        default: BLK_LAUNCH(BE_CHEB0); break;
    }
#undef BLK_LAUNCH
    h->cur.launches++;
    h->cur.edges += L.nnz * K;
    h->cur.bytes += 12 * L.nnz + (int64_t)(8 * K) * L.nnz + (int64_t)(40 * K) * L.n;
}
template <int K>
static unsigned spmm_grid(const Level &L) {
    return grid_for((L.nslices + L.nchunks) * 32, 256, 148 * 8);
}

// V-cycle on K columns (solve.cu cycle_rec, V mode, per-level kernels)
template <int K>
static void blk_vcycle(lap_hierarchy *h, BlockWork &W, int l, const double *b, double *xout, cudaStream_t s) {
    Level &L = h->lev[l];
    const int64_t n = L.n;
    if (L.kind == KIND_COARSEST) {
        launch_pdl(k_blk_coarse<K>, grid_for(n * 32, 256, 148), 256, s, n, (const double *)L.pinv_s, b, xout);
        h->cur.launches++;
        return;
    }
    Level &C = h->lev[l + 1];
    double *cb = W.lb[l + 1], *cx = W.lx[l + 1];
    if (L.kind == KIND_ELIM) {
        launch_pdl(k_blk_elim_restrict<K>, beg(C.n * K), 256, s, C.n, (const int32_t *)L.cid_s,
                   (const int64_t *)L.ct_ptr_s, (const int32_t *)L.ct_f_s, (const double *)L.ct_coef_s, b, cb);
        blk_vcycle<K>(h, W, l + 1, cb, cx, s);
        launch_pdl(k_blk_elim_prolong<K>, beg((C.n + L.nF) * K), 256, s, C.n, L.nF, (const int32_t *)L.cid_s,
                   (const int32_t *)L.flist, (const int32_t *)L.fmap_s, (const int64_t *)L.srp,
                   (const int32_t *)L.scol, (const double *)L.sw, (const double *)L.sd, b, (const double *)cx, xout);
        h->cur.launches += 2;
        return;
    }
    const int Kd = h->p.cheby_degree;
    const double theta = L.cheb_theta, delta = L.cheb_delta, sigma = L.cheb_sigma;
    double *cur = W.lx2[l], *alt = W.lt[l];
    const unsigned g = spmm_grid<K>(L);
    launch_pdl(k_blk_cheb_first<K>, beg(n * K), 256, s, n, b, (const double *)L.sd, 1.0 / theta, cur, W.ldv[l]);
    h->cur.launches++;
    double rho_old = 1.0 / sigma;
    BArgs a{};
    a.b = b;
    a.dv = W.ldv[l];
    for (int k = 1; k < Kd; k++) {
        double rho = 1.0 / (2.0 * sigma - rho_old);
        a.c1 = rho * rho_old;
        a.c2 = 2.0 * rho / delta;
        a.x = cur;
        a.y = alt;
        blk_spmv<K>(h, L, W.lcpart[l], W.lmdot[l], W.mdone, BE_CHEB, a, s, g);
        std::swap(cur, alt);
        rho_old = rho;
    }
    a.x = cur;
    a.y = W.lr[l];
    blk_spmv<K>(h, L, W.lcpart[l], W.lmdot[l], W.mdone, BE_RESID, a, s, g);
    launch_pdl(k_blk_restrict<K>, beg(L.m * K), 256, s, L.m, (const int64_t *)L.mem_ptr, (const int32_t *)L.members,
               (const double *)W.lr[l], cb);
    if (L.rs_nchunks > 0) {
        launch_pdl(k_blk_restrict_big<K>, grid_for(L.rs_nchunks, 1, 148 * 4), 256, s, L.rs_nchunks,
                   (const int32_t *)L.rs_crow, (const int32_t *)L.rs_cidx, (const int64_t *)L.mem_ptr,
                   (const int32_t *)L.members, (const double *)W.lr[l], cb);
        h->cur.launches++;
    }
    blk_vcycle<K>(h, W, l + 1, cb, cx, s);
    launch_pdl(k_blk_prolong<K>, beg(n * K), 256, s, n, (const int32_t *)L.agg_s, (const double *)cx, cur);
    h->cur.launches += 2;
    rho_old = 1.0 / sigma;
    for (int k = 0; k < Kd; k++) {
        double *dst = (k == Kd - 1) ? xout : alt;
        a.x = cur;
        a.y = dst;
        if (k == 0) {
            a.c1 = 0.0;
            a.c2 = 1.0 / theta;
            blk_spmv<K>(h, L, W.lcpart[l], W.lmdot[l], W.mdone, BE_CHEB0, a, s, g);
        } else {
            double rho = 1.0 / (2.0 * sigma - rho_old);
            a.c1 = rho * rho_old;
            a.c2 = 2.0 * rho / delta;
            blk_spmv<K>(h, L, W.lcpart[l], W.lmdot[l], W.mdone, BE_CHEB, a, s, g);
            rho_old = rho;
        }
        if (k < Kd - 1) std::swap(cur, alt);
    }
}

template <int K>
static BlockWork *block_work(lap_hierarchy *h, cudaStream_t s) {
    std::vector<void *> &cache = h->blk;
    for (void *p : cache)
        if (((BlockWork *)p)->K == K) return (BlockWork *)p;
    BlockWork *W = new BlockWork();
    W->K = K;
    for (auto &L : h->lev) {
        const size_t bytes = 8 * (size_t)K * (size_t)(L.n > 0 ? L.n : 1);
        W->lb.push_back((double *)dalloc(bytes, s));
        W->lx.push_back((double *)dalloc(bytes, s));
        W->lx2.push_back((double *)dalloc(bytes, s));
        W->lt.push_back((double *)dalloc(bytes, s));
        W->lr.push_back((double *)dalloc(bytes, s));
        W->ldv.push_back((double *)dalloc(bytes, s));
        W->lcpart.push_back((double *)dalloc(8 * (size_t)K * (size_t)(L.nchunks > 0 ? L.nchunks : 1), s));
        W->lmdot.push_back((double *)dalloc(8 * (size_t)K * (size_t)(L.nmulti > 0 ? L.nmulti : 1), s));
    }
    const size_t b0 = 8 * (size_t)K * (size_t)h->lev[0].n;
    double **vs[] = {&W->b, &W->x, &W->r, &W->z, &W->p, &W->q};
    for (double **v : vs) *v = (double *)dalloc(b0, s);
    W->sc = (double *)dalloc(8 * 16 * K, s);
    W->mdone = (int *)dalloc(sizeof(int), s);
    LAP_CUDA(cudaMemsetAsync(W->mdone, 0, sizeof(int), s));
    int64_t np = BLK_RED;
    for (auto &L : h->lev) np = std::max<int64_t>(np, (int64_t)spmm_grid<K>(L));
    W->part = (double *)dalloc(8 * 3 * K * (size_t)np, s);
    LAP_CUDA(cudaMallocHost(&W->hsc, 8 * 16 * K));
    // the block V-cycle as one graph
    cudaStream_t cs;
    LAP_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    LAP_CUDA(cudaStreamSynchronize(s));
    Stats save = h->cur;
    h->cur = Stats{};
    cudaGraph_t g;
    LAP_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    blk_vcycle<K>(h, *W, 0, W->r, W->z, cs);
    LAP_CUDA(cudaStreamEndCapture(cs, &g));
    W->vcounts = h->cur;
    h->cur = save;
    LAP_CUDA(cudaGraphInstantiate(&W->vgraph, g, 0));
    LAP_CUDA(cudaGraphDestroy(g));
    LAP_CUDA(cudaStreamDestroy(cs));
    cache.push_back(W);
    return W;
}

void free_block(lap_hierarchy *h) {
    for (void *p : h->blk) {
        BlockWork *W = (BlockWork *)p;
        if (W->vgraph) cudaGraphExecDestroy(W->vgraph);
        for (auto *v : {&W->lb, &W->lx, &W->lx2, &W->lt, &W->lr, &W->ldv, &W->lcpart, &W->lmdot})
            for (double *q : *v) dfree(q, nullptr);
        for (double *q : {W->b, W->x, W->r, W->z, W->p, W->q, W->sc, W->part}) dfree(q, nullptr);
        dfree(W->mdone, nullptr);
        if (W->hsc) cudaFreeHost(W->hsc);
        delete W;
    }
    h->blk.clear();
}

template <int K>
static void blk_launch_vcycle(lap_hierarchy *h, BlockWork &W, cudaStream_t s) {
    LAP_CUDA(cudaGraphLaunch(W.vgraph, s));
    h->cur.launches += W.vcounts.launches;
    h->cur.edges += W.vcounts.edges;
    h->cur.bytes += W.vcounts.bytes;
}

// per-column scalar slots (sc[16 c + slot]):
enum { S_RHO = 0, S_PQ = 1, S_RR = 2, S_SUMZ = 3, S_ACTIVE = 4, S_BB = 5, S_SUMR = 6, S_BETA = 7, S_RZ = 8,
       S_TMP = 9, S_TRUE = 10 };

template <int K, int NS>
static void blk_sums(lap_hierarchy *h, BlockWork &W, const double *a0, const double *a1, int s0, int s1, int s2,
                     cudaStream_t s) {
    const int64_t n = h->lev[0].n;
    if constexpr (K >= 16)
        launch_pdl(k_blk_sums_w<K, NS>, BLK_RED, 256, s, n, a0, a1, (const double *)nullptr, W.part);
    else
        launch_pdl(k_blk_sums<K, NS>, BLK_RED, 256, s, n, a0, a1, (const double *)nullptr, W.part);
    launch_pdl(k_blk_reduce, 1, 256, s, (const double *)W.part, BLK_RED, NS * K, NS, W.sc, s0, s1, s2);
    h->cur.launches += 2;
}

// z = V(r) ; z -= mean z ; rho' = r.z ; p = z + (rho'/rho) p   (O-S8, per column)
template <int K>
static void blk_precond(lap_hierarchy *h, BlockWork &W, bool first, cudaStream_t s) {
    const int64_t n = h->lev[0].n;
    blk_launch_vcycle<K>(h, W, s);
    blk_sums<K, 3>(h, W, W.z, W.r, S_SUMZ, S_RZ, S_SUMR, s);
    launch_pdl(k_blk_zfinish<K>, 1, 32, s, n, W.sc, first ? 1 : 0);
    launch_pdl(k_blk_p<K>, beg(n * K), 256, s, n, (const double *)W.z, W.p, (const double *)W.sc, first ? 1 : 0);
    h->cur.launches += 2;
}
// q = L p ; pq ; x += alpha p ; r -= alpha q ; rr
template <int K>
static void blk_spmv_part(lap_hierarchy *h, BlockWork &W, cudaStream_t s) {
    const Level &L0 = h->lev[0];
    const int64_t n = L0.n;
    const unsigned g = spmm_grid<K>(L0);
    BArgs a{};
    a.x = W.p;
    a.y = W.q;
    a.partials = W.part;
    blk_spmv<K>(h, L0, W.lcpart[0], W.lmdot[0], W.mdone, BE_DOT, a, s, g);
    launch_pdl(k_blk_reduce, 1, 256, s, (const double *)W.part, (int)g, K, 1, W.sc, (int)S_PQ, 0, 0);
    if constexpr (K >= 16)
        launch_pdl(k_blk_xr_w<K>, BLK_RED, 256, s, n, (const double *)W.p, (const double *)W.q, W.x, W.r,
                   (const double *)W.sc, W.part);
    else
        launch_pdl(k_blk_xr<K>, BLK_RED, 256, s, n, (const double *)W.p, (const double *)W.q, W.x, W.r,
               (const double *)W.sc, W.part);
    launch_pdl(k_blk_reduce, 1, 256, s, (const double *)W.part, BLK_RED, K, 1, W.sc, (int)S_RR, 0, 0);
    h->cur.launches += 3;
}
template <int K>
__global__ void k_blk_copy_cols(int64_t n, const double *__restrict__ src, double *__restrict__ dst,
                                const double *__restrict__ sc) {
    pdl_begin();  // columns with sc[S_TMP] != 0
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * K; t += (int64_t)gridDim.x * blockDim.x)
        if (sc[16 * (t % K) + S_TMP] != 0.0) dst[t] = src[t];
}

template <int K>
static void solve_block_k(lap_hierarchy *h, int k, const double *B, double *X, double tol, int32_t *iters,
                          double *relres, int *conv, cudaStream_t s) {
    BlockWork &W = *block_work<K>(h, s);
    const Level &L0 = h->lev[0];
    const int64_t n = L0.n;
    const int maxit = h->p.max_iters;
    double *hs = W.hsc;
    auto pull = [&]() {
        LAP_CUDA(cudaMemcpyAsync(hs, W.sc, 8 * 16 * K, cudaMemcpyDeviceToHost, s));
        LAP_CUDA(cudaStreamSynchronize(s));
    };
    auto push = [&]() { LAP_CUDA(cudaMemcpyAsync(W.sc, hs, 8 * 16 * K, cudaMemcpyHostToDevice, s)); };
    // b' = Pi b per column, projected; x = 0 ; r = b
    launch_pdl(k_blk_in<K>, beg(n * K), 256, s, n, k, (const int64_t *)h->cmap, B, W.b);
    h->cur.launches++;
    blk_sums<K, 1>(h, W, W.b, nullptr, S_TMP, 0, 0, s);
    launch_pdl(k_blk_sub_mean<K>, beg(n * K), 256, s, n, W.b, (const double *)W.sc, (int)S_TMP);
    h->cur.launches++;
    blk_sums<K, 1>(h, W, W.b, W.b, S_BB, 0, 0, s);
    LAP_CUDA(cudaMemsetAsync(W.x, 0, 8 * (size_t)K * n, s));
    LAP_CUDA(cudaMemcpyAsync(W.r, W.b, 8 * (size_t)K * n, cudaMemcpyDeviceToDevice, s));
    pull();
    std::vector<double> bn(K);
    int nactive = 0;
    for (int c = 0; c < K; c++) {
        bn[c] = std::sqrt(hs[16 * c + S_BB]);
        const bool act = c < k && bn[c] > 0.0;
        hs[16 * c + S_ACTIVE] = act ? 1.0 : 0.0;
        if (c < k) iters[c] = 0;
        nactive += act;
    }
    push();
    int it = 0;
    if (nactive) {
        blk_precond<K>(h, W, true, s);
        for (it = 1; it <= maxit; it++) {
            blk_spmv_part<K>(h, W, s);
            pull();
            bool check = false;
            for (int c = 0; c < K; c++)
                if (hs[16 * c + S_ACTIVE] != 0.0 && std::sqrt(hs[16 * c + S_RR]) / bn[c] <= tol) check = true;
            if (check) {  // O-R30: confirm with the true residual b - L x (into z: free until the next V-cycle)
                BArgs t{};
                t.x = W.x;
                t.b = W.b;
                t.y = W.z;
                blk_spmv<K>(h, L0, W.lcpart[0], W.lmdot[0], W.mdone, BE_RESID, t, s, spmm_grid<K>(L0));
                blk_sums<K, 1>(h, W, W.z, W.z, S_TRUE, 0, 0, s);
                pull();
                bool any_bad = false;
                for (int c = 0; c < K; c++) {
                    hs[16 * c + S_TMP] = 0.0;
                    if (hs[16 * c + S_ACTIVE] == 0.0 || !(std::sqrt(hs[16 * c + S_RR]) / bn[c] <= tol)) continue;
                    if (std::sqrt(hs[16 * c + S_TRUE]) / bn[c] <= tol) {
                        hs[16 * c + S_ACTIVE] = 0.0;  // converged: frozen from here on
                        iters[c] = it;
                        nactive--;
                    } else {
                        hs[16 * c + S_TMP] = 1.0;  // restart this column from its true residual
                        any_bad = true;
                    }
                }
                push();
                if (any_bad) {
                    launch_pdl(k_blk_copy_cols<K>, beg(n * K), 256, s, n, (const double *)W.z, W.r, (const double *)W.sc);
                    h->cur.launches++;
                }
            }
            if (nactive == 0 || it == maxit) break;
            blk_precond<K>(h, W, false, s);
            LAP_CHECK_LAUNCH();
        }
    }
    *conv = nactive == 0 ? 1 : 0;
    for (int c = 0; c < k; c++)
        if (hs[16 * c + S_ACTIVE] != 0.0) iters[c] = it < maxit ? it : maxit;
    // x -= mean x (per column, in k_blk_out) ; true relative residuals
    blk_sums<K, 1>(h, W, W.x, nullptr, S_SUMZ, 0, 0, s);
    BArgs t{};
    t.x = W.x;
    t.b = W.b;
    t.y = W.z;
    blk_spmv<K>(h, L0, W.lcpart[0], W.lmdot[0], W.mdone, BE_RESID, t, s, spmm_grid<K>(L0));
    blk_sums<K, 1>(h, W, W.z, W.z, S_TRUE, 0, 0, s);
    launch_pdl(k_blk_out<K>, beg(n * k), 256, s, n, k, (const int64_t *)h->cmap, (const double *)W.x,
               (const double *)W.sc, X);
    h->cur.launches++;
    pull();
    for (int c = 0; c < k; c++) relres[c] = bn[c] > 0.0 ? std::sqrt(hs[16 * c + S_TRUE]) / bn[c] : 0.0;
}

// k right-hand sides (1 <= k <= 32), device buffers in the caller's layout: B, X n x k column-major
// LAP_BLOCK_WIDE=1: every k > 8 on the lane-per-column SpMM (K = 16 / 32),
// the round-2 routing before column groups (tests, measurements)
static bool wide_forced() {
    const char *e = getenv("LAP_BLOCK_WIDE");
    return e && e[0] == '1';
}
void solve_block(lap_hierarchy *h, int k, const double *B, double *X, double tol, int32_t *iters, double *relres,
                 int *conv, cudaStream_t s) {
    if (k <= 2) solve_block_k<2>(h, k, B, X, tol, iters, relres, conv, s);
    else if (k <= 4) solve_block_k<4>(h, k, B, X, tol, iters, relres, conv, s);
    else if (k <= 8) solve_block_k<8>(h, k, B, X, tol, iters, relres, conv, s);
    else if (wide_forced()) {
        if (k <= 16) solve_block_k<16>(h, k, B, X, tol, iters, relres, conv, s);
        else solve_block_k<32>(h, k, B, X, tol, iters, relres, conv, s);
    } else if (k <= 16 || 10 * h->lev[0].n > h->lev[0].nnz) {
        // blocks of <= 8 columns one after the other: the thread-per-row K = 8
        // SpMM moves 8x the bytes per gather instruction of the lane-per-column
        // K = 16 one (measured 2.13x vs 1.66x the throughput of k single solves
        // on cfg 4, 1.71x vs 1.35x on cfg 2); past 16 columns K = 32 wins only
        // where the matrix bytes it shares dominate (>= 10 entries per row:
        // cfg 3 2.88x vs 2.03x) -- on mesh-like levels vectors dominate (cfg 2
        // K = 32 1.41x vs 1.71x)
        const int64_t n = h->lev[0].n;
        int all = 1;
        for (int c0 = 0; c0 < k; c0 += 8) {
            const int kc = k - c0 < 8 ? k - c0 : 8;
            int c = 0;
            if (kc <= 2) solve_block_k<2>(h, kc, B + c0 * n, X + c0 * n, tol, iters + c0, relres + c0, &c, s);
            else if (kc <= 4) solve_block_k<4>(h, kc, B + c0 * n, X + c0 * n, tol, iters + c0, relres + c0, &c, s);
            else solve_block_k<8>(h, kc, B + c0 * n, X + c0 * n, tol, iters + c0, relres + c0, &c, s);
            all = all && c;
        }
        *conv = all;
    } else {
        solve_block_k<32>(h, k, B, X, tol, iters, relres, conv, s);
    }
}

}  // namespace lap
