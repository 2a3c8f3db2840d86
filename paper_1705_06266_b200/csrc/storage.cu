// storage.cu -- the B200 solve-phase data layout.
//
// The method fixes each level's LOGICAL vertex ids (random order at level 0,
// P:371-376; aggregates by ascending root; C vertices order-preserving,
// O-R22).  Those ids are what the oracle sees and they stay bit-identical.
// The solve phase, however, is HBM/L2 bound, so each level is additionally
// stored in a STORAGE ORDER designed for sm_100a:
//   * rows grouped by degree class so each SpMV schedule (SELL-32 slices,
//     warp per row, block per row, split hub rows) is a contiguous range;
//   * within a class, rows ordered by a locality key inherited from the
//     caller's numbering (level 0 undoes Pi_rand; an aggregate takes the
//     smallest storage position of its members; a C vertex keeps its fine
//     position), so x-gathers of neighbouring rows share cache lines.
// A storage order is a symmetric permutation of L_l: it changes no value of
// the method, only the order in which the GPU sums (solve parity is by
// tolerance, O-P2).
#include <cub/cub.cuh>

#include <algorithm>
#include <string>
#include <vector>

#include "canon.cuh"
#include "lap_internal.cuh"

namespace lap {

static bool getenv_flag_off(const char *name) {
    const char *e = getenv(name);
    return e && e[0] == '0';
}

template <class T>
static T d2h(const T *p, cudaStream_t s) {
    T v;
    LAP_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, s));
    LAP_CUDA(cudaStreamSynchronize(s));
    return v;
}

#define GRID_STRIDE(i, n) for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

__global__ void k_key_level0(int64_t n, const int64_t *perm, uint64_t *key) {
    GRID_STRIDE(c, n) key[perm[c]] = (uint64_t)c;  // logical id perm[c] <- caller id c
}
__global__ void k_key_fill(int64_t n, uint64_t v, uint64_t *key) {
    GRID_STRIDE(i, n) key[i] = v;
}
__global__ void k_key_agg(int64_t nf, const int32_t *agg, const int32_t *fspos, unsigned long long *key) {
    GRID_STRIDE(i, nf) atomicMin(&key[agg[i]], (unsigned long long)fspos[i]);
}
__global__ void k_key_elim(int64_t nc, const int32_t *cid, const int32_t *fspos, uint64_t *key) {
    GRID_STRIDE(k, nc) key[k] = (uint64_t)fspos[cid[k]];
}
__device__ __forceinline__ int deg_class(int64_t dg) {
    return dg <= SHORT_MAX ? 0 : dg <= 1024 ? 1 : dg <= HUB_CHUNK ? 2 : 3;
}
// sort key: [40:39] degree class, [38:31] 255 - degree (short rows, only if
// degree-sorted), [30:0] locality key (< n < 2^31)
__global__ void k_class_key(int64_t n, const int64_t *rp, const uint64_t *key, uint64_t *skey, int32_t *ids,
                            unsigned long long *cnt, int by_degree, int hub_order) {
    GRID_STRIDE(i, n) {
        int64_t dg = rp[i + 1] - rp[i];
        int c = deg_class(dg);
        // 41 key bits: 6 radix passes instead of 8
        // hub_order: rows beyond SELL by descending degree within their class (the
        // most referenced x entries contiguous)
        const uint64_t loc = (hub_order && c > 0) ? (uint64_t)(0x7FFFFFFF - (dg < 0x7FFFFFFF ? dg : 0x7FFFFFFF)) : key[i];
        uint64_t k = loc | (((uint64_t)c) << 39);
        if (by_degree && c == 0) k |= ((uint64_t)(255 - dg)) << 31;
        skey[i] = k;
        ids[i] = (int32_t)i;
        if (cnt) {  // warp-aggregated class counts (one atomic per class per warp, not per row)
            const unsigned am = __activemask();
            for (int q = 0; q < NCLASS; q++) {
                unsigned m = __ballot_sync(am, c == q);
                if (m && (threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(&cnt[q], (unsigned long long)__popc(m));
            }
            // cnt[NCLASS]: entries of the short class (the SELL padding baseline)
            unsigned sd = __reduce_add_sync(am, c == 0 ? (unsigned)dg : 0u);  // <= 32 * 64
            if ((threadIdx.x & 31) == __ffs(am) - 1 && sd) atomicAdd(&cnt[NCLASS], (unsigned long long)sd);
        }
    }
}
// SELL-32 slice widths (max degree of the slice's rows) and padding statistic
__global__ void k_slice_width(int64_t nslices, int64_t nshort, const int32_t *sid, const int64_t *rp, int64_t *width,
                              unsigned long long *padded) {
    GRID_STRIDE(sl, nslices) {
        int64_t mx = 0;
        for (int64_t p = sl * 32; p < min(nshort, sl * 32 + 32); p++) {
            int64_t i = sid[p];
            mx = max(mx, rp[i + 1] - rp[i]);
        }
        width[sl] = 32 * mx;
        atomicAdd(padded, (unsigned long long)(32 * mx));
    }
}
// fill every slot of every slice, including the lanes past the last short row
// of a ragged final slice (col 0, w 0: gathered but contribute nothing)
__global__ void k_sell_fill(int64_t nslots, int64_t nshort, const int64_t *srp, const int32_t *scol, const double *sw,
                            const int64_t *slice_ptr, int32_t *ell_col, double *ell_w) {
    GRID_STRIDE(p, nslots) {
        int64_t sl = p >> 5, lane = p & 31;
        int64_t base = slice_ptr[sl] + lane, width = (slice_ptr[sl + 1] - slice_ptr[sl]) >> 5;
        bool row = p < nshort;
        int64_t a = row ? srp[p] : 0, dg = row ? srp[p + 1] - a : 0;
        for (int64_t k = 0; k < width; k++) {
            bool real = k < dg;
            ell_col[base + 32 * k] = real ? scol[a + k] : (row ? (int32_t)p : 0);
            ell_w[base + 32 * k] = real ? sw[a + k] : 0.0;
        }
    }
}
// SELL-C-sigma: re-sort the short rows by degree only WITHIN windows of sigma
// consecutive rows of the current (class, locality) order, keeping the gather
// locality of the order while cutting the slice padding.  Key = window << 9 |
// (255 - degree), class 0 rows only (the rest keep their position).
__global__ void k_window_key(int64_t n, int64_t nshort, int64_t sigma, const int32_t *sid, const int64_t *rp,
                             uint64_t *skey, int32_t *ids) {
    GRID_STRIDE(p, n) {
        const int32_t i = sid[p];
        uint64_t k;
        if (p < nshort) k = ((uint64_t)(p / sigma) << 9) | (uint64_t)(255 - (rp[i + 1] - rp[i]));
        else k = ((uint64_t)(nshort / sigma + 1 + p) << 9);  // long rows: unchanged order after the short ones
        skey[p] = k;
        ids[p] = i;
    }
}
__global__ void k_inverse(int64_t n, const int32_t *sid, int32_t *spos) {
    GRID_STRIDE(p, n) spos[sid[p]] = (int32_t)p;
}
__global__ void k_storage_deg(int64_t n, const int32_t *sid, const int64_t *rp, const double *d, int64_t *deg,
                              double *sd) {
    GRID_STRIDE(p, n) {
        int64_t i = sid[p];
        deg[p] = rp[i + 1] - rp[i];
        sd[p] = d[i];
    }
}
// copy logical row sid[p] into storage row p, columns translated; entry-
// parallel over the storage entries (hub rows do not serialise).  A block's
// 256 entries span few rows: two full searches per block bound the rows, the
// per-entry search runs inside that range (cfg 5 level 0: 2.1e9 entries)
__global__ void __launch_bounds__(256) k_storage_fill(int64_t n, int64_t nnz, const int32_t *sid, const int32_t *spos,
                                                      const int64_t *rp, const int32_t *col, const double *w,
                                                      const int64_t *srp, int32_t *scol, double *sw) {
    __shared__ int64_t plo, phi;
    for (int64_t b0 = (int64_t)blockIdx.x * 256; b0 < nnz; b0 += (int64_t)gridDim.x * 256) {
        if (threadIdx.x < 2) {
            const int64_t tt = threadIdx.x == 0 ? b0 : min(nnz, b0 + 256) - 1;
            const int64_t r = row_of(srp, n, tt);
            if (threadIdx.x == 0) plo = r;
            else phi = r;
        }
        __syncthreads();
        const int64_t t = b0 + threadIdx.x;
        if (t < nnz) {
            int64_t lo = plo, hi = phi;
            while (lo < hi) {
                const int64_t mid = (lo + hi + 1) >> 1;
                if (srp[mid] <= t) lo = mid;
                else hi = mid - 1;
            }
            const int64_t src = rp[sid[lo]] + (t - srp[lo]);
            scol[t] = spos[col[src]];
            sw[t] = w ? w[src] : 1.0;
        }
        __syncthreads();
    }
}
__global__ void k_to_u16(int64_t m, const int32_t *in, uint16_t *out) {
    GRID_STRIDE(i, m) out[i] = (uint16_t)in[i];
}
// LCHUNK work items over rows [row0, row0+nrows) of a CSR whose length
// exceeds minlen (the others get no chunk); slot = row - row0 for rows of
// several chunks (their arrival counter), -1 for one-chunk rows.
__global__ void k_chunk_counts(int64_t nrows, int64_t row0, const int64_t *rp, int64_t minlen, int64_t *cnt) {
    GRID_STRIDE(h, nrows) {
        int64_t i = row0 + h, dg = rp[i + 1] - rp[i];
        cnt[h] = dg > minlen ? (dg + LCHUNK - 1) / LCHUNK : 0;
    }
}
// slot = the row's index among the rows of several chunks (mpre: prefix of
// "several chunks" flags), so per-row side data (arrival counters, the solve's
// dot terms of such rows) can be compact and summed in slot order
__global__ void k_chunk_multi(int64_t nrows, const int64_t *first, int64_t *mflag) {
    GRID_STRIDE(h, nrows) mflag[h] = first[h + 1] - first[h] > 1 ? 1 : 0;
}
__global__ void k_chunk_fill(int64_t nrows, int64_t row0, const int64_t *first, const int64_t *mpre, int32_t *crow,
                             int32_t *cidx, int32_t *cslot) {
    GRID_STRIDE(h, nrows) {
        int64_t f = first[h], nch = first[h + 1] - f;
        for (int64_t j = 0; j < nch; j++) {
            crow[f + j] = (int32_t)(row0 + h);
            cidx[f + j] = (int32_t)j;
            cslot[f + j] = nch > 1 ? (int32_t)mpre[h] : -1;
        }
    }
}

template <class T>
static void scan_excl(const T *in, T *out, int64_t n, cudaStream_t s) {
    size_t bytes = 0;
    LAP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
    DBuf<char> tmp((int64_t)bytes, s);
    LAP_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, n, s));
    g_kl += 2;
}

// ---------------------------------------------------------------- per-row sorts
// Every row of a CSR sorted by column (rows independent, columns of a row
// distinct), by row length class:
//   <= 32 entries (most rows of every level): one THREAD per row, fused with
//        the permutation -- the row's (column << 8 | slot) words are loaded
//        straight from the source row into registers, sorted by a bitonic
//        network with compile-time indices (no shuffles, no shared memory),
//        and the weights gathered by slot on the way out;
//   33..64: one warp per row, bitonic network over two registers per lane;
//   65..256 / 257..2048: a block radix sort in shared memory (64 x 4 / 256 x 8);
//   > 2048 (hubs): cub's segmented sort over a list of just those rows.
// Replaces one device-wide segmented sort of every row (cfg 4: ~5 ms per
// launch, three per setup) and the emit + 64-bit-key radix sort of the
// level-0 relabel.
constexpr int ROWSORT_MED = 2048;  // 256 threads x 8 entries
constexpr int ROWSORT_SMALL = 256;  // 64 threads x 4 entries
constexpr int ROWSORT_SEG_AVG = 16384;  // long rows: cub segmented sort up to this average length
template <int N>
__device__ __forceinline__ void reg_bitonic(uint64_t (&a)[N]) {
#pragma unroll
    for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
            for (int i = 0; i < N; i++) {
                const int l = i ^ j;
                if (l > i) {
                    const uint64_t x = a[i], y = a[l];
                    const uint64_t mn = x < y ? x : y, mx = x < y ? y : x;
                    if ((i & k) == 0) a[i] = mn, a[l] = mx;
                    else a[i] = mx, a[l] = mn;
                }
            }
        }
    }
}
// rows with LO <= len <= N of P A P^T (new row p = old row sid[p], column c -> spos[c])
template <int N, int LO>
__global__ void __launch_bounds__(256) k_perm_sort_thread(int64_t n, const int32_t *__restrict__ sid,
                                                          const int32_t *__restrict__ spos,
                                                          const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                                                          const double *__restrict__ w, const int64_t *__restrict__ srp,
                                                          int32_t *__restrict__ kout, double *__restrict__ vout) {
    GRID_STRIDE(p, n) {
        const int64_t o = srp[p];
        const int64_t len = srp[p + 1] - o;
        if (len < LO || len > N) continue;
        const int64_t a0 = rp[sid[p]];
        uint64_t a[N];
#pragma unroll
        for (int q = 0; q < N; q++)
            a[q] = q < len ? ((uint64_t)(uint32_t)spos[col[a0 + q]] << 8) | (uint64_t)q : ~0ULL;
        reg_bitonic<N>(a);
#pragma unroll
        for (int q = 0; q < N; q++) {
            if (q < len) {
                kout[o + q] = (int32_t)(a[q] >> 8);
                vout[o + q] = w ? w[a0 + (int64_t)(a[q] & 255u)] : 1.0;
            }
        }
    }
}
// rows longer than minlen copied (columns translated through spos) to their
// output positions: rows of (minlen, maxlen] -> kt / vt (to be sorted); rows
// longer than maxlen and at most band_hi (left unsorted) straight to kbig / vbig
struct PermFill {
    int64_t n, minlen, maxlen, band_hi;
    const int32_t *__restrict__ sid;
    const int32_t *__restrict__ spos;
    const int64_t *__restrict__ rp;
    const int32_t *__restrict__ col;
    const double *__restrict__ w;
    const int64_t *__restrict__ srp;
    int32_t *__restrict__ kt;
    double *__restrict__ vt;
    int32_t *__restrict__ kbig;
    double *__restrict__ vbig;
};
constexpr int64_t PFILL_LONG = 1024;  // longer rows: a CTA each (k_perm_fill_rows)
// row p's entries [q0, len) with stride st: 4 column loads, then their 4 spos
// gathers, in flight per thread
__device__ __forceinline__ void perm_fill_row(const PermFill &A, int64_t p, int64_t o, int64_t len, int64_t q0,
                                              int64_t st) {
    const bool unsorted = len > A.maxlen && len <= A.band_hi;
    int32_t *kd = unsorted ? A.kbig : A.kt;
    double *vd = unsorted ? A.vbig : A.vt;
    const int64_t a0 = A.rp[A.sid[p]];
    int64_t q = q0;
    for (; q + 3 * st < len; q += 4 * st) {
        int32_t c[4];
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            c[u] = A.col[a0 + q + st * u];
            v[u] = A.w ? A.w[a0 + q + st * u] : 1.0;
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            kd[o + q + st * u] = A.spos[c[u]];
            vd[o + q + st * u] = v[u];
        }
    }
    for (; q < len; q += st) {
        kd[o + q] = A.spos[A.col[a0 + q]];
        vd[o + q] = A.w ? A.w[a0 + q] : 1.0;
    }
}
// G lanes per row (G near the average row length: several short rows per warp
// in flight instead of a warp per row with most lanes idle); rows longer than
// PFILL_LONG are listed for k_perm_fill_rows
template <int G>
__global__ void __launch_bounds__(256) k_perm_fill_grp(PermFill A, int32_t *__restrict__ longs,
                                                       int32_t *__restrict__ nlong) {
    GROUP_LOOP_BEGIN(G, A.n)
        const int64_t o = live ? A.srp[i] : 0, len = live ? A.srp[i + 1] - o : 0;
        if (len > PFILL_LONG) {
            if (gl == 0) longs[atomicAdd(nlong, 1)] = (int32_t)i;
        } else if (len > A.minlen) {
            perm_fill_row(A, i, o, len, gl, G);
        }
    GROUP_LOOP_END
}
__global__ void __launch_bounds__(256) k_perm_fill_rows(PermFill A, const int32_t *__restrict__ longs,
                                                        const int32_t *__restrict__ nlong) {
    const int64_t m = *nlong;
    for (int64_t b = blockIdx.x; b < m; b += gridDim.x) {
        const int64_t p = longs[b], o = A.srp[p], len = A.srp[p + 1] - o;
        perm_fill_row(A, p, o, len, threadIdx.x, blockDim.x);
    }
}
static void perm_fill(const PermFill &A, int64_t nnz, cudaStream_t s) {
    if (A.n <= 0) return;
    const double avg = (double)nnz / (double)A.n;
    const int G = avg <= 8.0 ? 4 : avg <= 32.0 ? 8 : avg <= 128.0 ? 16 : 32;
    DBuf<int32_t> longs(nnz / PFILL_LONG + 1, s), nlong(1, s);
    LAP_CUDA(cudaMemsetAsync(nlong.p, 0, sizeof(int32_t), s));
    LAUNCH_G(G, k_perm_fill_grp, A.n, s, A, longs.p, nlong.p);
    k_perm_fill_rows<<<grid_for(nnz / PFILL_LONG + 1, 1, 148 * 4), 256, 0, s>>>(A, longs.p, nlong.p);
    g_kl += 2;
}
template <int NH>
__device__ __forceinline__ void warp_bitonic(int (&k)[2], double (&v)[2], int lane) {
#pragma unroll
    for (int kk = 2; kk <= 32 * NH; kk <<= 1) {
#pragma unroll
        for (int j = kk >> 1; j > 0; j >>= 1) {
            if (j == 32) {  // partner in this lane's other register (kk = 64: ascending)
                if (k[1] < k[0]) {
                    const int tk = k[0];
                    const double tv = v[0];
                    k[0] = k[1], v[0] = v[1];
                    k[1] = tk, v[1] = tv;
                }
                continue;
            }
#pragma unroll
            for (int hh = 0; hh < NH; hh++) {
                const int ok = __shfl_xor_sync(0xffffffffu, k[hh], j);
                const double ov = __shfl_xor_sync(0xffffffffu, v[hh], j);
                const int i = hh * 32 + lane;
                const bool asc = (i & kk) == 0, lower = (lane & j) == 0;
                const bool take = (asc == lower) ? (ok < k[hh]) : (ok > k[hh]);
                if (take) k[hh] = ok, v[hh] = ov;
            }
        }
    }
}
// rows with minlen < len <= 64
__global__ void __launch_bounds__(256) k_rowsort_warp(int64_t n, int64_t minlen, const int64_t *__restrict__ rp,
                                                      const int32_t *__restrict__ kin, const double *__restrict__ vin,
                                                      int32_t *__restrict__ kout, double *__restrict__ vout) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < n; r += nwarps) {
        const int64_t a = rp[r];
        const int64_t len0 = rp[r + 1] - a;
        if (len0 > 64 || len0 <= minlen) continue;
        const int len = (int)len0;
        int k[2];
        double v[2];
#pragma unroll
        for (int hh = 0; hh < 2; hh++) {
            const int q = hh * 32 + lane;
            k[hh] = q < len ? kin[a + q] : INT_MAX;
            v[hh] = q < len ? vin[a + q] : 0.0;
        }
        if (len > 32) warp_bitonic<2>(k, v, lane);
        else if (len > 1) warp_bitonic<1>(k, v, lane);
#pragma unroll
        for (int hh = 0; hh < 2; hh++) {
            const int q = hh * 32 + lane;
            if (q < len) kout[a + q] = k[hh], vout[a + q] = v[hh];
        }
    }
}
__global__ void k_rowsort_lists(int64_t n, const int64_t *__restrict__ rp, int32_t *sml, int32_t *med, int32_t *lng,
                                int *cnt, int64_t sort_max, int32_t *cpy, int64_t band_hi) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t len = rp[r + 1] - rp[r];
        if (len > sort_max && len <= band_hi) cpy[atomicAdd(&cnt[3], 1)] = (int32_t)r;  // kept in the given order
        else if (len > ROWSORT_MED) lng[atomicAdd(&cnt[2], 1)] = (int32_t)r;  // order free: rows are independent
        else if (len > ROWSORT_SMALL) med[atomicAdd(&cnt[1], 1)] = (int32_t)r;
        else if (len > 64) sml[atomicAdd(&cnt[0], 1)] = (int32_t)r;
    }
}
template <int NT, int IPT>
__global__ void __launch_bounds__(NT) k_rowsort_block(int64_t m, const int32_t *__restrict__ list,
                                                      const int64_t *__restrict__ rp, int cbits,
                                                      const int32_t *__restrict__ kin, const double *__restrict__ vin,
                                                      int32_t *__restrict__ kout, double *__restrict__ vout) {
    typedef cub::BlockRadixSort<uint32_t, NT, IPT, double> BRS;
    __shared__ typename BRS::TempStorage ts;
    for (int64_t t = blockIdx.x; t < m; t += gridDim.x) {
        const int64_t r = list[t], a = rp[r];
        const int len = (int)(rp[r + 1] - a);
        uint32_t k[IPT];
        double v[IPT];
#pragma unroll
        for (int u = 0; u < IPT; u++) {  // blocked arrangement: thread t holds entries IPT t .. IPT t + IPT - 1
            const int q = threadIdx.x * IPT + u;
            k[u] = q < len ? (uint32_t)kin[a + q] : 0xFFFFFFFFu;
            v[u] = q < len ? vin[a + q] : 0.0;
        }
        BRS(ts).Sort(k, v, 0, cbits < 32 ? cbits + 1 : 32);  // (padding 0xFFFFFFFF still sorts last)
#pragma unroll
        for (int u = 0; u < IPT; u++) {
            const int q = threadIdx.x * IPT + u;
            if (q < len) kout[a + q] = (int32_t)k[u], vout[a + q] = v[u];
        }
        __syncthreads();
    }
}
__global__ void k_seg_bounds(int64_t m, const int32_t *__restrict__ list, const int64_t *__restrict__ rp,
                             int64_t *__restrict__ beg, int64_t *__restrict__ end) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        beg[t] = rp[list[t]];
        end[t] = rp[list[t] + 1];
    }
}

__global__ void k_seg_len(int64_t m, const int64_t *__restrict__ beg, const int64_t *__restrict__ end,
                          int64_t *__restrict__ len) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
        len[t] = end[t] - beg[t];
}
__global__ void k_long_gather(int64_t B, const int64_t *__restrict__ beg, const int64_t *__restrict__ loff, int cbits,
                              const int32_t *__restrict__ kin, const double *__restrict__ vin, uint64_t *__restrict__ k1,
                              double *__restrict__ v1) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < B; r += nwarps) {
        const int64_t a = beg[r], o = loff[r], len = loff[r + 1] - o;
        for (int64_t q = lane; q < len; q += 32) {
            k1[o + q] = ((uint64_t)r << cbits) | (uint64_t)(uint32_t)kin[a + q];
            v1[o + q] = vin[a + q];
        }
    }
}
__global__ void k_long_scatter(int64_t B, const int64_t *__restrict__ beg, const int64_t *__restrict__ loff, int cbits,
                               const uint64_t *__restrict__ k2, const double *__restrict__ v2, int32_t *__restrict__ kout,
                               double *__restrict__ vout) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t mask = (1ULL << cbits) - 1;
    for (int64_t r = warp; r < B; r += nwarps) {
        const int64_t a = beg[r], o = loff[r], len = loff[r + 1] - o;
        for (int64_t q = lane; q < len; q += 32) {
            kout[a + q] = (int32_t)(k2[o + q] & mask);
            vout[a + q] = v2[o + q];
        }
    }
}
// rows longer than sort_max copied as they are (warp per row)
__global__ void k_rowcopy_list(int64_t m, const int32_t *__restrict__ list, const int64_t *__restrict__ rp,
                               const int32_t *__restrict__ kin, const double *__restrict__ vin,
                               int32_t *__restrict__ kout, double *__restrict__ vout) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = warp; t < m; t += nwarps) {
        const int64_t r = list[t];
        for (int64_t k = rp[r] + lane; k < rp[r + 1]; k += 32) {
            kout[k] = kin[k];
            vout[k] = vin[k];
        }
    }
}
// rows of length > minlen (minlen >= 32) sorted: kin/vin -> kout/vout; rows
// longer than sort_max are copied unsorted
static void sort_rows_min(int64_t n, const int64_t *rp, int64_t nnz, int cbits, int64_t minlen, const int32_t *kin,
                          const double *vin, int32_t *kout, double *vout, cudaStream_t s,
                          int64_t sort_max = INT64_MAX, bool copy_big = true, int64_t band_hi = INT64_MAX) {
    if (n <= 0 || nnz <= 0) return;
    DBuf<int32_t> sml(n, s), med(n, s), lng(n, s), cpy(sort_max < INT64_MAX ? n : 1, s);
    DBuf<int> cnt(4, s);
    LAP_CUDA(cudaMemsetAsync(cnt.p, 0, 4 * sizeof(int), s));
    k_rowsort_lists<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(n, rp, sml.p, med.p, lng.p, cnt.p, sort_max, cpy.p,
                                                              band_hi);
    k_rowsort_warp<<<grid_for(n * 32, 256, 148 * 8), 256, 0, s>>>(n, minlen, rp, kin, vin, kout, vout);
    g_kl += 2;
    trace_mark("    rowsort: lists + warp rows");
    int hc[4];
    LAP_CUDA(cudaMemcpyAsync(hc, cnt.p, sizeof(hc), cudaMemcpyDeviceToHost, s));
    LAP_CUDA(cudaStreamSynchronize(s));
    if (hc[3] > 0 && copy_big) {
        k_rowcopy_list<<<grid_for((int64_t)hc[3] * 32, 256, 148 * 8), 256, 0, s>>>(hc[3], cpy.p, rp, kin, vin, kout,
                                                                                  vout);
        g_kl++;
    }
    if (hc[0] > 0) {
        k_rowsort_block<64, 4><<<grid_for(hc[0], 1, 148 * 16), 64, 0, s>>>(hc[0], sml.p, rp, cbits, kin, vin, kout, vout);
        g_kl++;
    }
    if (hc[1] > 0) {
        k_rowsort_block<256, 8><<<grid_for(hc[1], 1, 148 * 4), 256, 0, s>>>(hc[1], med.p, rp, cbits, kin, vin, kout,
                                                                           vout);
        g_kl++;
    }
    trace_mark("    rowsort: block rows");
    if (hc[2] > 0) {
        // rows longer than ROWSORT_MED (hubs, dense coarse rows): cub's segmented
        // sort over just those rows; when they are few and huge (cub gives a
        // segment to one block), ONE device-wide radix sort of their entries
        // keyed (list index << cbits | column) instead
        const int64_t B = hc[2];
        DBuf<int64_t> beg(B + 1, s), end(B + 1, s), len(B + 1, s), loff(B + 1, s);
        k_seg_bounds<<<grid_for(B, 256, 148 * 4), 256, 0, s>>>(B, lng.p, rp, beg.p, end.p);
        k_seg_len<<<grid_for(B, 256, 148 * 4), 256, 0, s>>>(B, beg.p, end.p, len.p);
        LAP_CUDA(cudaMemsetAsync(len.p + B, 0, sizeof(int64_t), s));
        scan_excl(len.p, loff.p, B + 1, s);
        const int64_t Tl = d2h(loff.p + B, s);
        if (Tl <= (int64_t)ROWSORT_SEG_AVG * B && nnz < ((int64_t)1 << 31)) {
            size_t bytes = 0;
            LAP_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int)nnz, (int)B, beg.p,
                                                         end.p, s));
            DBuf<char> tmp((int64_t)bytes, s);
            LAP_CUDA(cub::DeviceSegmentedSort::SortPairs(tmp.p, bytes, kin, kout, vin, vout, (int)nnz, (int)B, beg.p,
                                                         end.p, s));
            g_kl += 4;
            trace_mark("    rowsort: long rows (cub segmented)");
        } else {
            DBuf<uint64_t> k1(Tl, s), k2(Tl, s);
            DBuf<double> v1(Tl, s), v2(Tl, s);
            k_long_gather<<<grid_for(B * 32, 256, 148 * 8), 256, 0, s>>>(B, beg.p, loff.p, cbits, kin, vin, k1.p, v1.p);
            size_t bytes = 0;
            int lb = 1;
            while (lb < 40 && ((int64_t)1 << lb) <= B) lb++;
            const int end_bit = std::min(64, cbits + lb);
            LAP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k1.p, k2.p, v1.p, v2.p, Tl, 0, end_bit, s));
            DBuf<char> tmp((int64_t)bytes, s);
            LAP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, k1.p, k2.p, v1.p, v2.p, Tl, 0, end_bit, s));
            k_long_scatter<<<grid_for(B * 32, 256, 148 * 8), 256, 0, s>>>(B, beg.p, loff.p, cbits, k2.p, v2.p, kout, vout);
            g_kl += 5;
            trace_mark("    rowsort: long rows (global radix)");
        }
    }
    LAP_CHECK_LAUNCH();
}

void sort_rows(int64_t n, const int64_t *rp, int64_t nnz, int cbits, const int32_t *kin, const double *vin,
               int32_t *kout, double *vout, cudaStream_t s) {
    if (n <= 0 || nnz <= 0) return;
    k_rowsort_warp<<<grid_for(n * 32, 256, 148 * 8), 256, 0, s>>>(n, -1, rp, kin, vin, kout, vout);
    g_kl++;
    sort_rows_min(n, rp, nnz, cbits, 64, kin, vin, kout, vout, s);
}


int64_t build_chunks(const int64_t *rp, int64_t row0, int64_t nrows, int64_t minlen, int32_t **crow,
                            int32_t **cidx, int32_t **cslot, double **cpart, int32_t **ccnt, cudaStream_t s,
                            int64_t *nmulti) {
    if (nmulti) *nmulti = 0;
    if (nrows <= 0) return 0;
    DBuf<int64_t> cc(nrows + 1, s), first(nrows + 1, s);
    LAP_CUDA(cudaMemsetAsync(cc.p, 0, sizeof(int64_t) * (nrows + 1), s));
    k_chunk_counts<<<grid_for(nrows, 256, 148 * 8), 256, 0, s>>>(nrows, row0, rp, minlen, cc.p);
    g_kl++;
    scan_excl(cc.p, first.p, nrows + 1, s);
    int64_t nch = d2h(first.p + nrows, s);
    *crow = (int32_t *)dalloc(sizeof(int32_t) * (nch + 1), s);
    *cidx = (int32_t *)dalloc(sizeof(int32_t) * (nch + 1), s);
    *cslot = (int32_t *)dalloc(sizeof(int32_t) * (nch + 1), s);
    *cpart = (double *)dalloc(sizeof(double) * (nch + 1), s);
    *ccnt = (int32_t *)dalloc(sizeof(int32_t) * nrows, s);
    LAP_CUDA(cudaMemsetAsync(*ccnt, 0, sizeof(int32_t) * nrows, s));
    if (nch > 0) {
        DBuf<int64_t> mflag(nrows + 1, s), mpre(nrows + 1, s);
        LAP_CUDA(cudaMemsetAsync(mflag.p + nrows, 0, sizeof(int64_t), s));
        k_chunk_multi<<<grid_for(nrows, 256, 148 * 8), 256, 0, s>>>(nrows, first.p, mflag.p);
        scan_excl(mflag.p, mpre.p, nrows + 1, s);
        k_chunk_fill<<<grid_for(nrows, 256, 148 * 8), 256, 0, s>>>(nrows, row0, first.p, mpre.p, *crow, *cidx, *cslot);
        g_kl += 2;
        if (nmulti) *nmulti = d2h(mpre.p + nrows, s);
    }
    LAP_CHECK_LAUNCH();
    return nch;
}

__global__ void k_perm_deg(int64_t n, const int32_t *sid, const int64_t *rp, int64_t *deg) {
    GRID_STRIDE(p, n) deg[p] = rp[sid[p] + 1] - rp[sid[p]];
}
void permute_csr(int64_t n, int64_t nnz, const int32_t *sid, const int32_t *spos, const int64_t *rp,
                 const int32_t *col, const double *w, int64_t *srp, int32_t *scol, double *sw, bool sort_cols,
                 int64_t maxlen, cudaStream_t s) {
    DBuf<int64_t> deg(n + 1, s);
    LAP_CUDA(cudaMemsetAsync(deg.p + n, 0, sizeof(int64_t), s));
    if (n > 0) {
        k_perm_deg<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(n, sid, rp, deg.p);
        g_kl++;
    }
    scan_excl(deg.p, srp, n + 1, s);
    if (nnz <= 0) return;
    if (!sort_cols) {  // warp per row (a row's source entries are contiguous): 2.4 -> 1.2 ms on cfg 4 level 0
        perm_fill(PermFill{n, 0, INT64_MAX, INT64_MAX, sid, spos, rp, col, w, srp, scol, sw, nullptr, nullptr}, nnz, s);
        LAP_CHECK_LAUNCH();
        return;
    }
    permute_sorted_rows(n, nnz, sid, spos, rp, col, w, srp, scol, sw, maxlen, s, INT64_MAX);
}
// the rows of P A P^T sorted, srp given
void permute_sorted_rows(int64_t n, int64_t nnz, const int32_t *sid, const int32_t *spos, const int64_t *rp,
                         const int32_t *col, const double *w, const int64_t *srp, int32_t *scol, double *sw,
                         int64_t maxlen, cudaStream_t s, int64_t sort_max, int64_t band_hi) {
    if (n <= 0 || nnz <= 0) return;
    if (sort_max == 0) {  // only the rows longer than band_hi sorted (power-law levels)
        const bool any_long = maxlen > band_hi;
        DBuf<int32_t> c2(any_long ? nnz : 1, s);
        DBuf<double> w2(any_long ? nnz : 1, s);
        perm_fill(PermFill{n, 0, 0, band_hi, sid, spos, rp, col, w, srp, c2.p, w2.p, scol, sw}, nnz, s);
        trace_mark("    permute: rows filled");
        if (any_long)
            sort_rows_min(n, srp, nnz, bitlen_u64((uint64_t)n), band_hi, c2.p, w2.p, scol, sw, s, 0, false, band_hi);
        LAP_CHECK_LAUNCH();
        return;
    }
    // rows of <= 32 entries: permuted and sorted in one thread's registers
    k_perm_sort_thread<16, 0><<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(n, sid, spos, rp, col, w, srp, scol, sw);
    k_perm_sort_thread<32, 17><<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(n, sid, spos, rp, col, w, srp, scol, sw);
    g_kl += 2;
    trace_mark("    permute: short rows sorted");
    if (maxlen > 32) {  // longer rows: copied into a scratch at their positions, then sorted by length class
        DBuf<int32_t> c2(nnz, s);
        DBuf<double> w2(nnz, s);
        perm_fill(PermFill{n, 32, sort_max, band_hi, sid, spos, rp, col, w, srp, c2.p, w2.p, scol, sw}, nnz, s);
        trace_mark("    permute: long rows filled");
        sort_rows_min(n, srp, nnz, bitlen_u64((uint64_t)n), 32, c2.p, w2.p, scol, sw, s, sort_max, false, band_hi);
    }
    LAP_CHECK_LAUNCH();
}

// LAP_DEBUG_SYNC=1: host-side consistency check of a level's storage layout
static void validate_storage(const Level &L, cudaStream_t s) {
    LAP_CUDA(cudaStreamSynchronize(s));
    int64_t n = L.n;
    std::vector<int32_t> sid(n), spos(n);
    std::vector<int64_t> srp(n + 1), rp(n + 1);
    LAP_CUDA(cudaMemcpy(sid.data(), L.sid, 4 * n, cudaMemcpyDeviceToHost));
    LAP_CUDA(cudaMemcpy(spos.data(), L.spos, 4 * n, cudaMemcpyDeviceToHost));
    LAP_CUDA(cudaMemcpy(srp.data(), L.srp, 8 * (n + 1), cudaMemcpyDeviceToHost));
    LAP_CUDA(cudaMemcpy(rp.data(), L.row_ptr, 8 * (n + 1), cudaMemcpyDeviceToHost));
    std::vector<int32_t> scol(L.nnz + 1);
    if (L.nnz) LAP_CUDA(cudaMemcpy(scol.data(), L.scol, 4 * L.nnz, cudaMemcpyDeviceToHost));
    auto fail = [&](const std::string &m) { throw Error{LAP_ECUDA, "validate_storage: " + m}; };
    for (int64_t p = 0; p < n; p++) {
        if (sid[p] < 0 || sid[p] >= n || spos[sid[p]] != p) fail("sid/spos not inverse permutations");
        int64_t dg = rp[sid[p] + 1] - rp[sid[p]];
        if (srp[p + 1] - srp[p] != dg) fail("storage degree mismatch");
        int c = dg <= SHORT_MAX ? 0 : dg <= 1024 ? 1 : dg <= HUB_CHUNK ? 2 : 3;
        int64_t lo = c == 0 ? 0 : L.c_end[c - 1];
        if (p < lo || p >= L.c_end[c]) fail("class range mismatch at row " + std::to_string(p));
    }
    if (srp[n] != L.nnz) fail("srp[n] != nnz");
    for (int64_t k = 0; k < L.nnz; k++)
        if (scol[k] < 0 || scol[k] >= n) fail("scol out of range");
    if (L.nslices) {
        std::vector<int64_t> sp(L.nslices + 1);
        LAP_CUDA(cudaMemcpy(sp.data(), L.slice_ptr, 8 * (L.nslices + 1), cudaMemcpyDeviceToHost));
        std::vector<int32_t> ec(sp[L.nslices] + 1);
        LAP_CUDA(cudaMemcpy(ec.data(), L.ell_col, 4 * sp[L.nslices], cudaMemcpyDeviceToHost));
        if (sp[0] != 0) fail("slice_ptr[0] != 0");
        for (int64_t sl = 0; sl < L.nslices; sl++) {
            if (sp[sl + 1] < sp[sl] || (sp[sl + 1] - sp[sl]) % 32) fail("bad slice_ptr");
            int64_t wdt = (sp[sl + 1] - sp[sl]) / 32;
            for (int64_t r = sl * 32; r < std::min<int64_t>(L.c_end[0], sl * 32 + 32); r++)
                if (srp[r + 1] - srp[r] > wdt) fail("slice narrower than its row");
        }
        for (int64_t k = 0; k < sp[L.nslices]; k++)
            if (ec[k] < 0 || ec[k] >= n) fail("ell_col out of range at " + std::to_string(k));
    }
}

__global__ void k_flag_not_one(int64_t m, const double *__restrict__ w, int *flag) {
    GRID_STRIDE(k, m) {
        if (w[k] != 1.0) *flag = 1;
    }
}

void build_storage(lap_hierarchy *h, int l, cudaStream_t s) {
    Level &L = h->lev[l];
    int64_t n = L.n;
    unsigned g = grid_for(n, 256, 148 * 8);
    DBuf<uint64_t> key(n, s), key2(n, s);  // locality key, sort scratch
    DBuf<int32_t> ids(n, s);
    if (l == 0) {
        k_key_level0<<<g, 256, 0, s>>>(n, h->perm, key.p);
    } else {
        Level &F = h->lev[l - 1];
        if (F.kind == KIND_AGG) {
            k_key_fill<<<g, 256, 0, s>>>(n, ~0ULL, key.p);
            k_key_agg<<<grid_for(F.n, 256, 148 * 8), 256, 0, s>>>(F.n, F.agg, F.spos, (unsigned long long *)key.p);
            g_kl++;
        } else {
            k_key_elim<<<g, 256, 0, s>>>(n, F.cid, F.spos, key.p);
        }
    }
    g_kl++;
    DBuf<unsigned long long> cnt(NCLASS + 1, s);
    LAP_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long) * (NCLASS + 1), s));
    DBuf<uint64_t> skey(n, s);
    L.sid = (int32_t *)dalloc(sizeof(int32_t) * n, s);
    L.spos = (int32_t *)dalloc(sizeof(int32_t) * n, s);
    const char *ho = getenv("LAP_HUB_ORDER");  // experiments
    const int hub_order = ho ? atoi(ho) : 0;
    auto order_rows = [&](int by_degree, unsigned long long *counts) {
        k_class_key<<<g, 256, 0, s>>>(n, L.row_ptr, key.p, skey.p, ids.p, counts, by_degree, hub_order);
        size_t bytes = 0;
        LAP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, skey.p, key2.p, ids.p, L.sid, n, 0, 41, s));
        DBuf<char> tmp((int64_t)bytes, s);
        LAP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, skey.p, key2.p, ids.p, L.sid, n, 0, 41, s));
        g_kl += 3;
        LAP_CHECK_LAUNCH();
    };
    order_rows(0, cnt.p);
    trace_mark("    storage: row order");
    unsigned long long hc[NCLASS + 1];
    LAP_CUDA(cudaMemcpyAsync(hc, cnt.p, sizeof(hc), cudaMemcpyDeviceToHost, s));
    LAP_CUDA(cudaStreamSynchronize(s));
    int64_t acc = 0;
    for (int c = 0; c < NCLASS; c++) {
        acc += (int64_t)hc[c];
        L.c_end[c] = acc;
    }
    // which SpMV kernel serves this level (solve.cu): 8 (n <= 64K) or 4 (n <= 128K)
    // lanes per row over the CSR on levels without long rows (k_spmv_vec) -- a
    // row's ~15 gathers in one dependent round instead of two SELL batches, 8x
    // the CTAs: cfg 2 level 6 (14.5K rows) 6.6 -> 3.8 us per SpMV, level 5
    // 7.2 -> 3.6 us; on large levels SELL stays faster (level 2: 26.6 vs 65 us
    // per Chebyshev step).  LAP_SPMV_VEC=G (0, 4, 8, 16) overrides on every
    // level without long rows (experiments).
    {
        const bool smem = n <= SMEM_X_MAX && L.nnz >= SMEM_X_MIN_DEG * n && L.nnz > 0;
        const char *e = getenv("LAP_SPMV_VEC");
        const int G = e ? atoi(e) : (n <= 65536 ? 8 : n <= 131072 ? 4 : 0);
        L.spmv_vec = (G == 4 || G == 8 || G == 16) && l > 0 && n == L.c_end[0] && !smem ? G : 0;
    }
    // SELL-32 over the short class: degree-sort the short rows if natural order pads > 20%
    // (globally: keeps SELL's gathers as fast as the natural order on mesh levels, measured);
    // CSR-vector levels instead sort by degree within windows of 64 rows (SELL-C-sigma
    // ordering: a warp's 8 rows have similar lengths; cfg 2 level 4 Chebyshev step
    // 10.9 -> 8.5 us, level 6 4.4 -> 4.1 us)
    int64_t nshort = L.c_end[0];
    DBuf<int64_t> width;
    int64_t sell_tot = 0;  // padded SELL entries = sum of the slice widths
    if (nshort > 0) {
        L.nslices = (nshort + 31) / 32;
        width.alloc(L.nslices + 1, s);
        DBuf<unsigned long long> pad(1, s);
        const double rn = (double)hc[NCLASS];
        for (int pass = 0; pass < 2; pass++) {
            LAP_CUDA(cudaMemsetAsync(pad.p, 0, 8, s));
            LAP_CUDA(cudaMemsetAsync(width.p + L.nslices, 0, 8, s));
            k_slice_width<<<grid_for(L.nslices, 256, 148 * 8), 256, 0, s>>>(L.nslices, nshort, L.sid, L.row_ptr, width.p,
                                                                             pad.p);
            g_kl++;
            sell_tot = (int64_t)d2h(pad.p, s);
            const char *es = getenv("LAP_SELL_SIGMA");  // 0: global degree sort; sigma > 0: windows
            const int64_t sigma = es ? atoll(es) : (L.spmv_vec ? 64 : 0);
            if (pass == 1 || (sigma == 0 && (double)sell_tot <= 1.2 * rn + 64.0)) break;
            L.sell_sorted = true;
            if (sigma > 0) {
                DBuf<uint64_t> wk(n, s), wk2(n, s);
                DBuf<int32_t> wid(n, s), sid2(n, s);
                k_window_key<<<g, 256, 0, s>>>(n, nshort, sigma, L.sid, L.row_ptr, wk.p, wid.p);
                int eb = 9;
                while (eb < 64 && ((uint64_t)1 << eb) <= ((uint64_t)(nshort / sigma + 2 + n) << 9)) eb++;
                size_t bytes = 0;
                LAP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, wk.p, wk2.p, wid.p, sid2.p, n, 0, eb, s));
                DBuf<char> tmp((int64_t)bytes, s);
                LAP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, wk.p, wk2.p, wid.p, sid2.p, n, 0, eb, s));
                LAP_CUDA(cudaMemcpyAsync(L.sid, sid2.p, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
                g_kl += 3;
            } else {
                order_rows(1, nullptr);
            }
        }
    }
    k_inverse<<<g, 256, 0, s>>>(n, L.sid, L.spos);
    g_kl++;
    trace_mark("    storage: slices + inverse");
    // storage CSR
    DBuf<int64_t> deg(n + 1, s);
    LAP_CUDA(cudaMemsetAsync(deg.p + n, 0, sizeof(int64_t), s));
    L.sd = (double *)dalloc(sizeof(double) * n, s);
    k_storage_deg<<<g, 256, 0, s>>>(n, L.sid, L.row_ptr, L.d, deg.p, L.sd);
    g_kl++;
    L.srp = (int64_t *)dalloc(sizeof(int64_t) * (n + 1), s);
    scan_excl(deg.p, L.srp, n + 1, s);
    L.scol = (int32_t *)dalloc(sizeof(int32_t) * (L.nnz + 1), s);
    L.sw = (double *)dalloc(sizeof(double) * (L.nnz + 1), s);
    if (L.nnz) {
        // each storage row in ascending STORAGE column order: the u-th column of
        // consecutive rows of a SELL slice then point the same way (-z, -y, -x,
        // +x, ... on a grid-like level), so one gather instruction touches few
        // lines instead of one line per lane (the L1 tag rate bounds these
        // gathers); long rows too (gather locality of dense-ish rows), except on
        // huge levels (>= 2^28 entries, cfg 5), where only the short rows are
        // sorted (no double buffer over ~all entries of a power-law level)
        // elimination levels are never smoothed: their storage serves the PCG's
        // q = L_0 p (level 0) and the F-row solves, whose speed the row order does
        // not change (cfg 3 level 0: 104.5 vs 105.1 us per SpMV) -- no sort there
        // (cfg 3 setup -4 ms)
        const bool sort_on = !getenv_flag_off("LAP_SORT_ROWS") && L.kind != KIND_ELIM;
        const int cbits = bitlen_u64((uint64_t)n);
        // rows of SHORT_MAX < len <= ROWSORT_MED entries (one or two warp chunks of
        // a sparse row: sorting buys no line sharing) stay unsorted; the SELL rows
        // and the hub rows are sorted -- a hub row's chunk of 1024 sorted entries
        // covers a narrow column range, so its gathers share lines (cfg 4 level 1
        // step 286 -> 255 us sorted, medium rows alone 283) -- and so is every row
        // of a shared-memory-x level.  cfg 3 setup -3 ms, cfg 4 -1.5 ms for the
        // same solve (profiles/r02/sortmax_summary.txt; LAP_SORT_LONG=1: sort all)
        const char *sl = getenv("LAP_SORT_LONG");
        const char *sm = getenv("LAP_SORT_MAX");  // experiments: the band's lower end
        const bool smem_level = n <= SMEM_X_MAX && L.nnz >= SMEM_X_MIN_DEG * n;
        // power-law levels (rows beyond SELL exist): the SELL rows' order buys no
        // line sharing either (random neighbours; cfg 4 level 0 step 327.5 us
        // unsorted vs 326.5 sorted), so only the hub rows are sorted there
        // shared-memory-x levels gather from shared memory: no line sharing to win
        // either (cfg 4 level 2 step 80.0 vs 79.8 us, cfg 3 level 3 42.9 vs 42.7) --
        // nothing sorted there (cfg 4: the 1.5 ms segmented sort of level 2)
        const bool mesh_like = L.maxdeg <= SHORT_MAX;
        const int64_t sort_max = (sl && sl[0] == '1') ? INT64_MAX
                                 : sm                 ? atoll(sm)
                                 : smem_level         ? 0
                                 : mesh_like          ? SHORT_MAX
                                                      : 0;
        const int64_t band_hi = smem_level && !(sl && sl[0] == '1') ? INT64_MAX : ROWSORT_MED;
        if (sort_on && L.nnz < ((int64_t)1 << 28)) {
            permute_sorted_rows(n, L.nnz, L.sid, L.spos, L.row_ptr, L.col, L.w, L.srp, L.scol, L.sw,
                                L.maxdeg > 0 ? L.maxdeg : INT64_MAX, s, sort_max, band_hi);
        } else {
            k_storage_fill<<<grid_for(L.nnz, 256, 148 * 16), 256, 0, s>>>(n, L.nnz, L.sid, L.spos, L.row_ptr, L.col,
                                                                          L.w, L.srp, L.scol, L.sw);
            g_kl++;
            const int64_t short_nnz = nshort > 0 ? d2h(L.srp + nshort, s) : 0;
            if (sort_on && short_nnz > 0) {
                DBuf<int32_t> c2(short_nnz, s);
                DBuf<double> w2(short_nnz, s);
                sort_rows(nshort, L.srp, short_nnz, cbits, L.scol, L.sw, c2.p, w2.p, s);
                LAP_CUDA(cudaMemcpyAsync(L.scol, c2.p, sizeof(int32_t) * short_nnz, cudaMemcpyDeviceToDevice, s));
                LAP_CUDA(cudaMemcpyAsync(L.sw, w2.p, sizeof(double) * short_nnz, cudaMemcpyDeviceToDevice, s));
            }
        }
        LAP_CHECK_LAUNCH();
    }
    trace_mark("    storage: csr fill + row sorts");
    // SELL-32 slices of the short class
    if (nshort > 0) {
        L.slice_ptr = (int64_t *)dalloc(sizeof(int64_t) * (L.nslices + 1), s);
        scan_excl(width.p, L.slice_ptr, L.nslices + 1, s);
        int64_t tot = sell_tot;
        L.ell_col = (int32_t *)dalloc(sizeof(int32_t) * (tot + 1), s);
        L.ell_w = (double *)dalloc(sizeof(double) * (tot + 1), s);
        k_sell_fill<<<grid_for(L.nslices * 32, 256, 148 * 8), 256, 0, s>>>(L.nslices * 32, nshort, L.srp, L.scol, L.sw, L.slice_ptr, L.ell_col,
                                                                    L.ell_w);
        g_kl++;
    }
    trace_mark("    storage: sell fill");
    if (debug_sync()) validate_storage(L, s);
    // small dense-ish level: 16-bit column copies for the shared-memory-x SpMV
    if (n <= SMEM_X_MAX && L.nnz >= SMEM_X_MIN_DEG * n && L.nnz > 0) {
        L.smem_x = true;
        int64_t tot = L.nslices ? sell_tot : 0;
        L.ell_col16 = (uint16_t *)dalloc(sizeof(uint16_t) * (tot + 1), s);
        L.scol16 = (uint16_t *)dalloc(sizeof(uint16_t) * (L.nnz + 1), s);
        if (tot) k_to_u16<<<grid_for(tot, 256, 148 * 8), 256, 0, s>>>(tot, L.ell_col, L.ell_col16);
        k_to_u16<<<grid_for(L.nnz, 256, 148 * 8), 256, 0, s>>>(L.nnz, L.scol, L.scol16);
        g_kl += 2;
        LAP_CHECK_LAUNCH();
    }
    // SELL batch width: 4 (5 instead of 4 resident CTAs per SM) for big, low-degree
    // levels (3D grid level 0: 47.3 -> 44.2 us per Chebyshev step), 8 elsewhere
    // (a mid-size level got slower at 4); LAP_NB4_MAXNNZ=x forces 4 for nnz <= x
    {
        const char *e = getenv("LAP_NB4_MAXNNZ");
        if (e) L.spmv_nb = L.nnz <= atoll(e) ? 4 : 8;
        else L.spmv_nb = (L.nnz >= NB4_MIN_NNZ && L.nnz <= 8 * n) ? 4 : 8;
    }
    // pattern-only solve SpMV on a unit-weight level 0: the
    // weights stay stored (setup kernels, exports) but k_spmv does not read them
    // (1.0 * x_j = x_j: the same bits); LAP_UNIT=0 turns it off
    if (l == 0 && L.nnz > 0) {
        const char *e = getenv("LAP_UNIT");
        if (!(e && e[0] == '0')) {
            DBuf<int> flag(1, s);
            LAP_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
            k_flag_not_one<<<grid_for(L.nnz, 256, 148 * 8), 256, 0, s>>>(L.nnz, L.sw, flag.p);
            g_kl++;
            L.unit = d2h(flag.p, s) == 0;
        }
    }
    // long rows: LCHUNK-entry warp work items (solve.cu k_spmv)
    L.nchunks = build_chunks(L.srp, L.c_end[0], n - L.c_end[0], SHORT_MAX, &L.chunk_row, &L.chunk_idx, &L.chunk_slot,
                             &L.chunk_part, &L.chunk_cnt, s, &L.nmulti);
    // dot terms of the multi-chunk rows (3 per row; k_spmv adds them in slot
    // order, run-to-run reproducible) and the kernels' block-arrival counter
    L.mdot = (double *)dalloc(sizeof(double) * (size_t)(3 * L.nmulti + 3), s);
    L.mdone = (int *)dalloc(sizeof(int) * 2, s);
    LAP_CUDA(cudaMemsetAsync(L.mdot, 0, sizeof(double) * (size_t)(3 * L.nmulti + 3), s));
    LAP_CUDA(cudaMemsetAsync(L.mdone, 0, sizeof(int) * 2, s));
    LAP_CHECK_LAUNCH();
    // dense-ish level too big for x in shared memory: the column-tiled layout (xt.cu)
    if (xt_eligible(L, l)) build_xt(L, s);
}

// ---------------------------------------------------------------- transfer maps
__global__ void k_agg_s(int64_t n, const int32_t *sid, const int32_t *agg, const int32_t *cspos, int32_t *agg_s,
                        int32_t *ids) {
    GRID_STRIDE(p, n) {
        agg_s[p] = cspos[agg[sid[p]]];
        ids[p] = (int32_t)p;
    }
}
__global__ void k_lower_bound32(int64_t m, int64_t n, const int32_t *keys, int64_t *ptr) {
    GRID_STRIDE(a, m + 1) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < a) lo = mid + 1;
            else hi = mid;
        }
        ptr[a] = lo;
    }
}
__global__ void k_cid_s(int64_t nc, const int32_t *csid, const int32_t *cid, const int32_t *fspos, int32_t *cid_s) {
    GRID_STRIDE(k, nc) cid_s[k] = fspos[cid[csid[k]]];
}
__global__ void k_fflags(int64_t n, const int32_t *sid, const int32_t *fmap, const int32_t *cspos, int64_t *isf,
                         int32_t *fmap_s) {
    GRID_STRIDE(p, n) {
        int32_t f = fmap[sid[p]];
        isf[p] = f < 0 ? 1 : 0;
        fmap_s[p] = f < 0 ? -1 : cspos[f];
    }
}
__global__ void k_flist(int64_t n, const int64_t *isf, const int64_t *pos, int32_t *flist) {
    GRID_STRIDE(p, n) if (isf[p]) flist[pos[p]] = (int32_t)p;
}
__global__ void k_ct_deg(int64_t nc, const int32_t *csid, const int64_t *ct_ptr, int64_t *deg) {
    GRID_STRIDE(k, nc) {
        int64_t kc = csid[k];
        deg[k] = ct_ptr[kc + 1] - ct_ptr[kc];
    }
}
__global__ void k_ct_fill_s(int64_t nc, const int32_t *csid, const int64_t *ct_ptr, const int32_t *ct_f,
                            const double *ct_coef, const int32_t *fspos, const int64_t *ptr_s, int32_t *f_s,
                            double *coef_s) {
    GRID_STRIDE(k, nc) {
        int64_t kc = csid[k], o = ptr_s[k];
        for (int64_t q = ct_ptr[kc]; q < ct_ptr[kc + 1]; q++, o++) {
            f_s[o] = fspos[ct_f[q]];
            coef_s[o] = ct_coef[q];
        }
    }
}
__global__ void k_pinv_s(int64_t n, const int32_t *sid, const double *P, double *Ps) {
    GRID_STRIDE(t, n * n) {
        int64_t p = t / n, q = t % n;
        Ps[t] = P[(int64_t)sid[p] * n + sid[q]];
    }
}
__global__ void k_cmap(int64_t n, const int64_t *perm, const int32_t *spos0, int64_t *cmap) {
    GRID_STRIDE(c, n) cmap[c] = spos0[perm[c]];
}

void build_transfers(lap_hierarchy *h, cudaStream_t s) {
    for (size_t l = 0; l < h->lev.size(); l++) {
        Level &L = h->lev[l];
        int64_t n = L.n;
        unsigned g = grid_for(n, 256, 148 * 8);
        if (L.kind == KIND_AGG) {
            Level &C = h->lev[l + 1];
            DBuf<int32_t> ids(n, s), keys2(n, s);
            L.agg_s = (int32_t *)dalloc(sizeof(int32_t) * n, s);
            L.members = (int32_t *)dalloc(sizeof(int32_t) * n, s);
            L.mem_ptr = (int64_t *)dalloc(sizeof(int64_t) * (L.m + 1), s);
            k_agg_s<<<g, 256, 0, s>>>(n, L.sid, L.agg, C.spos, L.agg_s, ids.p);
            int end_bit = 1;
            while (end_bit < 31 && ((int64_t)1 << end_bit) <= L.m) end_bit++;
            size_t bytes = 0;
            LAP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, L.agg_s, keys2.p, ids.p, L.members, n, 0, end_bit, s));
            DBuf<char> tmp((int64_t)bytes, s);
            LAP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, L.agg_s, keys2.p, ids.p, L.members, n, 0, end_bit, s));
            k_lower_bound32<<<grid_for(L.m + 1, 256, 148 * 8), 256, 0, s>>>(L.m, n, keys2.p, L.mem_ptr);
            g_kl += 4;
            // hub aggregates (a hub and its thousands of neighbours): warp chunks of
            // LCHUNK members for the restriction (solve.cu k_restrict)
            L.rs_nchunks = build_chunks(L.mem_ptr, 0, L.m, RESTRICT_SHORT, &L.rs_crow, &L.rs_cidx, &L.rs_cslot,
                                        &L.rs_cpart, &L.rs_ccnt, s);
        } else if (L.kind == KIND_ELIM) {
            Level &C = h->lev[l + 1];
            int64_t nc = C.n;
            L.cid_s = (int32_t *)dalloc(sizeof(int32_t) * (nc + 1), s);
            k_cid_s<<<grid_for(nc, 256, 148 * 8), 256, 0, s>>>(nc, C.sid, L.cid, L.spos, L.cid_s);
            DBuf<int64_t> isf(n + 1, s), pos(n + 1, s);
            LAP_CUDA(cudaMemsetAsync(isf.p + n, 0, sizeof(int64_t), s));
            L.fmap_s = (int32_t *)dalloc(sizeof(int32_t) * n, s);
            k_fflags<<<g, 256, 0, s>>>(n, L.sid, L.fmap, C.spos, isf.p, L.fmap_s);
            scan_excl(isf.p, pos.p, n + 1, s);
            L.flist = (int32_t *)dalloc(sizeof(int32_t) * (L.nF + 1), s);
            k_flist<<<g, 256, 0, s>>>(n, isf.p, pos.p, L.flist);
            DBuf<int64_t> deg(nc + 1, s);
            LAP_CUDA(cudaMemsetAsync(deg.p + nc, 0, sizeof(int64_t), s));
            k_ct_deg<<<grid_for(nc, 256, 148 * 8), 256, 0, s>>>(nc, C.sid, L.ct_ptr, deg.p);
            L.ct_ptr_s = (int64_t *)dalloc(sizeof(int64_t) * (nc + 1), s);
            scan_excl(deg.p, L.ct_ptr_s, nc + 1, s);
            int64_t T = d2h(L.ct_ptr_s + nc, s);
            L.ct_f_s = (int32_t *)dalloc(sizeof(int32_t) * (T + 1), s);
            L.ct_coef_s = (double *)dalloc(sizeof(double) * (T + 1), s);
            k_ct_fill_s<<<grid_for(nc, 256, 148 * 8), 256, 0, s>>>(nc, C.sid, L.ct_ptr, L.ct_f, L.ct_coef, L.spos,
                                                                    L.ct_ptr_s, L.ct_f_s, L.ct_coef_s);
            g_kl += 5;
            L.ct_nchunks = build_chunks(L.ct_ptr_s, 0, nc, ELIM_SHORT, &L.ct_crow, &L.ct_cidx, &L.ct_cslot, &L.ct_cpart,
                                        &L.ct_ccnt, s);
        } else {
            L.pinv_s = (double *)dalloc(sizeof(double) * (size_t)(n * n > 0 ? n * n : 1), s);
            if (n * n > 0) k_pinv_s<<<grid_for(n * n, 256, 148 * 8), 256, 0, s>>>(n, L.sid, L.pinv, L.pinv_s);
            g_kl++;
        }
        LAP_CHECK_LAUNCH();
    }
    h->cmap = (int64_t *)dalloc(sizeof(int64_t) * h->n0, s);
    k_cmap<<<grid_for(h->n0, 256, 148 * 8), 256, 0, s>>>(h->n0, h->perm, h->lev[0].spos, h->cmap);
    g_kl++;
    LAP_CHECK_LAUNCH();
}

}  // namespace lap
