// setup.cu -- hierarchy construction on the GPU (sm_100a).
//
// Implements SURVEY.md O-S0..O-S10 (§3.3-3.6)
// with kernels; the host loop below only sequences them and reads back a few
// scalars per level (|F|, m, nnz, lambda-hat).  Every floating reduction that
// feeds a discrete decision (diagonals, test-vector sweeps, Schur and Galerkin
// sums) uses the canonical int128 sum of canon.cuh, so the hierarchy is
// bit-identical to the CPU oracle for any launch geometry.  IEEE rounding of
// each step is explicit (__dmul_rn/__dadd_rn/__ddiv_rn; the file is compiled
// with -fmad=false as well).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <ctime>
#include <string>
#include <vector>

#include "canon.cuh"
#include "lap_internal.cuh"

namespace lap {

int64_t g_kl = 0;  // kernels launched by setup (CUB calls counted once each)

// =========================================================================
// small utilities
// =========================================================================

template <class T>
static void h2d(T *dst, const T *src, int64_t n, cudaStream_t s) {
    LAP_CUDA(cudaMemcpyAsync(dst, src, sizeof(T) * (size_t)n, cudaMemcpyHostToDevice, s));
}
template <class T>
static T d2h_scalar(const T *src, cudaStream_t s) {
    T v;
    LAP_CUDA(cudaMemcpyAsync(&v, src, sizeof(T), cudaMemcpyDeviceToHost, s));
    LAP_CUDA(cudaStreamSynchronize(s));
    return v;
}

static void exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t n, cudaStream_t s) {
    size_t bytes = 0;
    LAP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
    DBuf<char> tmp((int64_t)bytes, s);
    LAP_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, n, s)); ++g_kl;
}

template <int G>
__device__ __forceinline__ i128 grp_sum_i128(i128 v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += shfl_xor_i128(v, o);
    return v;
}
// max |v| as an exact order-independent reduction (bit pattern of a
// non-negative double orders like the value).
__global__ void k_max_abs(const double *__restrict__ v, int64_t n, unsigned long long *out) {
    unsigned long long m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long b = (unsigned long long)__double_as_longlong(fabs(v[i]));
        m = b > m ? b : m;
    }
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long t = __shfl_xor_sync(0xffffffffu, m, o);
        m = t > m ? t : m;
    }
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

static double max_abs(const double *v, int64_t n, cudaStream_t s) {
    DBuf<unsigned long long> r(1, s);
    LAP_CUDA(cudaMemsetAsync(r.p, 0, 8, s));
    if (n > 0) {
        k_max_abs<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(v, n, r.p); ++g_kl;
        LAP_CHECK_LAUNCH();
    }
    unsigned long long b = d2h_scalar(r.p, s);
    double d;
    memcpy(&d, &b, 8);
    return d;
}

// =========================================================================
// O-S0 validation: warp per row
// =========================================================================

// pass 1 of the validation touches row_ptr only: monotone and within
// [0, nnz], so that pass 2 never reads col/w out of bounds
__global__ void k_validate_rowptr(int64_t n, int64_t nnz, const int64_t *__restrict__ row_ptr, int *flag,
                                  unsigned long long *maxdeg) {
    unsigned long long md = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = row_ptr[i], e = row_ptr[i + 1];
        if (a < 0 || e < a || e > nnz) atomicOr(flag, 1);
        else md = (unsigned long long)(e - a) > md ? (unsigned long long)(e - a) : md;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, md, o);
        md = t > md ? t : md;
    }
    if ((threadIdx.x & 31) == 0 && md) atomicMax(maxdeg, md);
}
// Symmetry fingerprint (hsum != NULL): two independent 64-bit multiset hashes,
// sum over entries of h(i, j, bits(w)) - h(j, i, bits(w)) mod 2^64.  A symmetric
// matrix has the same multiset of (i, j, w) and (j, i, w) tuples, so both sums
// are 0; an asymmetric one leaves a nonzero sum except with probability ~2^-128
// (a pseudo-random collision of both hashes).  Integer additions mod 2^64:
// order-free, so the atomics are deterministic.
__device__ __forceinline__ uint64_t sym_h1(uint64_t a, uint64_t b, uint64_t mw) {
    return mix64((a * 0x9E3779B97F4A7C15ULL + b * 0xD1B54A32D192ED03ULL) ^ mw);
}
__device__ __forceinline__ uint64_t sym_h2(uint64_t a, uint64_t b, uint64_t mw) {
    return mix64(mix64(a ^ 0x5851F42D4C957F2DULL) + (b ^ mw));
}
// one stored entry (i, j, w) at position k of row i starting at a
__device__ __forceinline__ void validate_entry(int64_t n, int64_t i, int64_t a, int64_t k,
                                               const int32_t *__restrict__ col, const double *__restrict__ w,
                                               int *flag, bool hash, uint64_t &s1, uint64_t &s2) {
    const int32_t j = col[k];
    bool bad = (j < 0) || (j >= n) || (j == i) || (k > a && col[k - 1] >= j);
    const double wk = w ? w[k] : 1.0;
    bad |= !(wk > 0.0) || !isfinite(wk);
    if (bad) atomicOr(flag, 1);
    if (hash) {
        const uint64_t wb = (uint64_t)__double_as_longlong(wk);
        const uint64_t m1 = mix64(wb), m2 = mix64(wb ^ 0x2545F4914F6CDD1DULL);
        s1 += sym_h1((uint64_t)i, (uint64_t)j, m1) - sym_h1((uint64_t)j, (uint64_t)i, m1);
        s2 += sym_h2((uint64_t)i, (uint64_t)j, m2) - sym_h2((uint64_t)j, (uint64_t)i, m2);
    }
}
__device__ __forceinline__ void hash_flush(uint64_t s1, uint64_t s2, unsigned long long *hsum) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if ((threadIdx.x & 31) == 0 && (s1 | s2)) {
        atomicAdd(&hsum[0], (unsigned long long)s1);
        atomicAdd(&hsum[1], (unsigned long long)s2);
    }
}
// rows longer than skip_long are left to k_validate_chunks (a hub row of 10^4
// - 10^6 entries would serialise one lane group: cfg 3's validation tail)
template <int G>
__global__ void k_validate(int64_t n, const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                           const double *__restrict__ w, int *flag, unsigned long long *hsum, int64_t skip_long) {
    uint64_t s1 = 0, s2 = 0;
    GROUP_LOOP_BEGIN(G, n)
    if (live) {
        int64_t a = row_ptr[i], e = row_ptr[i + 1];
        if (e - a <= skip_long)
            for (int64_t k = a + gl; k < e; k += G) validate_entry(n, i, a, k, col, w, flag, hsum != nullptr, s1, s2);
    }
    GROUP_LOOP_END
    if (hsum) hash_flush(s1, s2, hsum);
}
// LCHUNK-entry warp chunks of the long rows (order-free: flags and mod-2^64 sums)
__global__ void k_validate_chunks(int64_t nch, const int32_t *__restrict__ crow, const int32_t *__restrict__ cidx,
                                  int64_t n, const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                  const double *__restrict__ w, int *flag, unsigned long long *hsum) {
    uint64_t s1 = 0, s2 = 0;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp; c < nch; c += nwarps) {
        const int64_t i = crow[c], a = row_ptr[i], b = a + (int64_t)cidx[c] * LCHUNK, e = min(row_ptr[i + 1], b + LCHUNK);
        for (int64_t k = b + lane; k < e; k += 32) validate_entry(n, i, a, k, col, w, flag, hsum != nullptr, s1, s2);
    }
    if (hsum) hash_flush(s1, s2, hsum);
}

template <int G>
__global__ void k_rowof(int64_t n, const int64_t *__restrict__ row_ptr, int32_t *__restrict__ rowof) {
    GROUP_LOOP_BEGIN(G, n)
    if (live)
        for (int64_t k = row_ptr[i] + gl; k < row_ptr[i + 1]; k += G) rowof[k] = (int32_t)i;
    GROUP_LOOP_END
}

// Symmetry (w_ij == w_ji bitwise): the transposed entry list, sorted
// by (col, row), must equal the CSR list in (row, col) order entry for entry.
// An exact check with one radix sort instead of a binary search per entry
// (which serialises on hub rows).
template <int G, class IT>  // IT: entry index type (int32 below 2^31 entries: 4 sort bytes less per entry)
__global__ void k_sym_keys(int64_t n, int cbits, const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                           int32_t *__restrict__ rowof, uint64_t *__restrict__ tkey, IT *__restrict__ idx) {
    GROUP_LOOP_BEGIN(G, n)
    if (live)
        for (int64_t k = row_ptr[i] + gl; k < row_ptr[i + 1]; k += G) {
            rowof[k] = (int32_t)i;
            tkey[k] = ((uint64_t)(uint32_t)col[k] << cbits) | (uint64_t)i;
            idx[k] = (IT)k;
        }
    GROUP_LOOP_END
}
template <class IT>
__global__ void k_sym_check(int64_t nnz, int cbits, const int32_t *__restrict__ rowof, const int32_t *__restrict__ col,
                            const double *__restrict__ w, const uint64_t *__restrict__ tkey,
                            const IT *__restrict__ idx, int *flag) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nnz; t += (int64_t)gridDim.x * blockDim.x) {
        uint64_t want = ((uint64_t)(uint32_t)rowof[t] << cbits) | (uint64_t)(uint32_t)col[t];
        bool bad = tkey[t] != want;
        if (!bad && w) bad = __double_as_longlong(w[idx[t]]) != __double_as_longlong(w[t]);
        if (bad) atomicOr(flag, 1);
    }
}

template <class IT>
static bool is_symmetric_t(int64_t n, int64_t nnz, const int64_t *rp, const int32_t *col, const double *w,
                           cudaStream_t s) {
    DBuf<int32_t> rowof(nnz, s);
    DBuf<uint64_t> k1(nnz, s), k2(nnz, s);
    DBuf<IT> i1(nnz, s), i2(nnz, s);
    const int cbits = bitlen_u64((uint64_t)n);  // columns are validated < n before this check
#define SYM_KEYS(GG) k_sym_keys<GG, IT>
    {
        const int G = group_size(n, nnz);
        const unsigned gr = grid_for(n * G, 256, 148 * 16);
        switch (G) {
            case 1: SYM_KEYS(1)<<<gr, 256, 0, s>>>(n, cbits, rp, col, rowof.p, k1.p, i1.p); break;
            case 2: SYM_KEYS(2)<<<gr, 256, 0, s>>>(n, cbits, rp, col, rowof.p, k1.p, i1.p); break;
            case 4: SYM_KEYS(4)<<<gr, 256, 0, s>>>(n, cbits, rp, col, rowof.p, k1.p, i1.p); break;
            case 8: SYM_KEYS(8)<<<gr, 256, 0, s>>>(n, cbits, rp, col, rowof.p, k1.p, i1.p); break;
            case 16: SYM_KEYS(16)<<<gr, 256, 0, s>>>(n, cbits, rp, col, rowof.p, k1.p, i1.p); break;
            default: SYM_KEYS(32)<<<gr, 256, 0, s>>>(n, cbits, rp, col, rowof.p, k1.p, i1.p); break;
        }
        ++g_kl;
    }
#undef SYM_KEYS
    size_t bytes = 0;
    int end_bit = 2 * cbits;
    LAP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k1.p, k2.p, i1.p, i2.p, nnz, 0, end_bit, s));
    DBuf<char> tmp((int64_t)bytes, s);
    LAP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, k1.p, k2.p, i1.p, i2.p, nnz, 0, end_bit, s)); ++g_kl;
    DBuf<int> flag(1, s);
    LAP_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
    k_sym_check<IT><<<grid_for(nnz, 256, 148 * 16), 256, 0, s>>>(nnz, cbits, rowof.p, col, w, k2.p, i2.p, flag.p);
    ++g_kl;
    LAP_CHECK_LAUNCH();
    return d2h_scalar(flag.p, s) == 0;
}
// Symmetry without extra memory (large graphs: the sort above needs ~32 B per
// entry, 67 GB at cfg 5): every stored (i, j) looks i up in row j by binary
// search (rows are validated ascending) and compares the weight bit patterns.
// Entry-parallel; a block finds the rows of its 256 entries with two searches.
__global__ void __launch_bounds__(256) k_sym_search(int64_t n, int64_t nnz, const int64_t *__restrict__ rp,
                                                    const int32_t *__restrict__ col, const double *__restrict__ w,
                                                    int *flag) {
    __shared__ int64_t rlo, rhi;
    for (int64_t b0 = (int64_t)blockIdx.x * 256; b0 < nnz; b0 += (int64_t)gridDim.x * 256) {
        const int64_t t = b0 + threadIdx.x;
        if (threadIdx.x < 2) {
            const int64_t tt = threadIdx.x == 0 ? b0 : min(nnz, b0 + 256) - 1;
            rlo = 0;
            int64_t lo = 0, hi = n - 1;
            while (lo < hi) {
                const int64_t mid = (lo + hi + 1) >> 1;
                if (rp[mid] <= tt) lo = mid;
                else hi = mid - 1;
            }
            if (threadIdx.x == 0) rlo = lo;
            else rhi = lo;
        }
        __syncthreads();
        if (t < nnz) {
            int64_t lo = rlo, hi = rhi;
            while (lo < hi) {
                const int64_t mid = (lo + hi + 1) >> 1;
                if (rp[mid] <= t) lo = mid;
                else hi = mid - 1;
            }
            const int64_t i = lo, j = col[t];
            int64_t a = rp[j], e = rp[j + 1];
            while (a < e) {
                const int64_t mid = (a + e) >> 1;
                if (col[mid] < i) a = mid + 1;
                else e = mid;
            }
            bool ok = a < rp[j + 1] && col[a] == i;
            if (ok && w) ok = __double_as_longlong(w[a]) == __double_as_longlong(w[t]);
            if (!ok) atomicOr(flag, 1);
        }
        __syncthreads();
    }
}
// LAP_SYMCHECK = "hash" (default: the fingerprint computed by k_validate),
// "sort" (exact: one radix sort of the transposed entries), "search" (exact:
// a binary search per entry, no extra memory)
static int symcheck_mode() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("LAP_SYMCHECK");
        v = !e ? 0 : (e[0] == 's' && e[1] == 'e') ? 2 : (e[0] == 's' && e[1] == 'o') ? 1 : 0;
    }
    return v;
}
static bool symcheck_by_search(int64_t nnz) {
    return symcheck_mode() == 2 || (symcheck_mode() == 1 && nnz >= ((int64_t)1 << 28));
}
static bool is_symmetric(int64_t n, int64_t nnz, const int64_t *rp, const int32_t *col, const double *w,
                         cudaStream_t s) {
    if (nnz == 0) return true;
    if (symcheck_by_search(nnz)) {
        DBuf<int> flag(1, s);
        LAP_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
        k_sym_search<<<grid_for(nnz, 256, 148 * 16), 256, 0, s>>>(n, nnz, rp, col, w, flag.p); ++g_kl;
        LAP_CHECK_LAUNCH();
        return d2h_scalar(flag.p, s) == 0;
    }
    return nnz < ((int64_t)1 << 31) ? is_symmetric_t<int32_t>(n, nnz, rp, col, w, s)
                                    : is_symmetric_t<int64_t>(n, nnz, rp, col, w, s);
}

// ---- connectivity: lock-free union-find (parents only ever decrease) ----
__global__ void k_cc_init(int64_t n, int32_t *p) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (int32_t)i;
}
__device__ __forceinline__ int32_t cc_find(int32_t *p, int32_t v) {
    int32_t cur = p[v];
    if (cur != v) {
        int32_t prev = v, nxt;
        while (cur > (nxt = p[cur])) {  // path halving
            p[prev] = nxt;
            prev = cur;
            cur = nxt;
        }
    }
    return cur;
}
__device__ __forceinline__ void cc_link(int32_t *p, int32_t i, int32_t j) {
    if (j < i) return;                         // each undirected edge once
    int32_t a = cc_find(p, i), b = cc_find(p, j);
    while (a != b) {
        if (a < b) {
            int32_t t = a; a = b; b = t;
        }
        int32_t ret = atomicCAS(&p[a], a, b);  // hook the larger root under the smaller
        if (ret == a) break;
        a = ret;
    }
}
template <int G>
__global__ void k_cc_union(int64_t n, const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                           int32_t *p, int64_t skip_long) {
    GROUP_LOOP_BEGIN(G, n)
    if (live && row_ptr[i + 1] - row_ptr[i] <= skip_long)
        for (int64_t k = row_ptr[i] + gl; k < row_ptr[i + 1]; k += G) cc_link(p, (int32_t)i, col[k]);
    GROUP_LOOP_END
}
__global__ void k_cc_union_chunks(int64_t nch, const int32_t *__restrict__ crow, const int32_t *__restrict__ cidx,
                                  const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col, int32_t *p) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp; c < nch; c += nwarps) {
        const int64_t i = crow[c], b = row_ptr[i] + (int64_t)cidx[c] * LCHUNK, e = min(row_ptr[i + 1], b + LCHUNK);
        for (int64_t k = b + lane; k < e; k += 32) cc_link(p, (int32_t)i, col[k]);
    }
}
__global__ void k_cc_count_roots(int64_t n, int32_t *p, unsigned long long *cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (cc_find(p, (int32_t)i) == i) atomicAdd(cnt, 1ULL);
}

// the long rows' chunk list of the input graph (validation, connectivity)
struct InputChunks {
    int64_t nch = 0;
    int32_t *crow = nullptr, *cidx = nullptr, *cslot = nullptr, *ccnt = nullptr;
    double *cpart = nullptr;
    cudaStream_t s = nullptr;
    ~InputChunks() {
        for (void *q : {(void *)crow, (void *)cidx, (void *)cslot, (void *)ccnt, (void *)cpart}) dfree(q, s);
    }
};
static bool is_connected(int64_t n, int64_t nnz, const int64_t *row_ptr, const int32_t *col, cudaStream_t s,
                         const InputChunks &IC) {
    if (n <= 1) return true;
    DBuf<int32_t> p(n, s);
    unsigned g = grid_for(n, 256, 148 * 16);
    k_cc_init<<<g, 256, 0, s>>>(n, p.p); ++g_kl;
    LAUNCH_G(group_size(n, nnz), k_cc_union, n, s, n, row_ptr, col, p.p, IC.nch > 0 ? SETUP_LONG : INT64_MAX);
    if (IC.nch > 0) {
        k_cc_union_chunks<<<grid_for(IC.nch * 32, 256, 148 * 16), 256, 0, s>>>(IC.nch, IC.crow, IC.cidx, row_ptr, col,
                                                                                p.p);
        ++g_kl;
    }
    DBuf<unsigned long long> c(1, s);
    LAP_CUDA(cudaMemsetAsync(c.p, 0, 8, s));
    k_cc_count_roots<<<g, 256, 0, s>>>(n, p.p, c.p); ++g_kl;
    LAP_CHECK_LAUNCH();
    return d2h_scalar(c.p, s) == 1;
}

// LAP_SETUP_TRACE=1: synchronise and print the elapsed time of every setup
// phase to stderr (diagnostics only; changes the timing it reports on).
struct SetupTrace {
    bool on = false;
    int mode = 0;  // 1: synchronise per phase; 2: events per phase, no synchronisation, printed at the end
    double t0 = 0;
    cudaStream_t s = nullptr;
    struct M {
        std::string what;
        int l;
        cudaEvent_t e;
        double host;
    };
    std::vector<M> marks;
    ~SetupTrace() {
        if (mode != 2 || marks.empty()) return;
        cudaStreamSynchronize(s);
        for (size_t i = 1; i < marks.size(); i++) {
            float ms = 0;
            cudaEventElapsedTime(&ms, marks[i - 1].e, marks[i].e);
            fprintf(stderr, "[lap trace2] level %2d %-30s gpu %8.3f ms host %8.3f ms\n", marks[i].l, marks[i].what.c_str(),
                    ms, marks[i].host - marks[i - 1].host);
        }
        for (auto &m : marks) cudaEventDestroy(m.e);
    }
    static double now() {
        timespec ts;
        clock_gettime(CLOCK_MONOTONIC, &ts);
        return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
    }
    explicit SetupTrace(cudaStream_t st) : s(st) {
        const char *e = getenv("LAP_SETUP_TRACE");
        mode = e ? (e[0] == '1' ? 1 : e[0] == '2' ? 2 : 0) : 0;
        on = mode != 0;
        if (mode == 1) {
            cudaStreamSynchronize(s);
            t0 = now();
        }
        if (mode == 2) mark("start", -1);
    }
    void mark(const char *what, int l) {
        if (!on) return;
        if (mode == 2) {
            M m{what, l, nullptr, now()};
            cudaEventCreate(&m.e);
            cudaEventRecord(m.e, s);
            marks.push_back(m);
            return;
        }
        cudaStreamSynchronize(s);
        double t = now();
        uint64_t rsv = 0;
        cudaMemPoolGetAttribute(lib_pool(), cudaMemPoolAttrReservedMemCurrent, &rsv);
        fprintf(stderr, "[lap setup] level %2d %-18s %9.3f ms  (pool %.2f GB)\n", l, what, t - t0, rsv / 1e9);
        t0 = t;
    }
};

static SetupTrace *g_tr = nullptr;
static void tmark(const char *what) {
    if (g_tr) g_tr->mark(what, -1);
}
void trace_mark(const char *what) { tmark(what); }

// =========================================================================
// generic: sorted (row,col) terms -> CSR with canonical sums
// =========================================================================

__global__ void k_quantize(int64_t T, const double *__restrict__ v, int elo, I128 *__restrict__ q) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < T; k += (int64_t)gridDim.x * blockDim.x)
        q[k] = to_I128(canon_q(v[k], elo));
}

__global__ void k_terms_to_csr(int64_t U, const uint64_t *__restrict__ ukeys, const I128 *__restrict__ qsum,
                               int cb, int elo, int32_t *__restrict__ col, double *__restrict__ w) {
    uint64_t mask = (1ULL << cb) - 1;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x) {
        col[u] = (int32_t)(ukeys[u] & mask);
        w[u] = canon_result(from_I128(qsum[u]), elo);
    }
}

// CanonSum of segment u = terms v[off[u] .. off[u+1]) (sorted duplicates of key uk[u])
constexpr int64_t SEG_LONG = 128;
__global__ void k_seg_canon(int64_t U, const int64_t *__restrict__ off, const uint64_t *__restrict__ uk,
                            const double *__restrict__ v, int cb, int elo, int32_t *__restrict__ col,
                            double *__restrict__ w) {
    const uint64_t mask = (1ULL << cb) - 1;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x) {
        col[u] = (int32_t)(uk[u] & mask);
        const int64_t a = off[u], e = off[u + 1];
        if (e - a > SEG_LONG) continue;  // k_seg_canon_long
        i128 acc = 0;
        for (int64_t t = a; t < e; t++) acc += canon_q(v[t], elo);
        w[u] = canon_result(acc, elo);
    }
}
// long segments (> SEG_LONG terms; a dense coarse Galerkin has pairs of big
// aggregates with millions of terms): SEG_CHUNK-term warp chunks with int128
// partials, combined exactly per segment (integer addition: order-free)
constexpr int64_t SEG_CHUNK = 4096;
__global__ void k_seg_nchunks(int64_t U, const int64_t *__restrict__ off, int64_t *__restrict__ nch) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t len = off[u + 1] - off[u];
        nch[u] = len > SEG_LONG ? (len + SEG_CHUNK - 1) / SEG_CHUNK : 0;
    }
}
__global__ void k_seg_chunk_map(int64_t U, const int64_t *__restrict__ cfirst, int32_t *__restrict__ cseg) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x)
        for (int64_t c = cfirst[u]; c < cfirst[u + 1]; c++) cseg[c] = (int32_t)u;
}
__global__ void k_seg_chunk_sum(int64_t C, const int32_t *__restrict__ cseg, const int64_t *__restrict__ cfirst,
                                const int64_t *__restrict__ off, const double *__restrict__ v, int elo,
                                I128 *__restrict__ part) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp; c < C; c += nwarps) {
        const int64_t u = cseg[c], j = c - cfirst[u];
        const int64_t a = off[u] + j * SEG_CHUNK, e = min(off[u + 1], a + SEG_CHUNK);
        i128 acc = 0;
        for (int64_t t = a + lane; t < e; t += 32) acc += canon_q(v[t], elo);
        acc = warp_sum_i128(acc);
        if (lane == 0) part[c] = to_I128(acc);
    }
}
__global__ void k_seg_long_finish(int64_t U, const int64_t *__restrict__ cfirst, const I128 *__restrict__ part,
                                  int elo, double *__restrict__ w) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c0 = cfirst[u], c1 = cfirst[u + 1];
        if (c0 == c1) continue;
        i128 acc = 0;
        for (int64_t c = c0; c < c1; c++) acc += from_I128(part[c]);
        w[u] = canon_result(acc, elo);
    }
}

__global__ void k_decode_cols(int64_t T, const uint64_t *__restrict__ k, uint64_t mask, int32_t *__restrict__ c) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < T; i += (int64_t)gridDim.x * blockDim.x)
        c[i] = (int32_t)(k[i] & mask);
}

// row_ptr[r] = first u with (ukeys[u] >> cb) >= r
__global__ void k_row_ptr_from_keys(int64_t nrows, int64_t U, const uint64_t *__restrict__ ukeys, int cb,
                                    int64_t *__restrict__ row_ptr) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= nrows; r += (int64_t)gridDim.x * blockDim.x) {
        uint64_t key = ((uint64_t)r) << cb;
        int64_t lo = 0, hi = U;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (ukeys[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        row_ptr[r] = lo;
    }
}

// d_i = CanonSum of row i (warp per row); instance (e_max, K)
template <int G>
__global__ void k_row_canon_sum(int64_t n, const int64_t *__restrict__ row_ptr, const double *__restrict__ w,
                                int elo, double *__restrict__ d) {
    GROUP_LOOP_BEGIN(G, n)
    i128 acc = 0;
    if (live)
        for (int64_t k = row_ptr[i] + gl; k < row_ptr[i + 1]; k += G) acc += canon_q(w[k], elo);
    acc = grp_sum_i128<G>(acc);
    if (live && gl == 0) d[i] = canon_result(acc, elo);
    GROUP_LOOP_END
}

static void row_sums(int64_t n, int64_t nnz, const int64_t *row_ptr, const double *w, double *d, double *maxw_out,
                     cudaStream_t s) {
    double mw = max_abs(w, nnz, s);
    if (maxw_out) *maxw_out = mw;
    int elo = canon_elo(ilogb_pos(mw) + 1, nnz);
    if (n > 0) {
        LAUNCH_G(group_size(n, nnz), k_row_canon_sum, n, s, n, row_ptr, w, elo, d);
        LAP_CHECK_LAUNCH();
    }
}

// The combine step of csr_from_terms on terms already sorted by (row << cb | col):
// duplicates of a key are one segment; each segment's CanonSum (instance e_max, K)
// is formed directly from the fp64 terms.
static void csr_combine_sorted(int64_t nrows, int cb, int64_t T, DBuf<uint64_t> &k2, DBuf<double> &v2, int e_max,
                               int64_t K, Level &out, cudaStream_t s, bool sums) {
    int64_t U = 0;
    out.n = nrows;
    out.row_ptr = (int64_t *)dalloc(sizeof(int64_t) * (size_t)(nrows + 1), s);
    if (T > 0) {
        // duplicates of a key are one segment of the sorted terms: run-length
        // encode the keys, then each segment's CanonSum is formed directly from
        // the fp64 terms (thread per short segment, warp per long one)
        int elo = canon_elo(e_max, K);
        DBuf<uint64_t> uk(T, s);
        DBuf<int64_t> cnt(T + 1, s), off(T + 1, s), nu(1, s);
        size_t bytes = 0;
        LAP_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, bytes, k2.p, uk.p, cnt.p, nu.p, T, s));
        DBuf<char> tmp((int64_t)bytes, s);
        LAP_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.p, bytes, k2.p, uk.p, cnt.p, nu.p, T, s)); ++g_kl;
        U = d2h_scalar(nu.p, s);
        k2.release();
        tmark("  terms: rle");
        LAP_CUDA(cudaMemsetAsync(cnt.p + U, 0, sizeof(int64_t), s));
        exclusive_scan_i64(cnt.p, off.p, U + 1, s);
        out.nnz = U;
        out.col = (int32_t *)dalloc(sizeof(int32_t) * (size_t)(U + 1), s);
        out.w = (double *)dalloc(sizeof(double) * (size_t)(U + 1), s);
        tmark("  terms: offsets");
        if (U > 0) {
            k_seg_canon<<<grid_for(U, 256, 148 * 16), 256, 0, s>>>(U, off.p, uk.p, v2.p, cb, elo, out.col, out.w); ++g_kl;
            tmark("  terms: short segs");
            DBuf<int64_t> nch(U + 1, s), cfirst(U + 1, s);
            LAP_CUDA(cudaMemsetAsync(nch.p + U, 0, sizeof(int64_t), s));
            k_seg_nchunks<<<grid_for(U, 256, 148 * 16), 256, 0, s>>>(U, off.p, nch.p); ++g_kl;
            exclusive_scan_i64(nch.p, cfirst.p, U + 1, s);
            const int64_t C = d2h_scalar(cfirst.p + U, s);
            if (C > 0) {
                DBuf<int32_t> cseg(C, s);
                DBuf<I128> part(C, s);
                k_seg_chunk_map<<<grid_for(U, 256, 148 * 16), 256, 0, s>>>(U, cfirst.p, cseg.p); ++g_kl;
                k_seg_chunk_sum<<<grid_for(C * 32, 256, 148 * 16), 256, 0, s>>>(C, cseg.p, cfirst.p, off.p, v2.p, elo,
                                                                              part.p); ++g_kl;
                k_seg_long_finish<<<grid_for(U, 256, 148 * 16), 256, 0, s>>>(U, cfirst.p, part.p, elo, out.w); ++g_kl;
            }
            LAP_CHECK_LAUNCH();
        }
        tmark("  terms: canon sums");
        k_row_ptr_from_keys<<<grid_for(nrows + 1, 256, 148 * 16), 256, 0, s>>>(nrows, U, uk.p, cb, out.row_ptr); ++g_kl;
        LAP_CHECK_LAUNCH();
    } else {
        out.nnz = 0;
        out.col = (int32_t *)dalloc(sizeof(int32_t), s);
        out.w = (double *)dalloc(sizeof(double), s);
        k_row_ptr_from_keys<<<grid_for(nrows + 1, 256, 148 * 16), 256, 0, s>>>(nrows, 0, k2.p, cb, out.row_ptr); ++g_kl;
    }
    (void)U;
    if (!sums) return;  // a piece of a split build: the diagonal comes from the gathered rows
    out.d = (double *)dalloc(sizeof(double) * (size_t)(nrows > 0 ? nrows : 1), s);
    row_sums(nrows, out.nnz, out.row_ptr, out.w, out.d, &out.maxw, s);
    tmark("  terms: row sums");
}

// Build a level's CSR from unsorted (key=(row<<cb)|col, value) terms whose
// duplicates are combined by CanonSum with instance (e_max, K).
static void csr_from_terms(int64_t nrows, int cb, int64_t T, DBuf<uint64_t> &keys, DBuf<double> &vals,
                           int e_max, int64_t K, bool combine, Level &out, cudaStream_t s, bool sums = true) {
    int rb = bitlen_u64((uint64_t)(nrows > 0 ? nrows : 1));
    int end_bit = std::min(64, cb + rb);
    DBuf<uint64_t> k2(T, s);
    DBuf<double> v2(T, s);
    if (T > 0) {
        size_t bytes = 0;
        LAP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, k2.p, vals.p, v2.p, T, 0, end_bit, s));
        DBuf<char> tmp((int64_t)bytes, s);
        LAP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, keys.p, k2.p, vals.p, v2.p, T, 0, end_bit, s)); ++g_kl;
    }
    keys.release();
    vals.release();
    tmark("  terms: sort");
    if (combine) {
        csr_combine_sorted(nrows, cb, T, k2, v2, e_max, K, out, s, sums);
        return;
    }
    out.n = nrows;
    out.row_ptr = (int64_t *)dalloc(sizeof(int64_t) * (size_t)(nrows + 1), s);
    out.nnz = T;
    out.col = (int32_t *)dalloc(sizeof(int32_t) * (size_t)(T + 1), s);
    out.w = v2.take();
    if (T > 0) {
        k_decode_cols<<<grid_for(T, 256, 148 * 16), 256, 0, s>>>(T, k2.p, (1ULL << cb) - 1, out.col); ++g_kl;
        LAP_CHECK_LAUNCH();
    }
    k_row_ptr_from_keys<<<grid_for(nrows + 1, 256, 148 * 16), 256, 0, s>>>(nrows, T, k2.p, cb, out.row_ptr); ++g_kl;
    LAP_CHECK_LAUNCH();
    if (!sums) return;
    out.d = (double *)dalloc(sizeof(double) * (size_t)(nrows > 0 ? nrows : 1), s);
    row_sums(nrows, out.nnz, out.row_ptr, out.w, out.d, &out.maxw, s);
    tmark("  terms: row sums");
}

// =========================================================================
// Batched term builder (memory-lean: no global sort of all terms)
// =========================================================================
// A coarse (or relabelled) CSR whose entries are CanonSums of terms generated
// from a fine CSR, built in batches of OUTPUT rows: the terms of rows
// [o0, o1) are emitted, radix-sorted by (row - o0, col), run-length encoded
// and canonically summed, and appended; the next batch reuses the buffers.
// Every output entry is one CanonSum of exactly the method's multiset of terms
// (O-R23), so batching changes nothing in the result -- only the peak memory
// (terms of one batch instead of all nnz terms: the cfg 5 Galerkin and Schur
// products have ~2e9 terms) and the number of key bits each sort touches.
//
// Sources, as a "virtual CSR" over the fine rows (virtual row v -> fine row
// vfine[v] and output row vout[v]; output row o owns virtual rows
// [ostart[o], ostart[o+1]); vptr = prefix of the fine degrees in virtual order):
//   SRC_RELABEL  (O-S1): v = new id r, vfine = old row, terms
//                (r, perm[col], w) -- no duplicates, no sums;
//   SRC_SCHUR    (O-S2, O-R25): v = C index a, vfine = cid[a];
//                entry (i,j): j in C -> (a, fmap j, w_ij); j in F -> for every
//                b != i in N(j): (a, fmap b, fl(fl(w_ij w_jb) / d_j));
//   SRC_GALERKIN (O-S5): v = member slot (members grouped by
//                aggregate, ascending), vfine = the member, vout = its
//                aggregate a; entry (i,j) with agg_j != a -> (a, agg_j, w_ij).
enum { SRC_RELABEL = 0, SRC_SCHUR = 1, SRC_GALERKIN = 2 };
struct TermSrc {
    int kind = 0;
    const int64_t *rp = nullptr;
    const int32_t *col = nullptr;
    const double *w = nullptr;     // NULL: unit weights (RELABEL only)
    const double *d = nullptr;     // SCHUR: d_f
    const int32_t *vfine = nullptr;
    const int32_t *vout = nullptr;  // NULL: vout[v] = v
    const int64_t *ostart = nullptr;  // NULL: ostart[o] = o
    const int64_t *vptr = nullptr;
    const int64_t *perm = nullptr;  // RELABEL
    const uint8_t *F = nullptr;     // SCHUR
    const int32_t *fmap = nullptr;  // SCHUR
    const int32_t *agg = nullptr;   // GALERKIN
};
__device__ __forceinline__ int64_t src_ostart(const TermSrc &S, int64_t o) { return S.ostart ? S.ostart[o] : o; }
__device__ __forceinline__ int64_t src_vout(const TermSrc &S, int64_t v) { return S.vout ? (int64_t)S.vout[v] : v; }

// per virtual row: fine degree (for vptr) and number of terms (upper bound)
template <int G>
__global__ void k_src_counts(int64_t nv, TermSrc S, int64_t *__restrict__ vdeg, int64_t *__restrict__ vterms) {
    GROUP_LOOP_BEGIN(G, nv)
        int64_t c = 0, dg = 0;
        if (live) {
            const int64_t fi = S.vfine[i], a = S.rp[fi], e = S.rp[fi + 1];
            dg = e - a;
            if (S.kind == SRC_SCHUR) {
                for (int64_t k = a + gl; k < e; k += G) {
                    const int64_t j = S.col[k];
                    c += S.F[j] ? (S.rp[j + 1] - S.rp[j] - 1) : 1;
                }
            } else if (gl == 0) {
                c = dg;
            }
        }
        c = grp_sum<G>(c);
        if (live && gl == 0) {
            vdeg[i] = dg;
            vterms[i] = c;
        }
    GROUP_LOOP_END
}
// batch end: the largest o1 <= nout with vcp[ostart[o1]] - vcp[ostart[o0]] <= budget (at least o0 + 1)
__global__ void k_batch_end(int64_t o0, int64_t nout, int64_t budget, TermSrc S, const int64_t *__restrict__ vcp,
                            int64_t *out) {
    const int64_t base = vcp[src_ostart(S, o0)];
    int64_t lo = o0 + 1, hi = nout;
    if (vcp[src_ostart(S, lo)] - base > budget) {
        *out = lo;
        return;
    }
    while (lo < hi) {  // invariant: lo fits
        const int64_t mid = (lo + hi + 1) >> 1;
        if (vcp[src_ostart(S, mid)] - base <= budget) lo = mid;
        else hi = mid - 1;
    }
    *out = lo;
}
// emit the terms of the fine entries [t0, t1) (= the virtual rows [v0, v1)); a
// block claims its output space with one atomic (block scan of per-entry counts)
// rv[t - t0] = the virtual row of fine entry t, t in [vptr[v0], vptr[v1]) (G lanes per row)
template <int G>
__global__ void k_src_rowof(int64_t v0, int64_t v1, const int64_t *__restrict__ vptr, int64_t t0,
                            int32_t *__restrict__ rv) {
    GROUP_LOOP_BEGIN(G, v1 - v0)
    if (live) {
        const int64_t v = v0 + i;
        for (int64_t t = vptr[v] + gl; t < vptr[v + 1]; t += G) rv[t - t0] = (int32_t)v;
    }
    GROUP_LOOP_END
}
__global__ void __launch_bounds__(256) k_src_emit(TermSrc S, int64_t v0, int64_t v1, int64_t t0, int64_t t1,
                                                  int64_t o0, int cb, unsigned long long *cursor,
                                                  uint64_t *__restrict__ keys, double *__restrict__ vals,
                                                  const int32_t *__restrict__ rv) {
    typedef cub::BlockScan<int, 256> BS;
    __shared__ typename BS::TempStorage ts;
    __shared__ unsigned long long boff;
    __shared__ int64_t vlo_s, vhi_s;
    for (int64_t b0 = t0 + (int64_t)blockIdx.x * 256; b0 < t1; b0 += (int64_t)gridDim.x * 256) {
        const int64_t t = b0 + threadIdx.x;
        const int64_t blast = min(t1, b0 + 256) - 1;
        // virtual rows of the block's first and last entries (two searches per block),
        // unless the row of every entry is given (rv: no dependent search chains)
        if (!rv && threadIdx.x < 2) {
            const int64_t tt = threadIdx.x == 0 ? b0 : blast;
            int64_t lo = v0, hi = v1 - 1;
            while (lo < hi) {
                const int64_t mid = (lo + hi + 1) >> 1;
                if (S.vptr[mid] <= tt) lo = mid;
                else hi = mid - 1;
            }
            if (threadIdx.x == 0) vlo_s = lo;
            else vhi_s = lo;
        }
        __syncthreads();
        int cnt = 0;
        int64_t v = 0, i = 0, k = 0, j = 0;
        if (t < t1) {
            if (rv) {
                v = rv[t - t0];
            } else {
                int64_t lo = vlo_s, hi = vhi_s;
                while (lo < hi) {
                    const int64_t mid = (lo + hi + 1) >> 1;
                    if (S.vptr[mid] <= t) lo = mid;
                    else hi = mid - 1;
                }
                v = lo;
            }
            i = S.vfine[v];
            k = S.rp[i] + (t - S.vptr[v]);
            j = S.col[k];
            if (S.kind == SRC_RELABEL) cnt = 1;
            else if (S.kind == SRC_SCHUR) cnt = S.F[j] ? (int)(S.rp[j + 1] - S.rp[j] - 1) : 1;
            else cnt = (S.agg[j] != S.vout[v]) ? 1 : 0;
        }
        int rk, tot;
        BS(ts).ExclusiveSum(cnt, rk, tot);
        if (threadIdx.x == 0) boff = tot ? atomicAdd(cursor, (unsigned long long)tot) : 0ULL;
        __syncthreads();
        if (cnt > 0) {
            int64_t p = (int64_t)boff + rk;
            const uint64_t row = (uint64_t)(src_vout(S, v) - o0) << cb;
            if (S.kind == SRC_RELABEL) {
                keys[p] = row | (uint64_t)S.perm[j];
                vals[p] = S.w ? S.w[k] : 1.0;
            } else if (S.kind == SRC_GALERKIN) {
                keys[p] = row | (uint64_t)S.agg[j];
                vals[p] = S.w[k];
            } else if (!S.F[j]) {
                keys[p] = row | (uint64_t)S.fmap[j];
                vals[p] = S.w[k];
            } else {  // fill through f = j (O-R25): w_ij = w_ji bitwise, the product commutes
                const double wf = S.w[k], df = S.d[j];
                for (int64_t q = S.rp[j]; q < S.rp[j + 1]; q++) {
                    const int64_t bb = S.col[q];
                    if (bb == i) continue;
                    keys[p] = row | (uint64_t)S.fmap[bb];
                    vals[p] = __ddiv_rn(__dmul_rn(wf, S.w[q]), df);
                    p++;
                }
            }
        }
        __syncthreads();
    }
}
// row_ptr[o0 + r] = base + first u with (uk[u] >> cb) >= r, r in [0, nr)
__global__ void k_batch_row_ptr(int64_t nr, int64_t U, const uint64_t *__restrict__ uk, int cb, int64_t base,
                                int64_t *__restrict__ row_ptr) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nr; r += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = ((uint64_t)r) << cb;
        int64_t lo = 0, hi = U;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (uk[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        row_ptr[r] = base + lo;
    }
}
__global__ void k_set_i64(int64_t *p, int64_t v) { *p = v; }

static int64_t batch_budget_override() {  // read per product (tests switch it inside one process)
    const char *e = getenv("LAP_TERM_BATCH");  // tests: force small batches
    return e ? std::max<int64_t>(1, atoll(e)) : 0;
}

// output rows [olo, ohi) of the source -> `out` (ohi - olo rows, local row_ptr
// from 0, no diagonal): terms emitted, sorted and CanonSum-combined in batches
// of at most `budget` terms (S.vptr = fine-entry prefix, vcp = term prefix, both
// over the virtual rows)
static void csr_source_range(const TermSrc &S, const int64_t *vcp, int64_t olo, int64_t ohi, int cb, int e_max,
                             int64_t K, bool combine, int64_t budget, Level &out, cudaStream_t s) {
    const int64_t nr = ohi - olo;
    auto vrow = [&](int64_t o) {  // first virtual row of output row o
        int64_t vv = o;
        if (S.ostart) {
            LAP_CUDA(cudaMemcpyAsync(&vv, S.ostart + o, 8, cudaMemcpyDeviceToHost, s));
            LAP_CUDA(cudaStreamSynchronize(s));
        }
        return vv;
    };
    auto at = [&](const int64_t *p, int64_t v) { return d2h_scalar(p + v, s); };
    const int64_t vlo = vrow(olo), vhi = vrow(ohi);
    const int64_t Tr = at(vcp, vhi) - at(vcp, vlo);
    if (Tr <= budget) {  // one batch: the plain path
        DBuf<uint64_t> keys(Tr, s);
        DBuf<double> vals(Tr, s);
        DBuf<unsigned long long> cur(1, s);
        LAP_CUDA(cudaMemsetAsync(cur.p, 0, 8, s));
        const int64_t t0 = at(S.vptr, vlo), t1 = at(S.vptr, vhi);
        tmark("  terms: alloc");
        if (t1 > t0) {
            DBuf<int32_t> rv(t1 - t0, s);
            LAUNCH_G(8, k_src_rowof, vhi - vlo, s, vlo, vhi, S.vptr, t0, rv.p);
            k_src_emit<<<grid_for(t1 - t0, 256, 148 * 16), 256, 0, s>>>(S, vlo, vhi, t0, t1, olo, cb, cur.p, keys.p,
                                                                       vals.p, rv.p);
            ++g_kl;
            LAP_CHECK_LAUNCH();
        }
        const int64_t T = (int64_t)d2h_scalar(cur.p, s);
        tmark("  terms: emit");
        csr_from_terms(nr, cb, T, keys, vals, e_max, K, combine, out, s, false);
        return;
    }
    // several batches of output rows
    out.n = nr;
    out.row_ptr = (int64_t *)dalloc(sizeof(int64_t) * (size_t)(nr + 1), s);
    int32_t *ocol = (int32_t *)dalloc(sizeof(int32_t) * (size_t)(Tr + 1), s);
    double *ow = (double *)dalloc(sizeof(double) * (size_t)(Tr + 1), s);
    const int elo = canon_elo(e_max, K);
    DBuf<int64_t> o1d(1, s);
    DBuf<unsigned long long> cur(1, s);
    int64_t base = 0, o0 = olo;
    while (o0 < ohi) {
        k_batch_end<<<1, 1, 0, s>>>(o0, ohi, budget, S, vcp, o1d.p); ++g_kl;
        const int64_t o1 = d2h_scalar(o1d.p, s);
        int64_t vr[2] = {vrow(o0), vrow(o1)}, tr2[2], cr[2];
        for (int q = 0; q < 2; q++) {
            LAP_CUDA(cudaMemcpyAsync(&tr2[q], S.vptr + vr[q], 8, cudaMemcpyDeviceToHost, s));
            LAP_CUDA(cudaMemcpyAsync(&cr[q], vcp + vr[q], 8, cudaMemcpyDeviceToHost, s));
        }
        LAP_CUDA(cudaStreamSynchronize(s));
        const int64_t Tb = cr[1] - cr[0];
        DBuf<uint64_t> keys(Tb, s), k2(Tb, s);
        DBuf<double> vals(Tb, s), v2(Tb, s);
        LAP_CUDA(cudaMemsetAsync(cur.p, 0, 8, s));
        if (tr2[1] > tr2[0]) {
            DBuf<int32_t> rv(tr2[1] - tr2[0], s);
            LAUNCH_G(8, k_src_rowof, vr[1] - vr[0], s, vr[0], vr[1], S.vptr, tr2[0], rv.p);
            k_src_emit<<<grid_for(tr2[1] - tr2[0], 256, 148 * 16), 256, 0, s>>>(S, vr[0], vr[1], tr2[0], tr2[1], o0, cb,
                                                                              cur.p, keys.p, vals.p, rv.p);
            ++g_kl;
            LAP_CHECK_LAUNCH();
        }
        const int64_t T = (int64_t)d2h_scalar(cur.p, s);
        const int end_bit = std::min(64, cb + bitlen_u64((uint64_t)(o1 - o0)));
        if (T > 0) {
            size_t bytes = 0;
            LAP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, k2.p, vals.p, v2.p, T, 0, end_bit, s));
            DBuf<char> tmp((int64_t)bytes, s);
            LAP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, keys.p, k2.p, vals.p, v2.p, T, 0, end_bit, s));
            ++g_kl;
        }
        keys.release();
        vals.release();
        int64_t U = T;
        int64_t *rpo = out.row_ptr + (o0 - olo);
        if (combine && T > 0) {
            DBuf<uint64_t> uk(T, s);
            DBuf<int64_t> cnt(T + 1, s), off(T + 1, s), nu(1, s);
            size_t bytes = 0;
            LAP_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, bytes, k2.p, uk.p, cnt.p, nu.p, T, s));
            DBuf<char> tmp((int64_t)bytes, s);
            LAP_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.p, bytes, k2.p, uk.p, cnt.p, nu.p, T, s)); ++g_kl;
            U = d2h_scalar(nu.p, s);
            LAP_CUDA(cudaMemsetAsync(cnt.p + U, 0, sizeof(int64_t), s));
            exclusive_scan_i64(cnt.p, off.p, U + 1, s);
            k_seg_canon<<<grid_for(U, 256, 148 * 16), 256, 0, s>>>(U, off.p, uk.p, v2.p, cb, elo, ocol + base,
                                                                   ow + base); ++g_kl;
            DBuf<int64_t> nch(U + 1, s), cfirst(U + 1, s);
            LAP_CUDA(cudaMemsetAsync(nch.p + U, 0, sizeof(int64_t), s));
            k_seg_nchunks<<<grid_for(U, 256, 148 * 16), 256, 0, s>>>(U, off.p, nch.p); ++g_kl;
            exclusive_scan_i64(nch.p, cfirst.p, U + 1, s);
            const int64_t C = d2h_scalar(cfirst.p + U, s);
            if (C > 0) {
                DBuf<int32_t> cseg(C, s);
                DBuf<I128> part(C, s);
                k_seg_chunk_map<<<grid_for(U, 256, 148 * 16), 256, 0, s>>>(U, cfirst.p, cseg.p); ++g_kl;
                k_seg_chunk_sum<<<grid_for(C * 32, 256, 148 * 16), 256, 0, s>>>(C, cseg.p, cfirst.p, off.p, v2.p, elo,
                                                                              part.p); ++g_kl;
                k_seg_long_finish<<<grid_for(U, 256, 148 * 16), 256, 0, s>>>(U, cfirst.p, part.p, elo, ow + base); ++g_kl;
            }
            k_batch_row_ptr<<<grid_for(o1 - o0, 256, 148 * 8), 256, 0, s>>>(o1 - o0, U, uk.p, cb, base, rpo); ++g_kl;
        } else if (T > 0) {
            k_decode_cols<<<grid_for(T, 256, 148 * 16), 256, 0, s>>>(T, k2.p, (1ULL << cb) - 1, ocol + base); ++g_kl;
            LAP_CUDA(cudaMemcpyAsync(ow + base, v2.p, sizeof(double) * (size_t)T, cudaMemcpyDeviceToDevice, s));
            k_batch_row_ptr<<<grid_for(o1 - o0, 256, 148 * 8), 256, 0, s>>>(o1 - o0, T, k2.p, cb, base, rpo); ++g_kl;
        } else {
            k_batch_row_ptr<<<grid_for(o1 - o0, 256, 148 * 8), 256, 0, s>>>(o1 - o0, 0, k2.p, cb, base, rpo); ++g_kl;
        }
        LAP_CHECK_LAUNCH();
        base += U;
        o0 = o1;
    }
    k_set_i64<<<1, 1, 0, s>>>(out.row_ptr + nr, base); ++g_kl;
    out.nnz = base;
    if (base < Tr - Tr / 4) {  // shrink the over-allocation (Galerkin: entries inside aggregates vanish)
        out.col = (int32_t *)dalloc(sizeof(int32_t) * (size_t)(base + 1), s);
        out.w = (double *)dalloc(sizeof(double) * (size_t)(base + 1), s);
        LAP_CUDA(cudaMemcpyAsync(out.col, ocol, sizeof(int32_t) * (size_t)base, cudaMemcpyDeviceToDevice, s));
        LAP_CUDA(cudaMemcpyAsync(out.w, ow, sizeof(double) * (size_t)base, cudaMemcpyDeviceToDevice, s));
        dfree(ocol, s);
        dfree(ow, s);
    } else {
        out.col = ocol;
        out.w = ow;
    }
    tmark("  terms: batches");
}

// ---- the term build of a coarse operator split over the setup
// ranks.  Output rows are cut into P ranges of equal term counts
// (split_bounds); each rank builds the CSR of its range exactly as one GPU
// would (every entry is one CanonSum of its whole multiset of terms with the
// level's global instance (e_max, K): no partial sums cross ranks), the ranges
// are gathered into the full operator on every rank (dist.cu setup_gather:
// NCCL broadcasts per root, or device copies on a virtual grid) and the
// diagonal is formed from the gathered rows.  The hierarchy is therefore the
// single-GPU one bit for bit; per-rank term memory and term work divide by P.
static int64_t dsetup_min_terms() {
    const char *e = getenv("LAP_DSETUP_MIN");  // tests: 0 forces the split on tiny graphs
    return e ? atoll(e) : ((int64_t)1 << 22);
}
// split this term build? P > 1 and enough terms; with LAP_DSETUP_MIN=0 also a
// single NCCL rank (its gather path -- count allgather, broadcast, row_ptr
// shift -- then runs on one GPU: tests)
static bool dsetup_split(int64_t Ttot) {
    const int64_t mn = dsetup_min_terms();
    return (setup_nranks() > 1 || (mn == 0 && setup_has_comm())) && Ttot >= mn;
}
// bounds[r] = the first output row o with cum(o) * P >= r * total, cum(o) =
// terms of the output rows before o (cum[o] = vcp[ostart[o]]); bounds[0] = 0,
// bounds[P] = nout -- the same rule as lap_setup_split (host)
__global__ void k_split_bounds(int64_t nout, int P, const int64_t *__restrict__ vcp,
                               const int64_t *__restrict__ ostart, int64_t *__restrict__ bounds) {
    const int r = threadIdx.x;
    if (r > P) return;
    bounds[r] = split_bound(r, P, nout, [&](int64_t o) { return vcp[ostart ? ostart[o] : o]; });
}
static std::vector<int64_t> split_bounds(int64_t nout, int P, const int64_t *vcp, const int64_t *ostart,
                                         cudaStream_t s) {
    DBuf<int64_t> b(P + 1, s);
    k_split_bounds<<<1, 64, 0, s>>>(nout, P, vcp, ostart, b.p); ++g_kl;
    LAP_CHECK_LAUNCH();
    std::vector<int64_t> hb(P + 1);
    LAP_CUDA(cudaMemcpyAsync(hb.data(), b.p, 8 * (P + 1), cudaMemcpyDeviceToHost, s));
    LAP_CUDA(cudaStreamSynchronize(s));
    return hb;
}
// ---- the row-parallel passes over a level's logical CSR --
// elimination select (Alg. 2), affinity and the vote rounds
// (Alg. 3) -- split by rows over the setup ranks in ranges of equal entry
// counts (the term builds' rule with cum(o) = row_ptr[o]).  Each rank computes
// its rows exactly as one GPU does (every per-row result depends only on
// replicated round-start data), then the rows are shared (setup_share) and the
// votes summed (K4: integer sums); the hierarchy is the single-GPU one
// bit for bit, and each rank reads 1/P of the level's entries per pass.
struct RowSplit {
    bool on = false;
    std::vector<int64_t> rb{0, 0}, eb{0, 0};  // row / entry bounds of the P ranges
    std::vector<int> mine{0};                 // ranges this process computes
    std::vector<int64_t> bytes(const std::vector<int64_t> &b, int64_t esz) const {
        std::vector<int64_t> o(b.size());
        for (size_t r = 0; r < b.size(); r++) o[r] = b[r] * esz;
        return o;
    }
};
__global__ void k_split_rows(int64_t n, int P, const int64_t *__restrict__ row_ptr, int64_t *__restrict__ out) {
    const int r = threadIdx.x;
    if (r > P) return;
    const int64_t b = split_bound(r, P, n, [&](int64_t o) { return row_ptr[o]; });
    out[r] = b;
    out[P + 1 + r] = row_ptr[b];
}
static RowSplit row_split(int64_t n, int64_t nnz, const int64_t *row_ptr, cudaStream_t s) {
    RowSplit R;
    R.rb = {0, n};
    R.eb = {0, nnz};
    if (!dsetup_split(nnz)) return R;
    const int P = setup_nranks();
    DBuf<int64_t> b(2 * (P + 1), s);
    k_split_rows<<<1, 64, 0, s>>>(n, P, row_ptr, b.p); ++g_kl;
    LAP_CHECK_LAUNCH();
    std::vector<int64_t> hb(2 * (P + 1));
    LAP_CUDA(cudaMemcpyAsync(hb.data(), b.p, 8 * hb.size(), cudaMemcpyDeviceToHost, s));
    LAP_CUDA(cudaStreamSynchronize(s));
    R.on = true;
    R.rb.assign(hb.begin(), hb.begin() + P + 1);
    R.eb.assign(hb.begin() + P + 1, hb.end());
    R.mine = setup_local_ranks();
    return R;
}

// run build(lo, hi, piece) for this process's ranges and gather the full operator
template <class F>
static void build_split(int64_t nout, const std::vector<int64_t> &bounds, Level &out, cudaStream_t s, F build) {
    const int P = (int)bounds.size() - 1;
    std::vector<Level> pieces;
    std::vector<int> mine = setup_local_ranks();
    for (int r : mine) {
        pieces.emplace_back();
        build(bounds[r], bounds[r + 1], pieces.back());
    }
    setup_gather(pieces, mine, bounds, out, s);
    (void)P;
    out.n = nout;
    out.d = (double *)dalloc(sizeof(double) * (size_t)(nout > 0 ? nout : 1), s);
    row_sums(nout, out.nnz, out.row_ptr, out.w, out.d, &out.maxw, s);
    tmark("  terms: gathered + row sums");
}

// Build `out` (nout rows, column bits cb) from the source; CanonSum instance (e_max, K).
static void csr_from_source(const TermSrc &S0, int64_t nv, int64_t nout, int cb, int e_max, int64_t K, bool combine,
                            Level &out, cudaStream_t s) {
    TermSrc S = S0;
    DBuf<int64_t> vdeg(nv + 1, s), vterm(nv + 1, s), vptr(nv + 1, s), vcp(nv + 1, s);
    LAP_CUDA(cudaMemsetAsync(vdeg.p + nv, 0, sizeof(int64_t), s));
    LAP_CUDA(cudaMemsetAsync(vterm.p + nv, 0, sizeof(int64_t), s));
    if (nv > 0) {
        LAUNCH_G(S.kind == SRC_SCHUR ? 32 : 1, k_src_counts, nv, s, nv, S, vdeg.p, vterm.p);
        LAP_CHECK_LAUNCH();
    }
    exclusive_scan_i64(vdeg.p, vptr.p, nv + 1, s);
    exclusive_scan_i64(vterm.p, vcp.p, nv + 1, s);
    vdeg.release();
    vterm.release();
    S.vptr = vptr.p;
    const int64_t Ttot = d2h_scalar(vcp.p + nv, s);
    tmark("  terms: counts");
    // batch budget: ~56 B per term in flight (keys, values, their sort copies, RLE)
    int64_t budget = batch_budget_override();
    if (!budget) {
        // free-memory estimate without cudaMemGetInfo (measured: 0.5-29 ms per call,
        // randomly -- the setup-time outliers): device total minus what liblap's
        // pool holds in use (other allocators of the process are not seen)
        const size_t fr = device_free_estimate();
        budget = std::max<int64_t>((int64_t)1 << 24, std::min<int64_t>((int64_t)1 << 28, (int64_t)(fr / 4 / 64)));
    }
    tmark("  terms: budget");
    const int P = setup_nranks();
    if (dsetup_split(Ttot)) {
        const std::vector<int64_t> bounds = split_bounds(nout, P, vcp.p, S.ostart, s);
        build_split(nout, bounds, out, s, [&](int64_t lo, int64_t hi, Level &piece) {
            csr_source_range(S, vcp.p, lo, hi, cb, e_max, K, combine, budget, piece, s);
        });
        return;
    }
    csr_source_range(S, vcp.p, 0, nout, cb, e_max, K, combine, budget, out, s);
    out.d = (double *)dalloc(sizeof(double) * (size_t)(nout > 0 ? nout : 1), s);
    row_sums(nout, out.nnz, out.row_ptr, out.w, out.d, &out.maxw, s);
    tmark("  terms: row sums");
}

// =========================================================================
// O-S1 level 0: random order (O-R31) and relabel
// =========================================================================

__global__ void k_perm_keys(int64_t n, uint64_t salt, uint64_t *keys, int32_t *ids) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = mix64((uint64_t)i ^ salt);
        ids[i] = (int32_t)i;
    }
}
__global__ void k_perm_from_order(int64_t n, const int32_t *order, int64_t *perm) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        perm[order[r]] = r;
}
__global__ void k_inverse_perm(int64_t n, const int64_t *perm, int32_t *inv) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        inv[perm[i]] = (int32_t)i;
}
__global__ void k_perm_to_i32(int64_t n, const int64_t *perm, int32_t *p32) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p32[i] = (int32_t)perm[i];
}
__global__ void k_identity_i64(int64_t n, int64_t *p) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = i;
}
// emit (newrow<<cb | perm[col], w) for every stored entry; warp per old row
template <int G>
__global__ void k_relabel_emit(int64_t n, const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                               const double *__restrict__ w, const int64_t *__restrict__ perm, int cb,
                               uint64_t *__restrict__ keys, double *__restrict__ vals) {
    GROUP_LOOP_BEGIN(G, n)
    if (live) {
        uint64_t r = (uint64_t)perm[i];
        for (int64_t k = row_ptr[i] + gl; k < row_ptr[i + 1]; k += G) {
            keys[k] = (r << cb) | (uint64_t)perm[col[k]];
            vals[k] = w ? w[k] : 1.0;
        }
    }
    GROUP_LOOP_END
}

// =========================================================================
// O-S2 elimination (Alg. 2; O-R17..O-R22) and Schur
// =========================================================================

// h(j) = mix64(j XOR salt_2) (O-R17)
__device__ __forceinline__ uint64_t elim_hash(int64_t j, uint64_t salt2) { return mix64((uint64_t)j ^ salt2); }

__global__ void k_elim_select(int64_t r0, int64_t r1, const int64_t *__restrict__ row_ptr,
                              const int32_t *__restrict__ col, int maxdeg, uint64_t salt2, uint8_t *__restrict__ F,
                              unsigned long long *nF) {
    int64_t cnt = 0;
    for (int64_t i = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r1; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t a = row_ptr[i], e = row_ptr[i + 1];
        uint8_t f = 0;
        if (e - a <= maxdeg) {                       // candidate (O-R19)
            uint64_t bh = elim_hash(i, salt2);
            int64_t bj = i;
            for (int64_t k = a; k < e; k++) {         // oplus_elim over the closed neighbourhood
                int64_t j = col[k];
                if (row_ptr[j + 1] - row_ptr[j] > maxdeg) continue;
                uint64_t hj = elim_hash(j, salt2);
                if (hj < bh || (hj == bh && j < bj)) { bh = hj; bj = j; }
            }
            f = (bj == i);
        }
        F[i] = f;
        cnt += f;
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(nF, (unsigned long long)cnt);
}

__global__ void k_flag_not(int64_t n, const uint8_t *F, int64_t *isc) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        isc[i] = F[i] ? 0 : 1;
}
__global__ void k_flag_f(int64_t n, const uint8_t *F, int64_t *isf) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        isf[i] = F[i] ? 1 : 0;
}
// fmap: C -> coarse index (order preserving, O-R22), F -> -1-slot
__global__ void k_fmap(int64_t n, const uint8_t *F, const int64_t *cpos, const int64_t *fpos, int32_t *fmap,
                       int32_t *cid, int32_t *fid) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (F[i]) {
            fmap[i] = (int32_t)(-1 - fpos[i]);
            fid[fpos[i]] = (int32_t)i;
        } else {
            fmap[i] = (int32_t)cpos[i];
            cid[cpos[i]] = (int32_t)i;
        }
    }
}
// Schur complement terms (O-R25), generated where they are cheap:
//   * L_CC entries w_ab from the C rows (a group of G lanes per row, ballot-
//     compacted in ascending column order);
//   * fill fl(fl(w_fa w_fb)/d_f) for every ordered pair a != b of neighbours
//     of each f in F, from the F rows (F is independent, so all neighbours of
//     f are in C, and deg_f <= 4: a thread per f, at most 12 terms).
// The multiset of terms is the method's; their order is irrelevant (sorted
// and summed with CanonSum), so hub C rows no longer serialise the build.
// L_CC entries: every stored (i, j) with i, j both in C -> ((fmap_i << cb) | fmap_j, w)
__global__ void __launch_bounds__(256) k_schur_cc_emit(int64_t n, int64_t nnz, const int32_t *__restrict__ rowof,
                                                       const int32_t *__restrict__ col, const double *__restrict__ w,
                                                       const uint8_t *__restrict__ F, const int32_t *__restrict__ fmap,
                                                       int cb, unsigned long long *cursor, uint64_t *__restrict__ keys,
                                                       double *__restrict__ vals) {
    int64_t i = 0;
    ENTRY_EMIT_LOOP(nnz, cursor, (i = rowof[t], take = !F[i] && !F[col[t]]),
                    (keys[p] = ((uint64_t)fmap[i] << cb) | (uint64_t)fmap[col[t]], vals[p] = w[t]))
}
__global__ void k_schur_f_count(int64_t nF, const int32_t *__restrict__ fid, const int64_t *__restrict__ row_ptr,
                                int64_t *cnt) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nF; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t f = fid[t], dg = row_ptr[f + 1] - row_ptr[f];
        cnt[t] = dg * (dg - 1);
    }
}
__global__ void k_schur_f_emit(int64_t nF, const int32_t *__restrict__ fid, const int64_t *__restrict__ row_ptr,
                               const int32_t *__restrict__ col, const double *__restrict__ w,
                               const double *__restrict__ d, const int32_t *__restrict__ fmap,
                               const int64_t *__restrict__ off, int64_t base, int cb, uint64_t *__restrict__ keys,
                               double *__restrict__ vals) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nF; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = fid[t], kb = row_ptr[f], ke = row_ptr[f + 1];
        const double df = d[f];
        int64_t o = base + off[t];
        for (int64_t p = kb; p < ke; p++) {
            const uint64_t ra = ((uint64_t)fmap[col[p]]) << cb;
            for (int64_t q = kb; q < ke; q++) {
                if (q == p) continue;
                keys[o] = ra | (uint64_t)fmap[col[q]];
                vals[o] = __ddiv_rn(__dmul_rn(w[p], w[q]), df);
                o++;
            }
        }
    }
}
// transposed L_FC for the restriction: per coarse c, (f, w_fc/d_f) for f ~ c in F,
// in ascending f order (a group of G lanes per C row)
template <int G>
__global__ void k_ct_count(int64_t nc, const int32_t *__restrict__ cid, const int64_t *__restrict__ row_ptr,
                           const int32_t *__restrict__ col, const uint8_t *__restrict__ F, int64_t *cnt) {
    GROUP_LOOP_BEGIN(G, nc)
        int64_t c = 0;
        if (live) {
            const int64_t fi = cid[i];
            for (int64_t k = row_ptr[fi] + gl; k < row_ptr[fi + 1]; k += G) c += F[col[k]] ? 1 : 0;
        }
        c = grp_sum<G>(c);
        if (live && gl == 0) cnt[i] = c;
    GROUP_LOOP_END
}
template <int G>
__global__ void k_ct_fill(int64_t nc, const int32_t *__restrict__ cid, const int64_t *__restrict__ row_ptr,
                          const int32_t *__restrict__ col, const double *__restrict__ w, const double *__restrict__ d,
                          const uint8_t *__restrict__ F, const int64_t *__restrict__ off, int32_t *__restrict__ ct_f,
                          double *__restrict__ ct_coef) {
    GROUP_LOOP_BEGIN(G, nc)
        const int64_t fi = live ? cid[i] : 0;
        const int64_t kb = live ? row_ptr[fi] : 0, ke = live ? row_ptr[fi + 1] : 0;
        int64_t o = live ? off[i] : 0;
        GROUP_COMPACT_ROW(G, kb, ke, o, F[col[k]], (ct_f[p] = col[k], ct_coef[p] = w[k] / d[col[k]]))
    GROUP_LOOP_END
}

// =========================================================================
// O-S3 strength
// =========================================================================

// X0[i,k] = 2 u01(mix64(base ^ (4i+k))) - 1, base = mix64(salt3 ^ (2l+attempt))
__global__ void k_tv_init(int64_t n, uint64_t base, double *X) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 4 * n; t += (int64_t)gridDim.x * blockDim.x)
        X[t] = __dsub_rn(__dmul_rn(2.0, unit_from(mix64(base ^ (uint64_t)t))), 1.0);
}

// X0 in the storage order: Xs[4p+k] = X0[sid[p], k] (the counter is the logical id, O-R7/O-R33)
__global__ void k_tv_init_s(int64_t n, uint64_t base, const int32_t *__restrict__ sid, double *__restrict__ X) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 4 * n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = t >> 2, k = t & 3;
        const uint64_t c = 4 * (uint64_t)sid[p] + (uint64_t)k;
        X[t] = __dsub_rn(__dmul_rn(2.0, unit_from(mix64(base ^ c))), 1.0);
    }
}
__global__ void k_tv_unpermute(int64_t n, const int32_t *__restrict__ sid, const double *__restrict__ Xs,
                               double *__restrict__ X) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 4 * n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = t >> 2, k = t & 3;
        X[4 * (int64_t)sid[p] + k] = Xs[t];
    }
}
// E_lo of a sweep's CanonSum instance from the bit pattern of max |x| (O-S11)
__global__ void k_tv_elo(const unsigned long long *mxbits, int ew, int64_t K, int *elo) {
    double mx = __longlong_as_double((long long)*mxbits);
    int e_max = mx > 0.0 ? ew + ilogb(mx) + 2 : ew + 1;
    *elo = canon_elo(e_max, K);
}
// one synchronous damped-Jacobi sweep on the 4 columns; warp per row
template <int G>
__global__ void k_tv_sweep(int64_t n, const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                           const double *__restrict__ w, const double *__restrict__ d, const int *__restrict__ elo_p,
                           double omega, const double *__restrict__ X, double *__restrict__ Xn) {
    const int elo = *elo_p;
    GROUP_LOOP_BEGIN(G, n)
        i128 a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        const int64_t kb0 = live ? row_ptr[i] : 0, ke0 = live ? row_ptr[i + 1] : 0;
        const bool skip = ke0 - kb0 > SETUP_LONG;  // long rows: k_tv_chunk
        const int64_t kb = skip ? 0 : kb0, ke = skip ? 0 : ke0;
        for (int64_t k = kb + gl; k < ke; k += G) {
            int64_t j = col[k];
            double wk = w[k];
            const double2 *xj = reinterpret_cast<const double2 *>(X + 4 * j);
            double2 u = xj[0], v = xj[1];
            a0 += canon_q(__dmul_rn(wk, u.x), elo);
            a1 += canon_q(__dmul_rn(wk, u.y), elo);
            a2 += canon_q(__dmul_rn(wk, v.x), elo);
            a3 += canon_q(__dmul_rn(wk, v.y), elo);
        }
        a0 = grp_sum_i128<G>(a0);
        a1 = grp_sum_i128<G>(a1);
        a2 = grp_sum_i128<G>(a2);
        a3 = grp_sum_i128<G>(a3);
        if (live && !skip)
            for (int cq = gl; cq < 4; cq += G) {  // every lane holds all four sums
                i128 a = cq == 0 ? a0 : cq == 1 ? a1 : cq == 2 ? a2 : a3;
                double sk = canon_result(a, elo);
                double di = d[i];
                double xi = X[4 * i + cq];
                double r = __dsub_rn(__dmul_rn(di, xi), sk);
                double q = __ddiv_rn(r, di);
                Xn[4 * i + cq] = __dsub_rn(xi, __dmul_rn(omega, q));
            }
    GROUP_LOOP_END
}

// rows longer than SETUP_LONG (hubs, up to ~10^6 entries at cfg 5): LCHUNK-entry
// warp chunks of the four int128 sums; the last chunk of a row to arrive adds
// the row's partials (exact integer sums: any order) and applies the update
__global__ void k_tv_chunk(int64_t nchunks, const int32_t *__restrict__ crow, const int32_t *__restrict__ cidx,
                           const int32_t *__restrict__ cslot, int32_t *__restrict__ ccnt, I128 *__restrict__ part,
                           const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                           const double *__restrict__ w, const double *__restrict__ d, const int *__restrict__ elo_p,
                           double omega, const double *__restrict__ X, double *__restrict__ Xn) {
    const int elo = *elo_p;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp; c < nchunks; c += nwarps) {
        const int64_t i = crow[c], j = cidx[c], rb = row_ptr[i], re = row_ptr[i + 1];
        const int64_t b = rb + j * LCHUNK, e = min(re, b + LCHUNK);
        i128 a[4] = {0, 0, 0, 0};
        for (int64_t k = b + lane; k < e; k += 32) {
            const double wk = w[k];
            const double2 *xj = reinterpret_cast<const double2 *>(X + 4 * (int64_t)col[k]);
            const double2 u = xj[0], v = xj[1];
            a[0] += canon_q(__dmul_rn(wk, u.x), elo);
            a[1] += canon_q(__dmul_rn(wk, u.y), elo);
            a[2] += canon_q(__dmul_rn(wk, v.x), elo);
            a[3] += canon_q(__dmul_rn(wk, v.y), elo);
        }
#pragma unroll
        for (int q = 0; q < 4; q++) a[q] = warp_sum_i128(a[q]);
        const int nch = (int)((re - rb + LCHUNK - 1) / LCHUNK);
        int last = 0;
        if (lane == 0) {
            for (int q = 0; q < 4; q++) part[4 * c + q] = to_I128(a[q]);
            __threadfence();
            last = atomicAdd(&ccnt[cslot[c]], 1) == nch - 1;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (!last) continue;
        __threadfence();
        if (lane < 4) {
            i128 t = 0;
            for (int64_t q = c - j; q < c - j + nch; q++) {  // L2 reads: other SMs wrote them
                I128 pv;
                pv.lo = __ldcg(&part[4 * q + lane].lo);
                pv.hi = __ldcg(&part[4 * q + lane].hi);
                t += from_I128(pv);
            }
            const double sk = canon_result(t, elo), di = d[i], xi = X[4 * i + lane];
            const double r = __dsub_rn(__dmul_rn(di, xi), sk);
            Xn[4 * i + lane] = __dsub_rn(xi, __dmul_rn(omega, __ddiv_rn(r, di)));
        }
        if (lane == 0) ccnt[cslot[c]] = 0;
    }
}

__device__ __forceinline__ double dot4_rn(const double *a, const double *b) {
    double s = __dmul_rn(a[0], b[0]);
    s = __dadd_rn(s, __dmul_rn(a[1], b[1]));
    s = __dadd_rn(s, __dmul_rn(a[2], b[2]));
    s = __dadd_rn(s, __dmul_rn(a[3], b[3]));
    return s;
}

// C_ij of one stored entry (O-R5): fixed k-order, no FMA
__device__ __forceinline__ double affinity_of(const double *__restrict__ X, int64_t i, int64_t j, int power) {
    const double2 *xi2 = reinterpret_cast<const double2 *>(X + 4 * i), *xj2 = reinterpret_cast<const double2 *>(X + 4 * j);
    const double2 a0 = xi2[0], a1 = xi2[1], b0 = xj2[0], b1 = xj2[1];
    double xi[4] = {a0.x, a0.y, a1.x, a1.y}, xj[4] = {b0.x, b0.y, b1.x, b1.y};
    double ni = dot4_rn(xi, xi), nj = dot4_rn(xj, xj), g = dot4_rn(xi, xj);
    double num = __dmul_rn(g, g);
    double den = power == 2 ? __dmul_rn(__dmul_rn(ni, ni), __dmul_rn(nj, nj)) : __dmul_rn(ni, nj);
    return den > 0.0 ? __ddiv_rn(num, den) : 0.0;
}
// long rows (deg > SETUP_LONG), entry-parallel over their chunks: C, and the row
// max M_i as an atomic max of the bit pattern (non-negative doubles order like
// their bits; max is exact and order-free)
__global__ void k_affinity_long(int64_t nchunks, const int32_t *__restrict__ crow, const int32_t *__restrict__ cidx,
                                int64_t r0, int64_t r1, const int64_t *__restrict__ row_ptr,
                                const int32_t *__restrict__ col, const double *__restrict__ X, int power,
                                double *__restrict__ C, unsigned long long *__restrict__ Mbits) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp; c < nchunks; c += nwarps) {
        const int64_t i = crow[c];
        if (i < r0 || i >= r1) continue;  // another setup rank's row
        const int64_t b = row_ptr[i] + (int64_t)cidx[c] * LCHUNK, e = min(row_ptr[i + 1], b + LCHUNK);
        double mx = 0.0;
        for (int64_t k = b + lane; k < e; k += 32) {
            double cv = affinity_of(X, i, col[k], power);
            C[k] = cv;
            mx = cv > mx ? cv : mx;
        }
        for (int o = 16; o > 0; o >>= 1) {
            double t = __shfl_xor_sync(0xffffffffu, mx, o);
            mx = t > mx ? t : mx;
        }
        if (lane == 0) atomicMax(&Mbits[i], (unsigned long long)__double_as_longlong(mx));
    }
}
// C_ij (O-R5) and row max M_i; warp per row
// (64 registers: 4 CTAs per SM; 78 left 37 % of the warps resident and the
// 32-byte X gathers latency-bound, ncu profiles/r02)
template <int G>
__global__ void __launch_bounds__(256, 4) k_affinity(int64_t r0, int64_t r1, const int64_t *__restrict__ row_ptr,
                           const int32_t *__restrict__ col, const double *__restrict__ X, int power,
                           double *__restrict__ C, double *__restrict__ M) {
    GROUP_LOOP_RANGE_BEGIN(G, r0, r1)
        const int64_t ii = live ? i : 0;
        double xi[4] = {X[4 * ii], X[4 * ii + 1], X[4 * ii + 2], X[4 * ii + 3]};
        double ni = dot4_rn(xi, xi);
        double mx = 0.0;
        const int64_t kb0 = live ? row_ptr[i] : 0, ke0 = live ? row_ptr[i + 1] : 0;
        const bool skip = ke0 - kb0 > SETUP_LONG;  // long rows: k_affinity_long
        const int64_t kb = skip ? 0 : kb0, ke = skip ? 0 : ke0;
        // 4 column loads, then 4 independent 32-byte gathers of X_j in flight per lane
        for (int64_t k0 = kb + gl; k0 < ke; k0 += 4 * G) {
            int64_t jj[4];
#pragma unroll
            for (int u = 0; u < 4; u++) jj[u] = k0 + u * G < ke ? __ldcs(&col[k0 + u * G]) : 0;
            double2 u0[4], u1[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const double2 *xj2 = reinterpret_cast<const double2 *>(X + 4 * jj[u]);  // 32-byte aligned rows
                u0[u] = xj2[0];
                u1[u] = xj2[1];
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int64_t k = k0 + u * G;
                if (k >= ke) break;
                double xj[4] = {u0[u].x, u0[u].y, u1[u].x, u1[u].y};
                double nj = dot4_rn(xj, xj);
                double g = dot4_rn(xi, xj);
                double num = __dmul_rn(g, g);
                double den = power == 2 ? __dmul_rn(__dmul_rn(ni, ni), __dmul_rn(nj, nj)) : __dmul_rn(ni, nj);
                double c = den > 0.0 ? __ddiv_rn(num, den) : 0.0;
                C[k] = c;
                mx = c > mx ? c : mx;
            }
        }
        for (int o = G / 2; o > 0; o >>= 1) {
            double t = __shfl_xor_sync(0xffffffffu, mx, o);
            mx = t > mx ? t : mx;
        }
        if (live && gl == 0 && !skip) M[i] = mx;
    GROUP_LOOP_END
}
// S_ij = C_ij / max(M_i, M_j), 0 if that max is 0 (O-R16); in place,
// entry-parallel (hub rows do not serialise)
__global__ void k_normalize(int64_t n, int64_t nnz, const int32_t *__restrict__ rowof,
                            const int32_t *__restrict__ col, const double *__restrict__ M, double *__restrict__ CS) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const double mi = M[rowof[k]], mj = M[col[k]];
        const double den = mi > mj ? mi : mj;
        CS[k] = den > 0.0 ? __ddiv_rn(CS[k], den) : 0.0;
    }
}

// =========================================================================
// O-S4 voting (Alg. 3; O-R8..O-R15)
// =========================================================================
enum { ST_DEC = 0, ST_UND = 1, ST_SEED = 2 };

__global__ void k_vote_init(int64_t n, int8_t *st, int32_t *idx, int32_t *votes) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        st[i] = ST_UND;
        idx[i] = (int32_t)i;
        votes[i] = 0;
    }
}

// Long rows (deg > SETUP_LONG) of a vote round, chunk-parallel: the argmax
// under (rank(state), S, -j) is an atomic max of key = rank << 62 | bits(S)
// (S in (0, 1] has bits < 2^62) followed by an atomic min of j over the entries
// that hit the max; both are exact and order-free.  best / bestj are reset by
// k_vote_long_apply, so they only need initialising once.
__device__ __forceinline__ unsigned long long vote_key(const double *__restrict__ S, const int32_t *__restrict__ col,
                                                       const int8_t *__restrict__ st, int64_t k, double filt) {
    const double sv = S[k];
    if (sv == 0.0 || sv < filt) return 0ULL;
    const int r = st[col[k]];
    if (r == ST_DEC) return 0ULL;
    return ((unsigned long long)r << 62) | (unsigned long long)__double_as_longlong(sv);
}
__global__ void k_vote_long_max(int64_t nchunks, const int32_t *__restrict__ crow, const int32_t *__restrict__ cidx,
                                int64_t r0, int64_t r1, const int64_t *__restrict__ row_ptr,
                                const int32_t *__restrict__ col, const double *__restrict__ S, double filt, const int8_t *__restrict__ st,
                                unsigned long long *__restrict__ best) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp; c < nchunks; c += nwarps) {
        const int64_t i = crow[c];
        if (i < r0 || i >= r1 || st[i] != ST_UND) continue;
        const int64_t b = row_ptr[i] + (int64_t)cidx[c] * LCHUNK, e = min(row_ptr[i + 1], b + LCHUNK);
        unsigned long long m = 0;
        for (int64_t k = b + lane; k < e; k += 32) {
            unsigned long long key = vote_key(S, col, st, k, filt);
            m = key > m ? key : m;
        }
        for (int o = 16; o > 0; o >>= 1) {
            unsigned long long t = __shfl_xor_sync(0xffffffffu, m, o);
            m = t > m ? t : m;
        }
        if (lane == 0 && m) atomicMax(&best[i], m);
    }
}
__global__ void k_vote_long_argj(int64_t nchunks, const int32_t *__restrict__ crow, const int32_t *__restrict__ cidx,
                                 int64_t r0, int64_t r1, const int64_t *__restrict__ row_ptr,
                                 const int32_t *__restrict__ col,
                                 const double *__restrict__ S, double filt, const int8_t *__restrict__ st,
                                 const unsigned long long *__restrict__ best, int32_t *__restrict__ bestj) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp; c < nchunks; c += nwarps) {
        const int64_t i = crow[c];
        if (i < r0 || i >= r1 || st[i] != ST_UND || best[i] == 0) continue;
        const unsigned long long bk = best[i];
        const int64_t b = row_ptr[i] + (int64_t)cidx[c] * LCHUNK, e = min(row_ptr[i + 1], b + LCHUNK);
        int32_t jm = 0x7fffffff;
        for (int64_t k = b + lane; k < e; k += 32)
            if (vote_key(S, col, st, k, filt) == bk) jm = min(jm, col[k]);
        for (int o = 16; o > 0; o >>= 1) jm = min(jm, __shfl_xor_sync(0xffffffffu, jm, o));
        if (lane == 0 && jm != 0x7fffffff) atomicMin(&bestj[i], jm);
    }
}
__global__ void k_vote_long_apply(int64_t nchunks, const int32_t *__restrict__ crow, const int32_t *__restrict__ cidx,
                                  int64_t r0, int64_t r1, const int8_t *__restrict__ st, const int32_t *__restrict__ idx,
                                  unsigned long long *__restrict__ best, int32_t *__restrict__ bestj,
                                  int8_t *__restrict__ nst, int32_t *__restrict__ nidx, int32_t *__restrict__ votes) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nchunks; c += (int64_t)gridDim.x * blockDim.x) {
        if (cidx[c] != 0) continue;  // once per long row
        const int64_t i = crow[c];
        if (i < r0 || i >= r1) continue;
        const unsigned long long bk = best[i];
        const int br = bk ? (int)(bk >> 62) : -1;
        const bool act = st[i] == ST_UND;
        const bool dec = act && br == ST_SEED;
        nst[i] = dec ? (int8_t)ST_DEC : st[i];
        nidx[i] = dec ? bestj[i] : idx[i];
        if (act && br == ST_UND) atomicAdd(&votes[bestj[i]], 1);
        best[i] = 0;
        bestj[i] = 0x7fffffff;
    }
}
__global__ void k_vote_long_init(int64_t n, unsigned long long *best, int32_t *bestj) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        best[i] = 0;
        bestj[i] = 0x7fffffff;
    }
}
// ---- vote rounds over the ACTIVE rows only.  A row leaves Undecided once
// (Decided by a seed, or promoted to Seed) and never changes again (Alg. 3,
// O-R9), so each round runs over the rows still Undecided at its start: a
// list compacted after every round (late rounds of cfg 4 level 0 have a few
// per cent of the rows left).  The round writes nst / nidx of its listed
// rows; k_vote_commit then applies the promotion and copies them
// into st / idx (the rows not listed are final in st), and appends the rows
// still Undecided to the next list.  Order-free: same states, bit for bit.
// Levels of short rows (grids: fewer than 10 entries per row on average) keep
// the plain row order instead (list = nullptr, out = nullptr: every row of
// [lo, lo + n) each round, non-Undecided rows skipped): there the list's
// indirection and compaction cost more than the rows they skip.
// (round 1: list = nullptr, the rows lo, lo + 1, ... themselves)
__global__ void k_act_init(int64_t lo, int64_t hi, int32_t *__restrict__ cnt) { *cnt = (int32_t)(hi - lo); }
template <int G>
__global__ void k_vote_round_list(const int32_t *__restrict__ list, int64_t lo, const int32_t *__restrict__ nact_p,
                                  const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                  const double *__restrict__ S, double filt, const int8_t *__restrict__ st,
                                  int8_t *__restrict__ nst, int32_t *__restrict__ nidx, int32_t *__restrict__ votes) {
    const int64_t nact = *nact_p;
    GROUP_LOOP_BEGIN(G, nact)
        const int64_t ia = !live ? 0 : list ? list[i] : lo + i;  // a listed row is Undecided at the round's start
        const int sti = !live ? ST_DEC : list ? ST_UND : st[ia];
        const int64_t rb = live ? row_ptr[ia] : 0, re = live ? row_ptr[ia + 1] : 0;
        const bool lng = re - rb > SETUP_LONG;   // k_vote_long_*
        const bool act = sti == ST_UND && !lng;
        int br = -1;
        double bs = 0.0;
        int32_t bj = 0x7fffffff;
        const int64_t kb = act ? rb : 0, ke = act ? re : 0;
        for (int64_t k0 = kb + gl; k0 < ke; k0 += 4 * G) {
            double sv[4];
            int32_t jj[4];
            int rr[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int64_t k = k0 + u * G;
                sv[u] = k < ke ? __ldcs(&S[k]) : 0.0;
                jj[u] = k < ke ? __ldcs(&col[k]) : 0;
            }
#pragma unroll
            for (int u = 0; u < 4; u++)   // filter 2^-t, w != 0 (O-R13)
                rr[u] = (sv[u] == 0.0 || sv[u] < filt) ? ST_DEC : (int)st[jj[u]];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int r = rr[u];
                if (r == ST_DEC) continue;                  // (O-R12)
                if (r > br || (r == br && (sv[u] > bs || (sv[u] == bs && jj[u] < bj)))) { br = r; bs = sv[u]; bj = jj[u]; }
            }
        }
        for (int o = G / 2; o > 0; o >>= 1) {               // group arg-max under (rank, S, -j)
            int r2 = __shfl_xor_sync(0xffffffffu, br, o);
            double s2 = __shfl_xor_sync(0xffffffffu, bs, o);
            int32_t j2 = __shfl_xor_sync(0xffffffffu, bj, o);
            if (r2 > br || (r2 == br && (s2 > bs || (s2 == bs && j2 < bj)))) { br = r2; bs = s2; bj = j2; }
        }
        if (act && gl == 0) {
            const bool dec = br == ST_SEED;
            nst[ia] = dec ? (int8_t)ST_DEC : (int8_t)ST_UND;
            nidx[ia] = dec ? bj : (int32_t)ia;               // an Undecided row's idx is its own id
            if (br == ST_UND) atomicAdd(&votes[bj], 1);
        }
    GROUP_LOOP_END
}
__global__ void k_vote_commit(const int32_t *__restrict__ list, int64_t lo, const int32_t *__restrict__ nact_p,
                              const int8_t *__restrict__ nst, const int32_t *__restrict__ nidx,
                              const int32_t *__restrict__ votes, int thr, int8_t *__restrict__ st,
                              int32_t *__restrict__ idx, int32_t *__restrict__ out, int32_t *__restrict__ out_cnt) {
    const int64_t nact = *nact_p;
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31LL; base < nact; base += stride) {
        const int64_t t = base + lane;
        bool keep = false;
        int32_t i = 0;
        if (t < nact) {
            i = list ? list[t] : (int32_t)(lo + t);
            const bool fin = !list && st[i] != ST_UND;  // no list: rows already final are skipped
            int sv = fin ? -1 : nst[i];
            if (sv == ST_UND && votes[i] >= thr) sv = ST_SEED;  // promotion
            if (sv == ST_DEC || sv == ST_SEED) {                // (st[i] is Undecided, idx[i] = i)
                st[i] = (int8_t)sv;
                if (sv == ST_DEC) idx[i] = nidx[i];
            }
            keep = sv == ST_UND;
        }
        if (!out) continue;  // plain row order: no list
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        int pos = 0;
        if (lane == 0 && m) pos = atomicAdd(out_cnt, __popc(m));
        pos = __shfl_sync(0xffffffffu, pos, 0);
        if (keep) out[pos + __popc(m & ((1u << lane) - 1))] = i;
    }
}
__global__ void k_root_flags(int64_t n, const int8_t *st, int64_t *flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = st[i] != ST_DEC ? 1 : 0;
}
__global__ void k_agg_ids(int64_t n, const int8_t *st, const int32_t *idx, const int64_t *rid, int32_t *agg) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        agg[i] = (int32_t)(st[i] != ST_DEC ? rid[i] : rid[idx[i]]);
}

// =========================================================================
// O-S5 Galerkin (O-R24)
// =========================================================================

// Galerkin terms: every stored (i, j, w) with a = agg_i != b = agg_j
// becomes ((a << cb) | b, w); entry-parallel, so hub rows do not serialise.
__global__ void __launch_bounds__(256) k_gal_emit(int64_t n, int64_t nnz, const int32_t *__restrict__ rowof,
                                                  const int32_t *__restrict__ col, const double *__restrict__ w,
                                                  const int32_t *__restrict__ agg, int cb,
                                                  unsigned long long *cursor, uint64_t *__restrict__ keys,
                                                  double *__restrict__ vals) {
    uint64_t a = 0, bb = 0;
    ENTRY_EMIT_LOOP(nnz, cursor,
                    (a = (uint64_t)agg[rowof[t]], bb = (uint64_t)agg[col[t]], take = a != bb),
                    (keys[p] = (a << cb) | bb, vals[p] = w[t]))
}

// =========================================================================
// O-S6 lambda-hat: Lanczos on D^-1/2 L D^-1/2 (O-R3)
// =========================================================================

// lambda-hat is computed with canonical sums (reading R-lambda of DESIGN.md:
// O-R23 extended to the Lanczos SpMV and dots), on the logical CSR, so it is a
// deterministic function of the level and bit-identical to the oracle's
// orc_lanczos.  Exponent bounds (every |term| < 2^e_max, computed from exact
// maxima; |v_i| < 2 since v = y / ||y||):
//   ||v0||^2 : e_max = 1                                  K = n
//   (L u)_i  : e_max = e(max w) + e(max rs) + 3           K = nnz
//   alpha    : e_max = e(max|y|) + 2                      K = n
//   beta^2   : e_max = 2 (max(e(max|y|)+1, e(alpha)+2) + 2)   K = n
// e(m) = ilogb(m) for m > 0, else -1000.  One step = four launches:
//   A  v_prev = v, v = fl(y / beta), u = fl(rs v)  (+ records alpha, beta of the
//      previous step and the breakdown test beta <= 1e-14 |alpha|)
//   B  y = fl(fl(rs fl(fl(d u) - s)) - fl(beta_prev v_prev)), s = CanonSum_j fl(w u_j); max |y|
//   C  alpha = CanonSum fl(y v)
//   D  y = fl(y - fl(alpha v)), beta^2 = CanonSum fl(y y)
// Exact int128 accumulators are global (two 64-bit atomics with carry).
struct LzState {
    I128 acc_a, acc_b;          // alpha and beta^2 accumulators
    unsigned long long maxy;    // bit pattern of max |y|
    double alpha, bprev;
    int elo_b;                  // E_lo of the beta^2 instance being read by pass A
    int stop, k;
};
__device__ __forceinline__ int ebound_dev(double m) { return m > 0.0 ? ilogb(m) : -1000; }
__device__ __forceinline__ void atomic_add_i128(I128 *acc, i128 v) {
    const unsigned long long lo = (unsigned long long)(u128)v;
    const unsigned long long hi = (unsigned long long)((u128)v >> 64);
    const unsigned long long old = atomicAdd(&acc->lo, lo);
    const unsigned long long carry = (old + lo < old) ? 1ULL : 0ULL;
    atomicAdd((unsigned long long *)&acc->hi, hi + carry);
}
// block-wide exact int128 sum, added once per block into *acc
__device__ __forceinline__ void block_add_i128(I128 *acc, i128 v) {
    __shared__ I128 sh[32];
    v = warp_sum_i128(v);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh[wid] = to_I128(v);
    __syncthreads();
    if (wid == 0) {
        i128 t = lane < (int)(blockDim.x >> 5) ? from_I128(sh[lane]) : (i128)0;
        t = warp_sum_i128(t);
        if (lane == 0 && t != 0) atomic_add_i128(acc, t);
    }
}
__device__ __forceinline__ double lz_start_value(uint64_t base, int64_t i) {
    return __dsub_rn(__dmul_rn(2.0, unit_from(mix64(base ^ (uint64_t)i))), 1.0);
}
// y = the unnormalised start vector, rs = fl(1 / fl(sqrt(d))), acc_b += q(y^2)
__global__ void k_lzc_init(int64_t n, uint64_t base, const double *__restrict__ d, double *__restrict__ y,
                           double *__restrict__ rs, double *__restrict__ vp, LzState *st, int elo) {
    i128 acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = lz_start_value(base, i);
        y[i] = v;
        vp[i] = 0.0;
        rs[i] = __ddiv_rn(1.0, __dsqrt_rn(d[i]));
        acc += canon_q(__dmul_rn(v, v), elo);
    }
    block_add_i128(&st->acc_b, acc);
}
// pass A (also the final record-only pass after the last step)
__global__ void __launch_bounds__(256) k_lzc_next(int64_t n, int first, int record_only, const double *__restrict__ y,
                                                  double *__restrict__ v, double *__restrict__ vp,
                                                  double *__restrict__ u, const double *__restrict__ rs, LzState *st,
                                                  double *alpha_rec, double *beta_rec) {
    if (st->stop) return;
    const double b = __dsqrt_rn(canon_result(from_I128(st->acc_b), st->elo_b));
    bool stop = false;
    if (!first) {
        const double a = st->alpha;
        stop = b <= __dmul_rn(1e-14, fabs(a));
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            alpha_rec[st->k] = a;
            beta_rec[st->k] = b;
        }
    }
    __syncthreads();  // every block has read st before block 0 updates it
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (!first) st->k += 1;
        if (stop) st->stop = 1;
        st->bprev = first ? 0.0 : b;
        st->acc_a.lo = 0;
        st->acc_a.hi = 0;
        st->maxy = 0;
    }
    if (stop || record_only) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double vn = __ddiv_rn(y[i], b);
        if (!first) vp[i] = v[i];
        v[i] = vn;
        u[i] = __dmul_rn(rs[i], vn);
    }
}
__device__ __forceinline__ double lzc_row_epilogue(int64_t i, double sk, const double *__restrict__ d,
                                                   const double *__restrict__ u, const double *__restrict__ rs,
                                                   const double *__restrict__ vp, double bprev,
                                                   double *__restrict__ y) {
    const double li = __dsub_rn(__dmul_rn(d[i], u[i]), sk);
    const double yi = __dsub_rn(__dmul_rn(rs[i], li), __dmul_rn(bprev, vp[i]));
    y[i] = yi;
    return fabs(yi);
}
// max |y| of a warp, one atomic per warp (a single address takes one atomic per
// row otherwise: 4M serialised atomics on cfg 4 level 0)
__device__ __forceinline__ void warp_atomic_max(unsigned long long *maxy, double v) {
    unsigned long long b = (unsigned long long)__double_as_longlong(v);
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, b, o);
        b = t > b ? t : b;
    }
    if ((threadIdx.x & 31) == 0 && b) atomicMax(maxy, b);
}
// pass B, rows up to SETUP_LONG entries (G lanes per row)
template <int G>
__global__ void k_lzc_spmv(int64_t n, const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                           const double *__restrict__ w, const double *__restrict__ d, const double *__restrict__ u,
                           const double *__restrict__ rs, const double *__restrict__ vp, int elo, LzState *st,
                           double *__restrict__ y) {
    if (st->stop) return;
    const double bprev = st->bprev;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->acc_b.lo = 0;  // read by pass A only; pass A of this step has finished
        st->acc_b.hi = 0;
    }
    GROUP_LOOP_BEGIN(G, n)
        i128 a = 0;
        const int64_t kb0 = live ? row_ptr[i] : 0, ke0 = live ? row_ptr[i + 1] : 0;
        const bool skip = ke0 - kb0 > SETUP_LONG;  // long rows: k_lzc_chunk
        const int64_t kb = skip ? 0 : kb0, ke = skip ? 0 : ke0;
        for (int64_t k = kb + gl; k < ke; k += G) a += canon_q(__dmul_rn(w[k], u[col[k]]), elo);
        a = grp_sum_i128<G>(a);
        double ya = 0.0;
        if (live && !skip && gl == 0) ya = lzc_row_epilogue(i, canon_result(a, elo), d, u, rs, vp, bprev, y);
        warp_atomic_max(&st->maxy, ya);
    GROUP_LOOP_END
}
// pass B, rows longer than SETUP_LONG: LCHUNK warp chunks, the last chunk of a
// row to arrive adds the row's exact partials and applies the epilogue
__global__ void k_lzc_chunk(int64_t nchunks, const int32_t *__restrict__ crow, const int32_t *__restrict__ cidx,
                            const int32_t *__restrict__ cslot, int32_t *__restrict__ ccnt, I128 *__restrict__ part,
                            const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                            const double *__restrict__ w, const double *__restrict__ d, const double *__restrict__ u,
                            const double *__restrict__ rs, const double *__restrict__ vp, int elo, LzState *st,
                            double *__restrict__ y) {
    if (st->stop) return;
    const double bprev = st->bprev;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp; c < nchunks; c += nwarps) {
        const int64_t i = crow[c], j = cidx[c], rb = row_ptr[i], re = row_ptr[i + 1];
        const int64_t b = rb + j * LCHUNK, e = min(re, b + LCHUNK);
        i128 a = 0;
        for (int64_t k = b + lane; k < e; k += 32) a += canon_q(__dmul_rn(w[k], u[col[k]]), elo);
        a = warp_sum_i128(a);
        const int nch = (int)((re - rb + LCHUNK - 1) / LCHUNK);
        int last = 0;
        if (lane == 0) {
            part[c] = to_I128(a);
            __threadfence();
            last = atomicAdd(&ccnt[cslot[c]], 1) == nch - 1;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (!last) continue;
        __threadfence();
        if (lane == 0) {
            i128 t = 0;
            for (int64_t q = c - j; q < c - j + nch; q++) {
                I128 pv;
                pv.lo = __ldcg(&part[q].lo);
                pv.hi = __ldcg(&part[q].hi);
                t += from_I128(pv);
            }
            const double ya = lzc_row_epilogue(i, canon_result(t, elo), d, u, rs, vp, bprev, y);
            atomicMax(&st->maxy, (unsigned long long)__double_as_longlong(ya));
            ccnt[cslot[c]] = 0;
        }
    }
}
// ---- canonical SpMV over the SOLVE STORAGE (SELL slices | long-row chunks):
// the same order-independent CanonSum per row as the logical-CSR kernels above,
// but in the storage order (locality of the caller's numbering, coalesced
// SELL loads, hub rows in 1024-entry warp chunks): NC = 1 (Lanczos, x = u) or
// 4 (test-vector sweep, x = the n x 4 block).  Any order gives the same bits.
enum { CS_LANCZOS = 0, CS_SWEEP = 1 };
struct CStore {
    int64_t nslices, nshort, nchunks;
    const int64_t *__restrict__ slice_ptr;
    const int32_t *__restrict__ ell_col;
    const double *__restrict__ ell_w;
    const int64_t *__restrict__ srp;
    const int32_t *__restrict__ scol;
    const double *__restrict__ sw;
    const double *__restrict__ sd;
    const int32_t *__restrict__ crow, *__restrict__ cidx, *__restrict__ cslot;
    int32_t *__restrict__ ccnt;
    I128 *__restrict__ cpart;  // NC per chunk
    // the work of one setup rank (SURVEY N1 row-split sweeps): slices [s_lo, s_hi)
    // and the chunks of the long rows [p_lo, p_hi); cstore_of: everything
    int64_t s_lo, s_hi, p_lo, p_hi;
};
struct CSweep {  // CS_SWEEP: x_new = x - omega ((d x - s) / d), per column
    const double *__restrict__ X;
    double *__restrict__ Xn;
    const int *__restrict__ elo_p;
    double omega;
};
template <int NC>
__device__ __forceinline__ void cs_gather(const double *__restrict__ x, int64_t c, double wk, int elo, double s2,
                                          i128 *acc) {
    if (NC == 1) {
        acc[0] += canon_q_s(__dmul_rn(wk, x[c]), s2, elo);
    } else {
        const double2 *xj = reinterpret_cast<const double2 *>(x + 4 * c);
        const double2 u = xj[0], v = xj[1];
        acc[0] += canon_q_s(__dmul_rn(wk, u.x), s2, elo);
        acc[1] += canon_q_s(__dmul_rn(wk, u.y), s2, elo);
        acc[2] += canon_q_s(__dmul_rn(wk, v.x), s2, elo);
        acc[3] += canon_q_s(__dmul_rn(wk, v.y), s2, elo);
    }
}
// NC x-values of column c (the gather half of cs_gather, issued ahead of the sums)
#ifndef CS_SB4
#define CS_SB4 4
#endif
template <int NC>
struct CsX {
    double v[NC];
};
template <int NC>
__device__ __forceinline__ CsX<NC> cs_load(const double *__restrict__ x, int64_t c) {
    CsX<NC> r;
    if (NC == 1) {
        r.v[0] = x[c];
    } else {
        const double2 *xj = reinterpret_cast<const double2 *>(x + 4 * c);
        const double2 u = xj[0], v = xj[1];
        r.v[0] = u.x;
        r.v[1] = u.y;
        r.v[2] = v.x;
        r.v[3] = v.y;
    }
    return r;
}
template <int NC, int MODE>
__device__ __forceinline__ double cs_epilogue(int64_t p, const i128 *acc, int elo, const CStore &C,
                                              const double *__restrict__ u, const double *__restrict__ rs,
                                              const double *__restrict__ vp, double bprev, double *__restrict__ y,
                                              const CSweep &W) {
    if (MODE == CS_LANCZOS) return lzc_row_epilogue(p, canon_result(acc[0], elo), C.sd, u, rs, vp, bprev, y);
    const double di = C.sd[p];
#pragma unroll
    for (int k = 0; k < NC; k++) {
        const double sk = canon_result(acc[k], elo), xi = W.X[4 * p + k];
        const double r = __dsub_rn(__dmul_rn(di, xi), sk);
        W.Xn[4 * p + k] = __dsub_rn(xi, __dmul_rn(W.omega, __ddiv_rn(r, di)));
    }
    return 0.0;
}
// XS: the whole x staged in shared memory first (small dense-ish levels, as
// the solve's k_spmv_smem: random gathers from a ~100 KB x are bound by the L1
// tag rate); one 1024-thread CTA per SM
// (occupancy: 78 / 128 registers left 35 % / 25 % of the warps resident and the
// gathers latency-bound, ncu profiles/r02; the bounds cap them at 64 / 80)
template <int NC, int MODE, bool XS = false>
__global__ void __launch_bounds__(XS ? 1024 : 256, XS ? 1 : 4) k_cspmv_store(CStore C, const double *__restrict__ x0,
                                                                 const double *__restrict__ rs,
                                                                 const double *__restrict__ vp, int elo_fixed,
                                                                 LzState *st, double *__restrict__ y, CSweep W,
                                                                 int64_t nx) {
    extern __shared__ double xs_dyn[];
    if (MODE == CS_LANCZOS && st->stop) return;
    if (XS) {
        for (int64_t i = threadIdx.x; i < nx; i += blockDim.x) xs_dyn[i] = x0[i];
        __syncthreads();
    }
    const double *__restrict__ x = XS ? xs_dyn : x0;
    const double bprev = MODE == CS_LANCZOS ? st->bprev : 0.0;
    const int elo = W.elo_p ? *W.elo_p : elo_fixed;
    const double s2 = canon_scale(elo);
    if (MODE == CS_LANCZOS && blockIdx.x == 0 && threadIdx.x == 0) {
        st->acc_b.lo = 0;  // read by pass A only; pass A of this step has finished
        st->acc_b.hi = 0;
    }
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nsl = C.s_hi - C.s_lo;
    const int64_t nitems = nsl + C.nchunks;
    for (int64_t t = warp; t < nitems; t += nwarps) {
        if (t < nsl) {  // SELL-32 slice: a thread per row, 8 independent loads per batch
            const int64_t ts = C.s_lo + t;
            const int64_t p = ts * 32 + lane, beg = C.slice_ptr[ts];
            const int width = (int)((C.slice_ptr[ts + 1] - beg) >> 5);
            i128 acc[NC];
#pragma unroll
            for (int k = 0; k < NC; k++) acc[k] = 0;
            constexpr int SB = (NC == 1 || XS) ? 8 : CS_SB4;  // SELL columns per batch (registers: NC = 4 holds 4 x-rows each)
            for (int q = 0; q < width; q += SB) {
                int cc[SB];
                double wv[SB];
#pragma unroll
                for (int uu = 0; uu < SB; uu++) {
                    cc[uu] = 0;
                    wv[uu] = 0.0;
                    if (q + uu < width) {
                        cc[uu] = __ldcs(&C.ell_col[beg + (int64_t)(q + uu) * 32 + lane]);
                        wv[uu] = __ldcs(&C.ell_w[beg + (int64_t)(q + uu) * 32 + lane]);
                    }
                }
#pragma unroll
                for (int uu = 0; uu < SB; uu++)
                    if (q + uu < width) cs_gather<NC>(x, cc[uu], wv[uu], elo, s2, acc);
            }
            double ya = 0.0;
            if (p < C.nshort) ya = cs_epilogue<NC, MODE>(p, acc, elo, C, x, rs, vp, bprev, y, W);
            if (MODE == CS_LANCZOS) warp_atomic_max(&st->maxy, ya);
        } else {  // a 1024-entry chunk of a long row: warp-wide, int128 partials combined by the last arrival
            const int64_t c = t - nsl;
            const int64_t p = C.crow[c];
            if (p < C.p_lo || p >= C.p_hi) continue;  // another setup rank's long row (warp-uniform)
            const int64_t j = C.cidx[c], rb = C.srp[p], re = C.srp[p + 1];
            const int64_t b = rb + j * LCHUNK, e = min(re, b + LCHUNK);
            i128 acc[NC];
#pragma unroll
            for (int k = 0; k < NC; k++) acc[k] = 0;
            // 8 (col, w) loads and then 8 gathers in flight per lane (long rows of
            // aggregated levels carry most entries; the sum is order-free)
            constexpr int U = NC == 1 ? 8 : 2;
            for (int64_t k0 = b + lane; k0 < e; k0 += 32 * U) {
                int32_t cc[U];
                double wv[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int64_t k = k0 + 32 * u;
                    cc[u] = k < e ? __ldcs(&C.scol[k]) : 0;
                    wv[u] = k < e ? __ldcs(&C.sw[k]) : 0.0;
                }
                CsX<NC> xv[U];
#pragma unroll
                for (int u = 0; u < U; u++)
                    if (k0 + 32 * u < e) xv[u] = cs_load<NC>(x, cc[u]);
#pragma unroll
                for (int u = 0; u < U; u++)
                    if (k0 + 32 * u < e)
#pragma unroll
                        for (int kk = 0; kk < NC; kk++) acc[kk] += canon_q_s(__dmul_rn(wv[u], xv[u].v[kk]), s2, elo);
            }
#pragma unroll
            for (int k = 0; k < NC; k++) acc[k] = warp_sum_i128(acc[k]);
            const int slot = C.cslot[c];
            bool fin = slot < 0;
            if (!fin) {
                const int nch = (int)((re - rb + LCHUNK - 1) / LCHUNK);
                int last = 0;
                if (lane == 0) {
                    for (int k = 0; k < NC; k++) C.cpart[NC * c + k] = to_I128(acc[k]);
                    __threadfence();
                    last = atomicAdd(&C.ccnt[slot], 1) == nch - 1;
                }
                last = __shfl_sync(0xffffffffu, last, 0);
                if (last) {
                    __threadfence();
                    if (lane == 0) {
                        for (int k = 0; k < NC; k++) acc[k] = 0;
                        for (int64_t q = c - j; q < c - j + nch; q++)
                            for (int k = 0; k < NC; k++) {
                                I128 pv;
                                pv.lo = __ldcg(&C.cpart[NC * q + k].lo);
                                pv.hi = __ldcg(&C.cpart[NC * q + k].hi);
                                acc[k] += from_I128(pv);
                            }
                        C.ccnt[slot] = 0;
                    }
                    fin = true;
                }
            }
            if (fin && lane == 0) {
                const double ya = cs_epilogue<NC, MODE>(p, acc, elo, C, x, rs, vp, bprev, y, W);
                if (MODE == CS_LANCZOS) atomicMax(&st->maxy, (unsigned long long)__double_as_longlong(ya));
            }
        }
    }
}
static CStore cstore_of(const Level &L, I128 *cpart) {
    CStore C;
    C.nslices = L.nslices;
    C.nshort = L.c_end[0];
    C.nchunks = L.nchunks;
    C.slice_ptr = L.slice_ptr;
    C.ell_col = L.ell_col;
    C.ell_w = L.ell_w;
    C.srp = L.srp;
    C.scol = L.scol;
    C.sw = L.sw;
    C.sd = L.sd;
    C.crow = L.chunk_row;
    C.cidx = L.chunk_idx;
    C.cslot = L.chunk_slot;
    C.ccnt = L.chunk_cnt;
    C.cpart = cpart;
    C.s_lo = 0;
    C.s_hi = L.nslices;
    C.p_lo = 0;
    C.p_hi = (int64_t)1 << 62;
    return C;
}
// N1: a level's solve storage split over the setup ranks for the test-vector
// sweeps: slices by entries (cum = slice_ptr), long rows [c_end[0], n) by
// entries (cum = srp); out = P+1 slice bounds, then P+1 long-row bounds
__global__ void k_split_store(int64_t nslices, const int64_t *__restrict__ slice_ptr, int64_t nshort, int64_t n,
                              const int64_t *__restrict__ srp, int P, int64_t *__restrict__ out) {
    const int r = threadIdx.x;
    if (r > P) return;
    out[r] = split_bound(r, P, nslices, [&](int64_t o) { return slice_ptr[o]; });
    out[P + 1 + r] = nshort + split_bound(r, P, n - nshort, [&](int64_t o) { return srp[nshort + o] - srp[nshort]; });
}
struct StoreSplit {
    bool on = false;
    int P = 1;
    std::vector<int64_t> sb, lb;  // slice bounds, long-row (storage row) bounds
    std::vector<int> mine{0};
    CStore range(CStore C, int r) const {
        C.s_lo = sb[r];
        C.s_hi = sb[r + 1];
        C.p_lo = lb[r];
        C.p_hi = lb[r + 1];
        return C;
    }
    unsigned grid(const CStore &C, int64_t nchunks) const {
        return grid_for((C.s_hi - C.s_lo + nchunks / P + 1) * 32, 256, 148 * 8);
    }
    // share rows of a storage-order array of rsz bytes per row: the SELL rows,
    // then the long rows of every rank
    void share(void *buf, int64_t rsz, int64_t nshort, cudaStream_t s) const {
        if (!on) return;
        std::vector<int64_t> a(P + 1), b(P + 1);
        for (int r = 0; r <= P; r++) {
            a[r] = rsz * std::min<int64_t>(32 * sb[r], nshort);
            b[r] = rsz * lb[r];
        }
        setup_share(buf, a, s);
        setup_share(buf, b, s);
    }
};
static StoreSplit store_split(const Level &L, cudaStream_t s) {
    StoreSplit T;
    T.sb = {0, L.nslices};
    T.lb = {L.c_end[0], L.n};
    if (!dsetup_split(L.nnz)) return T;
    T.on = true;
    T.P = setup_nranks();
    T.mine = setup_local_ranks();
    DBuf<int64_t> b(2 * (T.P + 1), s);
    k_split_store<<<1, 64, 0, s>>>(L.nslices, L.slice_ptr, L.c_end[0], L.n, L.srp, T.P, b.p); ++g_kl;
    LAP_CHECK_LAUNCH();
    std::vector<int64_t> hb(2 * (T.P + 1));
    LAP_CUDA(cudaMemcpyAsync(hb.data(), b.p, 8 * hb.size(), cudaMemcpyDeviceToHost, s));
    LAP_CUDA(cudaStreamSynchronize(s));
    T.sb.assign(hb.begin(), hb.begin() + T.P + 1);
    T.lb.assign(hb.begin() + T.P + 1, hb.end());
    return T;
}
static unsigned cstore_grid(const Level &L) { return grid_for((L.nslices + L.nchunks) * 32, 256, 148 * 8); }

// pass C: acc_a += q(fl(y v))
__global__ void __launch_bounds__(256) k_lzc_alpha(int64_t n, const double *__restrict__ y,
                                                   const double *__restrict__ v, LzState *st) {
    if (st->stop) return;
    const int ey = ebound_dev(__longlong_as_double((long long)st->maxy));
    const int elo = canon_elo(ey + 2, n);
    i128 acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += canon_q(__dmul_rn(y[i], v[i]), elo);
    block_add_i128(&st->acc_a, acc);
}
// pass D: alpha, y -= alpha v, acc_b += q(y^2)
__global__ void __launch_bounds__(256) k_lzc_update(int64_t n, double *__restrict__ y, const double *__restrict__ v,
                                                    LzState *st) {
    if (st->stop) return;
    const int ey = ebound_dev(__longlong_as_double((long long)st->maxy));
    const double a = canon_result(from_I128(st->acc_a), canon_elo(ey + 2, n));
    const int ea = ebound_dev(fabs(a));
    const int elo = canon_elo(2 * ((ey + 1 > ea + 2 ? ey + 1 : ea + 2) + 2), n);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->alpha = a;
        st->elo_b = elo;
    }
    i128 acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double yi = __dsub_rn(y[i], __dmul_rn(a, v[i]));
        y[i] = yi;
        acc += canon_q(__dmul_rn(yi, yi), elo);
    }
    block_add_i128(&st->acc_b, acc);
}
// largest eigenvalue of the k x k tridiagonal by Sturm bisection (one thread)
__global__ void k_tridiag_max(const double *alpha, const double *beta, const int *kp, double *out) {
    int k = *kp;
    if (k <= 0) { *out = 0.0; return; }
    double lo = alpha[0], hi = alpha[0];
    for (int i = 0; i < k; i++) {
        double r = (i > 0 ? fabs(beta[i - 1]) : 0.0) + (i < k - 1 ? fabs(beta[i]) : 0.0);
        lo = fmin(lo, alpha[i] - r);
        hi = fmax(hi, alpha[i] + r);
    }
    for (int it = 0; it < 200; it++) {
        double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        int le = 0;
        double q = 1.0;
        for (int i = 0; i < k; i++) {
            q = (alpha[i] - mid) - (i > 0 ? beta[i - 1] * beta[i - 1] / q : 0.0);
            if (q == 0.0) q = -1e-300;
            le += q < 0.0;
        }
        if (le == k) hi = mid;
        else lo = mid;
    }
    *out = hi;
}

static int num_sms_dev() {
    static int v = 0;
    if (!v) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (v <= 0) v = 148;
    }
    return v;
}
// start vector and rs in the storage order (p holds logical vertex sid[p])
__global__ void k_lzc_init_s(int64_t n, uint64_t base, const int32_t *__restrict__ sid, const double *__restrict__ sd,
                             double *__restrict__ y, double *__restrict__ rs, double *__restrict__ vp, LzState *st,
                             int elo) {
    if (blockIdx.x == 0 && threadIdx.x == 0) st->elo_b = elo;  // (st zeroed by a memset before)
    i128 acc = 0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const double v = lz_start_value(base, sid[p]);
        y[p] = v;
        vp[p] = 0.0;
        rs[p] = __ddiv_rn(1.0, __dsqrt_rn(sd[p]));
        acc += canon_q(__dmul_rn(v, v), elo);
    }
    block_add_i128(&st->acc_b, acc);
}

// E_lo of the Lanczos SpMV instance on the device (no host round trip): the
// exponent bound ilogb(max w) + ilogb(max rs) + 3 of the products w_ij rs_j v_j
__global__ void k_lz_spmv_elo(const unsigned long long *mxrs, int ew, int64_t nnz, int *elo) {
    const double mr = __longlong_as_double((long long)*mxrs);
    *elo = canon_elo(ew + (mr > 0.0 ? ilogb(mr) : -1000) + 3, nnz);
}
// lambda-hat on the level's solve storage (built before this is called): the
// Lanczos vectors live in the storage order; every sum is a CanonSum, so the
// order changes no bit (the tridiagonal equals the oracle's).
// Enqueued on its own stream (build_hierarchy): lambda-hat is needed only by
// the solve, so the Lanczos steps of level l overlap the strength, voting and
// Galerkin work of levels >= l; it only reads the level's storage and has its
// own arrival counters; lambda-hat lands in *host_out (pinned) when s gets there.
static void lanczos(lap_hierarchy *h, Level &L, int l, cudaStream_t s, double *host_out) {
    const int64_t n = L.n, nnz = L.nnz;
    const int steps = h->p.lanczos_steps;
    DBuf<double> v(n, s), vp(n, s), y(n, s), u(n, s), rs(n, s), al(64, s), be(64, s), lam(1, s);
    DBuf<LzState> st(1, s);
    DBuf<int> kk(1, s);
    DBuf<I128> cpart(L.nchunks > 0 ? L.nchunks : 1, s);
    DBuf<int32_t> ccnt(L.nmulti > 0 ? L.nmulti : 1, s);  // not the sweeps' counters: they may run meanwhile
    LAP_CUDA(cudaMemsetAsync(ccnt.p, 0, sizeof(int32_t) * (size_t)(L.nmulti > 0 ? L.nmulti : 1), s));
    // no host synchronisation anywhere below: this runs on the side stream while
    // the host keeps enqueueing the setup's main work
    LAP_CUDA(cudaMemsetAsync(st.p, 0, sizeof(LzState), s));
    const uint64_t base = mix64(salt_of(h->p.seed, 4) ^ (uint64_t)(2 * l));
    const unsigned g = grid_for(n, 256, 148 * 8);
    k_lzc_init_s<<<g, 256, 0, s>>>(n, base, L.sid, L.sd, y.p, rs.p, vp.p, st.p, canon_elo(1, n)); ++g_kl;
    LAP_CHECK_LAUNCH();
    DBuf<unsigned long long> mxrs(1, s);
    DBuf<int> elo_d(1, s);
    LAP_CUDA(cudaMemsetAsync(mxrs.p, 0, sizeof(unsigned long long), s));
    k_max_abs<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(rs.p, n, mxrs.p); ++g_kl;
    k_lz_spmv_elo<<<1, 1, 0, s>>>(mxrs.p, L.maxw > 0.0 ? ilogb(L.maxw) : -1000, nnz, elo_d.p); ++g_kl;
    LAP_CHECK_LAUNCH();
    const int elo_spmv = 0;  // (read from elo_d by the SpMV)
    CStore C = cstore_of(L, cpart.p);
    C.ccnt = ccnt.p;
    CSweep W{};
    W.elo_p = elo_d.p;
    // N1: the SpMV of each step split over the setup ranks (rows of y shared,
    // max |y| combined: an exact max); the dots run on the whole vectors on every
    // rank.  Only in line on the setup stream (lanczos_in_line), and not on
    // shared-memory-x levels (small)
    const bool xs = L.smem_x && n <= SMEM_X_MAX;
    const StoreSplit T = xs ? StoreSplit{} : store_split(L, s);
    if (xs) {
        static bool attr = false;
        if (!attr) {
            LAP_CUDA(cudaFuncSetAttribute(k_cspmv_store<1, CS_LANCZOS, true>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(8 * SMEM_X_MAX)));
            attr = true;
        }
    }
    for (int j = 0; j < steps && j < 64; j++) {
        k_lzc_next<<<g, 256, 0, s>>>(n, j == 0, 0, y.p, v.p, vp.p, u.p, rs.p, st.p, al.p, be.p); ++g_kl;
        if (xs)
            k_cspmv_store<1, CS_LANCZOS, true><<<num_sms_dev(), 1024, 8 * n, s>>>(C, u.p, rs.p, vp.p, elo_spmv, st.p,
                                                                                  y.p, W, n);
        else if (!T.on)
            k_cspmv_store<1, CS_LANCZOS><<<cstore_grid(L), 256, 0, s>>>(C, u.p, rs.p, vp.p, elo_spmv, st.p, y.p, W, 0);
        else
            for (int r : T.mine) {
                const CStore Cr = T.range(C, r);
                k_cspmv_store<1, CS_LANCZOS><<<T.grid(Cr, L.nchunks), 256, 0, s>>>(Cr, u.p, rs.p, vp.p, elo_spmv,
                                                                                   st.p, y.p, W, 0);
            }
        ++g_kl;
        if (T.on) {
            T.share(y.p, 8, L.c_end[0], s);
            setup_max_u64(&st.p->maxy, s);
        }
        k_lzc_alpha<<<g, 256, 0, s>>>(n, y.p, v.p, st.p); ++g_kl;
        k_lzc_update<<<g, 256, 0, s>>>(n, y.p, v.p, st.p); ++g_kl;
        LAP_CHECK_LAUNCH();
    }
    k_lzc_next<<<g, 256, 0, s>>>(n, 0, 1, y.p, v.p, vp.p, u.p, rs.p, st.p, al.p, be.p); ++g_kl;  // record the last step
    LAP_CUDA(cudaMemcpyAsync(kk.p, &st.p->k, sizeof(int), cudaMemcpyDeviceToDevice, s));
    k_tridiag_max<<<1, 1, 0, s>>>(al.p, be.p, kk.p, lam.p); ++g_kl;
    LAP_CHECK_LAUNCH();
    h->cur.edges += (int64_t)steps * L.nnz;
    LAP_CUDA(cudaMemcpyAsync(host_out, lam.p, sizeof(double), cudaMemcpyDeviceToHost, s));
}
// the side stream of the Lanczos runs (joined, and its resources released, at
// the end of the setup or when an error unwinds it)
struct LanczosStream {
    cudaStream_t ls = nullptr;
    cudaEvent_t ev = nullptr;
    double *lam = nullptr;  // pinned, one per level
    std::vector<int> levels;
    void start(int l, cudaStream_t s) {  // after the level's storage is enqueued on s
        if (!ls) {
            LAP_CUDA(cudaStreamCreateWithFlags(&ls, cudaStreamNonBlocking));
            LAP_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            LAP_CUDA(cudaMallocHost(&lam, sizeof(double) * 64));
        }
        LAP_CUDA(cudaEventRecord(ev, s));
        LAP_CUDA(cudaStreamWaitEvent(ls, ev, 0));
        levels.push_back(l);
    }
    void join(lap_hierarchy *h, cudaStream_t s) {  // s continues after every Lanczos run
        if (!ls) return;
        LAP_CUDA(cudaStreamSynchronize(ls));
        for (int l : levels) h->lev[l].lambda = lam[l];
        LAP_CUDA(cudaEventRecord(ev, ls));
        LAP_CUDA(cudaStreamWaitEvent(s, ev, 0));
    }
    ~LanczosStream() {
        if (ls) {
            cudaStreamSynchronize(ls);
            cudaStreamDestroy(ls);
            cudaEventDestroy(ev);
            cudaFreeHost(lam);
        }
    }
};

// =========================================================================
// O-S10 coarsest pseudo-inverse (O-R26): ground the last vertex,
// in-place Gauss-Jordan inverse of the SPD block, project with I - J/n.
// =========================================================================

__global__ void k_dense_fill(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *w,
                             const double *d, double *A) {
    int64_t g = n - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g; i += (int64_t)gridDim.x * blockDim.x) {
        A[i * g + i] = d[i];
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; k++)
            if (col[k] < g) A[i * g + col[k]] = -w[k];
    }
}
// one pivot step of the in-place Gauss-Jordan (sweep) inversion
__global__ void k_gj_pivot_row(int64_t g, int64_t kk, double *A, double *colbuf, double *rowbuf) {
    double piv = A[kk * g + kk];
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < g; t += (int64_t)gridDim.x * blockDim.x) {
        colbuf[t] = A[t * g + kk];
        rowbuf[t] = (t == kk) ? 1.0 / piv : A[kk * g + t] / piv;
    }
}
__global__ void k_gj_update(int64_t g, int64_t kk, double *A, const double *colbuf, const double *rowbuf) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < g * g; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = t / g, j = t % g;
        if (i == kk) {
            A[t] = rowbuf[j];
        } else {
            double c = colbuf[i];
            A[t] = (j == kk) ? -c * rowbuf[kk] : A[t] - c * rowbuf[j];
        }
    }
}
// single-CTA variant for small g (one launch for all pivots)
__global__ void __launch_bounds__(1024, 1) k_gj_small(int64_t g, double *A, double *colbuf, double *rowbuf) {
    for (int64_t kk = 0; kk < g; kk++) {
        double piv = A[kk * g + kk];
        for (int64_t t = threadIdx.x; t < g; t += blockDim.x) {
            colbuf[t] = A[t * g + kk];
            rowbuf[t] = (t == kk) ? 1.0 / piv : A[kk * g + t] / piv;
        }
        __syncthreads();
        for (int64_t t = threadIdx.x; t < g * g; t += blockDim.x) {
            int64_t i = t / g, j = t % g;
            if (i == kk) A[t] = rowbuf[j];
            else {
                double c = colbuf[i];
                A[t] = (j == kk) ? -c * rowbuf[kk] : A[t] - c * rowbuf[j];
            }
        }
        __syncthreads();
    }
}
// G = [[Ainv,0],[0,0]] (n x n); pinv = G - r_i/n - c_j/n + tot/n^2 (row sums r, col sums c)
__global__ void k_pinv_sums(int64_t n, const double *Ai, double *rsum, double *csum) {
    int64_t g = n - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double r = 0.0, c = 0.0;
        if (i < g)
            for (int64_t j = 0; j < g; j++) {
                r += Ai[i * g + j];
                c += Ai[j * g + i];
            }
        rsum[i] = r;
        csum[i] = c;
    }
}
__global__ void k_pinv_total(int64_t n, const double *rsum, double *tot) {
    double t = 0.0;
    for (int64_t i = 0; i < n; i++) t += rsum[i];
    *tot = t;
}
__global__ void k_pinv_assemble(int64_t n, const double *Ai, const double *rsum, const double *csum,
                                const double *tot, double *P) {
    int64_t g = n - 1;
    double T = *tot, nn = (double)n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * n; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = t / n, j = t % n;
        double G = (i < g && j < g) ? Ai[i * g + j] : 0.0;
        P[t] = G - rsum[i] / nn - csum[j] / nn + T / (nn * nn);
    }
}

static void coarse_pinv(Level &L, cudaStream_t s) {
    int64_t n = L.n;
    L.pinv = (double *)dalloc(sizeof(double) * (size_t)(n * n), s);
    if (n <= 1) {
        LAP_CUDA(cudaMemsetAsync(L.pinv, 0, sizeof(double) * (size_t)(n * n > 0 ? n * n : 1), s));
        return;
    }
    int64_t g = n - 1;
    DBuf<double> A(g * g, s), cb(g, s), rb(g, s), rsum(n, s), csum(n, s), tot(1, s);
    LAP_CUDA(cudaMemsetAsync(A.p, 0, sizeof(double) * (size_t)(g * g), s));
    k_dense_fill<<<grid_for(g, 128, 148 * 4), 128, 0, s>>>(n, L.row_ptr, L.col, L.w, L.d, A.p); ++g_kl;
    if (g <= 1024) {
        k_gj_small<<<1, 1024, 0, s>>>(g, A.p, cb.p, rb.p); ++g_kl;
    } else {
        for (int64_t kk = 0; kk < g; kk++) {
            k_gj_pivot_row<<<grid_for(g, 256, 148 * 4), 256, 0, s>>>(g, kk, A.p, cb.p, rb.p); ++g_kl;
            k_gj_update<<<grid_for(g * g, 256, 148 * 16), 256, 0, s>>>(g, kk, A.p, cb.p, rb.p); ++g_kl;
        }
    }
    k_pinv_sums<<<grid_for(n, 128, 148 * 4), 128, 0, s>>>(n, A.p, rsum.p, csum.p); ++g_kl;
    k_pinv_total<<<1, 1, 0, s>>>(n, rsum.p, tot.p); ++g_kl;
    k_pinv_assemble<<<grid_for(n * n, 256, 148 * 8), 256, 0, s>>>(n, A.p, rsum.p, csum.p, tot.p, L.pinv); ++g_kl;
    LAP_CHECK_LAUNCH();
}

// =========================================================================
// per-level builders
// =========================================================================

static int64_t elim_select(lap_hierarchy *h, Level &L, DBuf<uint8_t> &F, cudaStream_t s) {
    F.alloc(L.n, s);
    DBuf<unsigned long long> nF(1, s);
    LAP_CUDA(cudaMemsetAsync(nF.p, 0, 8, s));
    const RowSplit R = row_split(L.n, L.nnz, L.row_ptr, s);  // N1: rows over the setup ranks
    for (int r : R.mine) {
        const int64_t r0 = R.rb[r], r1 = R.rb[r + 1];
        k_elim_select<<<grid_for(r1 - r0, 256, 148 * 16), 256, 0, s>>>(r0, r1, L.row_ptr, L.col,
                                                                        h->p.elim_max_degree, salt_of(h->p.seed, 2),
                                                                        F.p, nF.p); ++g_kl;
    }
    LAP_CHECK_LAUNCH();
    if (R.on) {
        setup_share(F.p, R.rb, s);  // one byte per row
        setup_sum_u64(nF.p, 1, s);
    }
    h->cur.edges += L.nnz;
    return (int64_t)d2h_scalar(nF.p, s);
}

static void build_ct_lists(Level &L, const uint8_t *Fp, int64_t nc, cudaStream_t s);
static void build_elim_level(lap_hierarchy *h, Level &L, const DBuf<uint8_t> &F, int64_t nF, Level &N,
                             cudaStream_t s) {
    int64_t n = L.n, nc = n - nF;
    L.kind = KIND_ELIM;
    L.nF = nF;
    DBuf<int64_t> isc(n, s), cpos(n, s), isf(n, s), fpos(n, s);
    unsigned g = grid_for(n, 256, 148 * 16);
    k_flag_not<<<g, 256, 0, s>>>(n, F.p, isc.p); ++g_kl;
    k_flag_f<<<g, 256, 0, s>>>(n, F.p, isf.p); ++g_kl;
    LAP_CHECK_LAUNCH();
    exclusive_scan_i64(isc.p, cpos.p, n, s);
    exclusive_scan_i64(isf.p, fpos.p, n, s);
    L.fmap = (int32_t *)dalloc(sizeof(int32_t) * n, s);
    L.cid = (int32_t *)dalloc(sizeof(int32_t) * (nc + 1), s);
    L.fid = (int32_t *)dalloc(sizeof(int32_t) * (nF + 1), s);
    k_fmap<<<g, 256, 0, s>>>(n, F.p, cpos.p, fpos.p, L.fmap, L.cid, L.fid); ++g_kl;
    LAP_CHECK_LAUNCH();
    // the Schur complement, row by row of C (batched terms, CanonSum per entry)
    {
        TermSrc S;
        S.kind = SRC_SCHUR;
        S.rp = L.row_ptr;
        S.col = L.col;
        S.w = L.w;
        S.d = L.d;
        S.vfine = L.cid;
        S.F = F.p;
        S.fmap = L.fmap;
        const int cb = bitlen_u64((uint64_t)(nc > 0 ? nc : 1));
        csr_from_source(S, nc, nc, cb, ilogb_pos(L.maxw) + 1, 4 * L.nnz, true, N, s);
    }
    build_ct_lists(L, F.p, nc, s);
    h->cur.edges += L.nnz;
}

// transposed L_FC for the restriction P^T b: per C vertex its F neighbours and
// w_fc / d_f (logical numbering)
static void build_ct_lists(Level &L, const uint8_t *Fp, int64_t nc, cudaStream_t s) {
    const int64_t n = L.n;
    const int G = group_size(n, L.nnz);
    struct { const uint8_t *p; } F{Fp};
    DBuf<int64_t> tc(nc + 1, s);
    LAP_CUDA(cudaMemsetAsync(tc.p, 0, sizeof(int64_t) * (nc + 1), s));
    LAUNCH_G(G, k_ct_count, nc, s, nc, L.cid, L.row_ptr, L.col, F.p, tc.p);
    L.ct_ptr = (int64_t *)dalloc(sizeof(int64_t) * (nc + 1), s);
    exclusive_scan_i64(tc.p, L.ct_ptr, nc + 1, s);
    int64_t TT = d2h_scalar(L.ct_ptr + nc, s);
    L.ct_f = (int32_t *)dalloc(sizeof(int32_t) * (TT + 1), s);
    L.ct_coef = (double *)dalloc(sizeof(double) * (TT + 1), s);
    LAUNCH_G(G, k_ct_fill, nc, s, nc, L.cid, L.row_ptr, L.col, L.w, L.d, F.p, L.ct_ptr, L.ct_f, L.ct_coef);
    LAP_CHECK_LAUNCH();
}

// strength + voting for one attempt; returns m, fills L.agg
static int64_t aggregate_attempt(lap_hierarchy *h, Level &L, int l, int attempt, DBuf<double> &S, cudaStream_t s) {
    int64_t n = L.n, nnz = L.nnz;
    const lap_params &p = h->p;
    unsigned ge = grid_for(n, 256, 148 * 16);
    const int G = group_size(n, nnz, L.maxdeg <= SHORT_MAX);
    // lanes per row of the affinity / vote passes (LAP_AFF_G / LAP_VOTE_G: experiments)
    auto env_g = [&](const char *name) {
        const char *e = getenv(name);
        const int v = e ? atoi(e) : 0;
        return (v == 1 || v == 2 || v == 4 || v == 8 || v == 16 || v == 32) ? v : G;
    };
    // votes: at most 8 lanes per row (the group argmax is most of a round's
    // instructions: cfg 4 G = 16 -> 8 setup 76.0 -> 73.4 ms, cfg 3 neutral;
    // profiles/r02/gsweep_summary.txt)
    const int Ga = env_g("LAP_AFF_G"), Gv = getenv("LAP_VOTE_G") ? env_g("LAP_VOTE_G") : std::min(G, 8);
    // test vectors: swept on the solve storage (canonical sums:
    // the order is free), then laid out in the logical order for the affinity
    DBuf<double> X(4 * n, s), Xn(4 * n, s), M(n, s);
    uint64_t base = mix64(salt_of(p.seed, 3) ^ (uint64_t)(2 * l + attempt));
    k_tv_init_s<<<grid_for(4 * n, 256, 148 * 16), 256, 0, s>>>(n, base, L.sid, X.p); ++g_kl;
    LAP_CHECK_LAUNCH();
    int ew = ilogb_pos(L.maxw);
    DBuf<unsigned long long> mxb(1, s);
    DBuf<int> elo(1, s);
    // long rows (deg > SETUP_LONG): LCHUNK warp chunks (logical CSR)
    int32_t *lc_row = nullptr, *lc_idx = nullptr, *lc_slot = nullptr, *lc_cnt = nullptr;
    double *lc_dummy = nullptr;
    const int64_t nlc = L.maxdeg <= SETUP_LONG ? 0
                        : build_chunks(L.row_ptr, 0, n, SETUP_LONG, &lc_row, &lc_idx, &lc_slot, &lc_dummy, &lc_cnt, s);
    struct FreeLc {
        void *p[5];
        cudaStream_t s;
        ~FreeLc() {
            for (void *q : p) dfree(q, s);
        }
    } free_lc{{lc_row, lc_idx, lc_slot, lc_cnt, lc_dummy}, s};
    DBuf<I128> cpart(4 * (L.nchunks > 0 ? L.nchunks : 1), s);
    // N1: each setup rank sweeps its slices and long rows (ranges of equal entry
    // counts, k_split_store); the rows' new vectors (32 B each) are shared after
    // every sweep.  Per-row CanonSums: bit-identical to one GPU.
    const StoreSplit T = store_split(L, s);
    for (int sw = 0; sw < p.tv_sweeps; sw++) {
        // CanonSum instance of this sweep: e_max from the exact max |x| (O-S11), computed on
        // the device (no host round trip)
        LAP_CUDA(cudaMemsetAsync(mxb.p, 0, sizeof(unsigned long long), s));
        k_max_abs<<<grid_for(4 * n, 256, 148 * 8), 256, 0, s>>>(X.p, 4 * n, mxb.p); ++g_kl;
        k_tv_elo<<<1, 1, 0, s>>>(mxb.p, ew, nnz, elo.p); ++g_kl;
        const CSweep W{X.p, Xn.p, elo.p, p.tv_omega};
        for (int r : T.mine) {
            const CStore C = T.range(cstore_of(L, cpart.p), r);
            k_cspmv_store<4, CS_SWEEP><<<T.grid(C, L.nchunks), 256, 0, s>>>(C, X.p, nullptr, nullptr, 0, nullptr,
                                                                            nullptr, W, 0);
            ++g_kl;
        }
        LAP_CHECK_LAUNCH();
        T.share(Xn.p, 32, L.c_end[0], s);  // n x 4 doubles
        std::swap(X.p, Xn.p);
        h->cur.edges += nnz;
    }
    // storage order -> logical order (Xn is free)
    k_tv_unpermute<<<grid_for(4 * n, 256, 148 * 16), 256, 0, s>>>(n, L.sid, X.p, Xn.p); ++g_kl;
    std::swap(X.p, Xn.p);
    tmark("  test vectors");
    // affinity + normalisation; C_ij and M_i of each setup rank's
    // rows (N1), shared before the (replicated, entry-parallel) normalisation
    const RowSplit R = row_split(n, nnz, L.row_ptr, s);
    if (nlc > 0) LAP_CUDA(cudaMemsetAsync(M.p, 0, sizeof(double) * n, s));
    for (int r : R.mine) {
        const int64_t r0 = R.rb[r], r1 = R.rb[r + 1];
        LAUNCH_G(Ga, k_affinity, r1 - r0, s, r0, r1, L.row_ptr, L.col, X.p, p.affinity_power, S.p, M.p);
        if (nlc > 0) {
            k_affinity_long<<<grid_for(nlc * 32, 256, 148 * 16), 256, 0, s>>>(
                nlc, lc_row, lc_idx, r0, r1, L.row_ptr, L.col, X.p, p.affinity_power, S.p, (unsigned long long *)M.p);
            ++g_kl;
        }
    }
    if (R.on) {
        setup_share(S.p, R.bytes(R.eb, 8), s);
        setup_share(M.p, R.bytes(R.rb, 8), s);
    }
    if (nnz > 0) {
        k_normalize<<<grid_for(nnz, 256, 148 * 16), 256, 0, s>>>(n, nnz, L.rowof, L.col, M.p, S.p);
        ++g_kl;
    }
    LAP_CHECK_LAUNCH();
    h->cur.edges += 2 * nnz;
    tmark("  affinity");
    // voting rounds (Alg. 3)
    DBuf<int8_t> st(n, s), nst(n, s);
    DBuf<int32_t> idx(n, s), nidx(n, s), votes(n, s);
    k_vote_init<<<ge, 256, 0, s>>>(n, st.p, idx.p, votes.p); ++g_kl;
    // N1 over NCCL: this rank's own votes accumulate in vloc, votes = their sum
    // over the ranks (K4); otherwise every range adds into votes directly
    const bool vsum = R.on && setup_nccl();
    DBuf<int32_t> vloc(vsum ? n : 1, s);
    if (vsum) LAP_CUDA(cudaMemsetAsync(vloc.p, 0, sizeof(int32_t) * n, s));
    int32_t *vp = vsum ? vloc.p : votes.p;
    DBuf<unsigned long long> vbest(nlc > 0 ? n : 1, s);
    DBuf<int32_t> vbestj(nlc > 0 ? n : 1, s);
    if (nlc > 0) {
        k_vote_long_init<<<ge, 256, 0, s>>>(n, vbest.p, vbestj.p);
        ++g_kl;
    }
    // the active list: this process's rows (all of them without a communicator or
    // on a virtual grid), compacted after every round
    const int64_t alo = R.rb[R.mine.front()], ahi = R.rb[R.mine.back() + 1];
    DBuf<int32_t> alist(ahi - alo, s), blist(ahi - alo, s), acnt(2, s);
    k_act_init<<<1, 1, 0, s>>>(alo, ahi, acnt.p); ++g_kl;
    int32_t *cur = nullptr, *nxt = alist.p, *ccur = acnt.p, *cnxt = acnt.p + 1;
    const char *vle = getenv("LAP_VOTE_LIST");  // 0 / 1: force (tests); default by row length
    const bool vlist = vle ? vle[0] == '1' : nnz >= 10 * n;
    for (int t = 1; t <= p.vote_rounds; t++) {
        double filt = ldexp(1.0, -t);
        LAUNCH_G(Gv, k_vote_round_list, ahi - alo, s, cur, alo, ccur, L.row_ptr, L.col, S.p, filt, st.p, nst.p, nidx.p,
                 vp);
        if (nlc > 0) {
            for (int r : R.mine) {
                const int64_t r0 = R.rb[r], r1 = R.rb[r + 1];
                const unsigned gc = grid_for(nlc * 32, 256, 148 * 16);
                k_vote_long_max<<<gc, 256, 0, s>>>(nlc, lc_row, lc_idx, r0, r1, L.row_ptr, L.col, S.p, filt, st.p,
                                                   vbest.p);
                k_vote_long_argj<<<gc, 256, 0, s>>>(nlc, lc_row, lc_idx, r0, r1, L.row_ptr, L.col, S.p, filt, st.p,
                                                    vbest.p, vbestj.p);
                k_vote_long_apply<<<grid_for(nlc, 256, 148 * 8), 256, 0, s>>>(
                    nlc, lc_row, lc_idx, r0, r1, st.p, idx.p, vbest.p, vbestj.p, nst.p, nidx.p, vp);
                g_kl += 3;
            }
        }
        if (vsum) setup_sum_i32(vloc.p, votes.p, n, s);  // the round's votes summed over the ranks (K4)
        if (vlist) LAP_CUDA(cudaMemsetAsync(cnxt, 0, sizeof(int32_t), s));
        k_vote_commit<<<grid_for(ahi - alo, 256, 148 * 8), 256, 0, s>>>(cur, alo, ccur, nst.p, nidx.p, votes.p,
                                                                        p.vote_threshold, st.p, idx.p,
                                                                        vlist ? nxt : nullptr, cnxt);
        ++g_kl;
        LAP_CHECK_LAUNCH();
        if (R.on) {  // every rank's rows of the committed states (NCCL; no-op on one process)
            setup_share(st.p, R.rb, s);
            setup_share(idx.p, R.bytes(R.rb, 4), s);
        }
        if (vlist) {
            cur = nxt;  // the list just written; the next round writes the other one
            nxt = cur == alist.p ? blist.p : alist.p;
            std::swap(ccur, cnxt);
        }
        h->cur.edges += nnz;
    }
    tmark("  votes");
    // renumber roots by ascending id (O-R15)
    DBuf<int64_t> flag(n + 1, s), rid(n + 1, s);
    LAP_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int64_t) * (n + 1), s));
    k_root_flags<<<ge, 256, 0, s>>>(n, st.p, flag.p); ++g_kl;
    exclusive_scan_i64(flag.p, rid.p, n + 1, s);
    if (!L.agg) L.agg = (int32_t *)dalloc(sizeof(int32_t) * n, s);
    k_agg_ids<<<ge, 256, 0, s>>>(n, st.p, idx.p, rid.p, L.agg); ++g_kl;
    LAP_CHECK_LAUNCH();
    return d2h_scalar(rid.p + n, s);
}

__global__ void k_iota_agg(int64_t n, const int32_t *agg, uint32_t *key, int32_t *ids) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        key[i] = (uint32_t)agg[i];
        ids[i] = (int32_t)i;
    }
}
__global__ void k_mem_ptr(int64_t m, int64_t n, const uint32_t *skey, int64_t *ptr) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a <= m; a += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)skey[mid] < a) lo = mid + 1;
            else hi = mid;
        }
        ptr[a] = lo;
    }
}

// ---- aggregate-ordered Galerkin (N3: "a matrix-matrix product
// that exploits the special structure of R and P"): the members of every
// aggregate are consecutive member slots, so emitting the fine entries slot
// by slot (self-terms agg_j == a dropped, positions by a prefix sum of the
// per-slot counts -- deterministic, no atomics) leaves the terms of coarse row
// a contiguous; only each row's terms need sorting by agg_j (per-row sorts by
// length class, sort_rows), not one device-wide 64-bit-key radix sort of all
// terms.  Each (a, b) entry is then one CanonSum of exactly the method's
// multiset of terms (O-R23): bit-identical to the global-sort path.
template <int G>
__global__ void k_gal_slot_cnt(int64_t ns, const int32_t *__restrict__ members, const uint32_t *__restrict__ slot_agg,
                               const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                               const int32_t *__restrict__ agg, int64_t *__restrict__ cnt) {
    GROUP_LOOP_BEGIN(G, ns)
    int64_t c = 0;
    int32_t fi = 0, a = 0;
    if (live) {
        fi = members[i];
        a = (int32_t)slot_agg[i];
        for (int64_t k = rp[fi] + gl; k < rp[fi + 1]; k += G) c += agg[col[k]] != a;
    }
    c = grp_sum<G>(c);
    if (live && gl == 0) cnt[i] = c;
    GROUP_LOOP_END
}
template <int G>
__global__ void k_gal_slot_emit(int64_t ns, const int32_t *__restrict__ members, const uint32_t *__restrict__ slot_agg,
                                const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                                const double *__restrict__ w, const int32_t *__restrict__ agg,
                                const int64_t *__restrict__ pv, int32_t *__restrict__ tk, double *__restrict__ tv) {
    GROUP_LOOP_BEGIN(G, ns)
    int64_t kb = 0, ke = 0, o = 0;
    int32_t a = 0;
    if (live) {
        const int32_t fi = members[i];
        a = (int32_t)slot_agg[i];
        kb = rp[fi];
        ke = rp[fi + 1];
        o = pv[i];
    }
    GROUP_COMPACT_ROW(G, kb, ke, o, agg[col[k]] != a, (tk[p] = agg[col[k]], tv[p] = w[k]))
    GROUP_LOOP_END
}
constexpr int64_t GAL_ORDERED_MAX_AVG = 256;  // terms per coarse row (average) for the ordered Galerkin
static bool gal_fast_enabled() {  // read per level (tests switch it inside one process)
    const char *e = getenv("LAP_GAL_FAST");  // 0: the batched global-sort path (tests, experiments)
    return !(e && e[0] == '0');
}
static void csr_combine_sorted(int64_t nrows, int cb, int64_t T, DBuf<uint64_t> &k2, DBuf<double> &v2, int e_max,
                               int64_t K, Level &out, cudaStream_t s, bool sums);
// local prefix of a slot range: pl[v] = pv[s0 + v] - pv[s0], v in [0, ns]
__global__ void k_sub_prefix(int64_t ns, const int64_t *__restrict__ pv, int64_t *__restrict__ pl) {
    const int64_t b = pv[0];
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= ns; v += (int64_t)gridDim.x * blockDim.x)
        pl[v] = pv[v] - b;
}
// row pointers of the coarse rows [alo, ahi): pa[a] = pl[mem_ptr[alo + a] - s0]
__global__ void k_gal_row_ptr_r(int64_t mr, const int64_t *__restrict__ mem_ptr, int64_t s0,
                                const int64_t *__restrict__ pl, int64_t *__restrict__ pa) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a <= mr; a += (int64_t)gridDim.x * blockDim.x)
        pa[a] = pl[mem_ptr[a] - s0];
}
template <int G>
__global__ void k_gal_keys(int64_t m, const int64_t *__restrict__ pa, const int32_t *__restrict__ sk, int cb,
                           uint64_t *__restrict__ key) {
    GROUP_LOOP_BEGIN(G, m)
    if (live)
        for (int64_t k = pa[i] + gl; k < pa[i + 1]; k += G) key[k] = ((uint64_t)i << cb) | (uint64_t)(uint32_t)sk[k];
    GROUP_LOOP_END
}
static void galerkin_fast(lap_hierarchy *h, Level &L, Level &N, const int32_t *members, const uint32_t *slot_agg,
                          const int64_t *mem_ptr, cudaStream_t s) {
    const int64_t n = L.n, m = L.m;
    const int cb = bitlen_u64((uint64_t)(m > 0 ? m : 1));
    const int G = group_size(n, L.nnz, L.maxdeg <= SHORT_MAX);
    const int e_max = ilogb_pos(L.maxw) + 1;
    DBuf<int64_t> cnt(n + 1, s), pv(n + 1, s);
    LAP_CUDA(cudaMemsetAsync(cnt.p + n, 0, sizeof(int64_t), s));
    LAUNCH_G(G, k_gal_slot_cnt, n, s, n, members, slot_agg, L.row_ptr, L.col, L.agg, cnt.p);
    exclusive_scan_i64(cnt.p, pv.p, n + 1, s);
    cnt.release();
    const int64_t Ttot = d2h_scalar(pv.p + n, s);
    // coarse rows [alo, ahi) -> out (local rows, no diagonal)
    auto range = [&](int64_t alo, int64_t ahi, Level &out) {
        const int64_t mr = ahi - alo;
        const int64_t s0 = d2h_scalar(mem_ptr + alo, s), s1 = d2h_scalar(mem_ptr + ahi, s), ns = s1 - s0;
        DBuf<int64_t> pl(ns + 1, s), pa(mr + 1, s);
        k_sub_prefix<<<grid_for(ns + 1, 256, 148 * 8), 256, 0, s>>>(ns, pv.p + s0, pl.p); ++g_kl;
        const int64_t T = d2h_scalar(pl.p + ns, s);
        DBuf<int32_t> tk(T + 1, s);
        DBuf<double> tv(T + 1, s);
        if (ns > 0) LAUNCH_G(G, k_gal_slot_emit, ns, s, ns, members + s0, slot_agg + s0, L.row_ptr, L.col, L.w, L.agg,
                             pl.p, tk.p, tv.p);
        k_gal_row_ptr_r<<<grid_for(mr + 1, 256, 148 * 8), 256, 0, s>>>(mr, mem_ptr + alo, s0, pl.p, pa.p); ++g_kl;
        LAP_CHECK_LAUNCH();
        pl.release();
        tmark("  galerkin: ordered emit");
        DBuf<int32_t> sk(T + 1, s);
        DBuf<double> sv(T + 1, s);
        sort_rows(mr, pa.p, T, cb, tk.p, tv.p, sk.p, sv.p, s);
        tk.release();
        tv.release();
        tmark("  galerkin: row sorts");
        DBuf<uint64_t> key(T + 1, s);
        if (T > 0) LAUNCH_G(group_size(mr, T), k_gal_keys, mr, s, mr, pa.p, sk.p, cb, key.p);
        LAP_CHECK_LAUNCH();
        sk.release();
        csr_combine_sorted(mr, cb, T, key, sv, e_max, L.nnz, out, s, false);
    };
    const int P = setup_nranks();
    if (dsetup_split(Ttot)) {
        build_split(m, split_bounds(m, P, pv.p, mem_ptr, s), N, s, range);
        return;
    }
    range(0, m, N);
    N.d = (double *)dalloc(sizeof(double) * (size_t)(m > 0 ? m : 1), s);
    row_sums(m, N.nnz, N.row_ptr, N.w, N.d, &N.maxw, s);
    tmark("  terms: row sums");
}

static void galerkin(lap_hierarchy *h, Level &L, Level &N, cudaStream_t s) {
    const int64_t n = L.n, m = L.m;
    // members of every aggregate, ascending (stable radix sort by aggregate id)
    DBuf<uint32_t> k1(n, s), k2(n, s);
    DBuf<int32_t> ids(n, s), members(n, s);
    DBuf<int64_t> mem_ptr(m + 1, s);
    k_iota_agg<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, L.agg, k1.p, ids.p); ++g_kl;
    {
        size_t bytes = 0;
        const int eb = bitlen_u64((uint64_t)(m > 0 ? m : 1));
        LAP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k1.p, k2.p, ids.p, members.p, n, 0, eb, s));
        DBuf<char> tmp((int64_t)bytes, s);
        LAP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, k1.p, k2.p, ids.p, members.p, n, 0, eb, s)); ++g_kl;
    }
    k_mem_ptr<<<grid_for(m + 1, 256, 148 * 8), 256, 0, s>>>(m, n, k2.p, mem_ptr.p); ++g_kl;
    LAP_CHECK_LAUNCH();
    ids.release();
    k1.release();
    tmark("  galerkin members");
    TermSrc S;
    S.kind = SRC_GALERKIN;
    S.rp = L.row_ptr;
    S.col = L.col;
    S.w = L.w;
    S.vfine = members.p;
    S.vout = (const int32_t *)k2.p;  // aggregate of member slot v (sorted keys)
    S.ostart = mem_ptr.p;
    S.agg = L.agg;
    const int cb = bitlen_u64((uint64_t)(m > 0 ? m : 1));
    // the ordered path pays off when coarse rows are short (per-row sorts); dense
    // coarse levels (thousands of terms per row: cfg 3/4 below level 0) keep the
    // one device-wide radix sort
    if (gal_fast_enabled() && L.nnz < ((int64_t)1 << 28) && L.nnz <= GAL_ORDERED_MAX_AVG * m)
        galerkin_fast(h, L, N, members.p, k2.p, mem_ptr.p, s);
    else csr_from_source(S, n, m, cb, ilogb_pos(L.maxw) + 1, L.nnz, true, N, s);
    h->cur.edges += L.nnz;
}

// =========================================================================
// O-S9 hierarchy loop
// =========================================================================

__global__ void k_max_deg(int64_t n, const int64_t *__restrict__ rp, unsigned long long *out) {
    unsigned long long m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long dg = (unsigned long long)(rp[i + 1] - rp[i]);
        m = dg > m ? dg : m;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, m, o);
        m = t > m ? t : m;
    }
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}
static int64_t max_degree(int64_t n, const int64_t *rp, cudaStream_t s) {
    DBuf<unsigned long long> r(1, s);
    LAP_CUDA(cudaMemsetAsync(r.p, 0, 8, s));
    if (n > 0) {
        k_max_deg<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(n, rp, r.p); ++g_kl;
        LAP_CHECK_LAUNCH();
    }
    return (int64_t)d2h_scalar(r.p, s);
}
static void release_logical(lap_hierarchy *h, int l, cudaStream_t s);
// the level's solve storage (built after the level below it), then release
static void finish_level(lap_hierarchy *h, int l, cudaStream_t s) {
    build_storage(h, l, s);
    if (g_tr) g_tr->mark("storage", l);
    release_logical(h, l, s);
}
// release the logical CSR of a big level once its storage exists
// (params.keep_logical: 1 keep, 0 release, -1 release when nnz >= 2^28)
static void release_logical(lap_hierarchy *h, int l, cudaStream_t s) {
    Level &L = h->lev[l];
    const int kl = h->p.keep_logical;
    const bool rel = L.kind != KIND_COARSEST && (kl == 0 || (kl < 0 && L.nnz >= ((int64_t)1 << 28)));
    if (rel) {
        dfree(L.row_ptr, s);
        dfree(L.col, s);
        dfree(L.w, s);
        L.row_ptr = nullptr;
        L.col = nullptr;
        L.w = nullptr;
        L.logical_released = true;
    }
}

void build_hierarchy(lap_hierarchy *h, const lap_graph *g, cudaStream_t s) {
    SetupTrace tr(s);
    g_tr = tr.on ? &tr : nullptr;
    struct Reset {
        ~Reset() { g_tr = nullptr; }
    } reset_tr;
    const lap_params &p = h->p;
    int64_t n = g->n;
    h->n0 = n;
    // --- input on device
    DBuf<int64_t> rp_in;
    DBuf<int32_t> col_in;
    DBuf<double> w_in;
    const int64_t *rp;
    const int32_t *col;
    const double *w;
    int64_t nnz;
    if (g->on_device) {
        rp = g->row_ptr;
        col = g->col;
        w = g->w;
        nnz = d2h_scalar(g->row_ptr + n, s);
    } else {
        nnz = g->row_ptr[n];
        if (g->row_ptr[0] != 0 || nnz < 0 || nnz >= (int64_t)1 << 40)
            throw Error{LAP_EGRAPH, "row_ptr[0] != 0 or row_ptr[n] outside [0, 2^40)"};
        rp_in.alloc(n + 1, s);
        col_in.alloc(nnz, s);
        h2d(rp_in.p, g->row_ptr, n + 1, s);
        if (nnz) h2d(col_in.p, g->col, nnz, s);
        if (g->w) {
            w_in.alloc(nnz, s);
            if (nnz) h2d(w_in.p, g->w, nnz, s);
        }
        rp = rp_in.p;
        col = col_in.p;
        w = g->w ? w_in.p : nullptr;
    }
    if (nnz < 0) throw Error{LAP_EGRAPH, "row_ptr[n] < 0"};
    if (nnz >= (int64_t)1 << 40 || n >= ((int64_t)1 << 31) - 1) throw Error{LAP_EINVAL, "graph too large"};
    // --- O-S0 validate
    {
        InputChunks IC;
        IC.s = s;
        DBuf<int> flag(1, s);
        DBuf<unsigned long long> hsum(2, s);
        LAP_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
        if (n > 0) {
            int64_t first = d2h_scalar(rp, s);
            if (first != 0) throw Error{LAP_EGRAPH, "row_ptr[0] != 0"};
            DBuf<unsigned long long> mdeg(1, s);
            LAP_CUDA(cudaMemsetAsync(mdeg.p, 0, sizeof(unsigned long long), s));
            k_validate_rowptr<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(n, nnz, rp, flag.p, mdeg.p); ++g_kl;
            LAP_CHECK_LAUNCH();
            if (d2h_scalar(flag.p, s)) throw Error{LAP_EGRAPH, "row_ptr is not monotone within [0, nnz]"};
            const int64_t maxdeg0 = (int64_t)d2h_scalar(mdeg.p, s);
            LAP_CUDA(cudaMemsetAsync(hsum.p, 0, 2 * sizeof(unsigned long long), s));
            // rows longer than SETUP_LONG in warp chunks (row_ptr is valid now) when some
            // row is long enough to be the kernels' tail (cfg 3: validation 2.66 -> 0.97 ms,
            // connectivity 2.09 -> 0.86; on cfg 4, max degree ~2^14, the chunk list costs
            // more than it saves)
            if (maxdeg0 > 8 * SETUP_LONG)
                IC.nch = build_chunks(rp, 0, n, SETUP_LONG, &IC.crow, &IC.cidx, &IC.cslot, &IC.cpart, &IC.ccnt, s);
            unsigned long long *hs = symcheck_mode() == 0 ? hsum.p : nullptr;
            LAUNCH_G(group_size(n, nnz), k_validate, n, s, n, rp, col, w, flag.p, hs,
                     IC.nch > 0 ? SETUP_LONG : INT64_MAX);
            if (IC.nch > 0) {
                k_validate_chunks<<<grid_for(IC.nch * 32, 256, 148 * 16), 256, 0, s>>>(IC.nch, IC.crow, IC.cidx, n, rp,
                                                                                        col, w, flag.p, hs);
                ++g_kl;
            }
            LAP_CHECK_LAUNCH();
        }
        if (d2h_scalar(flag.p, s)) throw Error{LAP_EGRAPH, "graph is not a valid symmetric positive-weight adjacency"};
        tr.mark("validate", 0);
        if (symcheck_mode() == 0) {
            unsigned long long hh[2] = {0, 0};
            if (n > 0) {
                LAP_CUDA(cudaMemcpyAsync(hh, hsum.p, sizeof(hh), cudaMemcpyDeviceToHost, s));
                LAP_CUDA(cudaStreamSynchronize(s));
            }
            if (hh[0] | hh[1]) throw Error{LAP_EGRAPH, "graph is not symmetric (w_ij != w_ji)"};
        } else if (!is_symmetric(n, nnz, rp, col, w, s)) {
            throw Error{LAP_EGRAPH, "graph is not symmetric (w_ij != w_ji)"};
        }
        tr.mark("symmetry", 0);
        if (!is_connected(n, nnz, rp, col, s, IC)) throw Error{LAP_EDISCONNECTED, "graph is disconnected"};
        tr.mark("connectivity", 0);
    }
    // --- O-S1 level 0
    h->perm = (int64_t *)dalloc(sizeof(int64_t) * (size_t)n, s);
    if (p.random_order && n > 1) {
        DBuf<uint64_t> k1(n, s), k2(n, s);
        DBuf<int32_t> i1(n, s), i2(n, s);
        k_perm_keys<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, salt_of(p.seed, 1), k1.p, i1.p); ++g_kl;
        LAP_CHECK_LAUNCH();
        size_t bytes = 0;
        LAP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k1.p, k2.p, i1.p, i2.p, n, 0, 64, s));
        DBuf<char> tmp((int64_t)bytes, s);
        LAP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, k1.p, k2.p, i1.p, i2.p, n, 0, 64, s)); ++g_kl;
        k_perm_from_order<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, i2.p, h->perm); ++g_kl;
    } else {
        k_identity_i64<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, h->perm); ++g_kl;
    }
    LAP_CHECK_LAUNCH();
    h->lev.clear();
    h->lev.reserve(64);
    h->lev.emplace_back();
    {
        Level &L0 = h->lev[0];
        int cb = bitlen_u64((uint64_t)(n > 0 ? n : 1));
        DBuf<int32_t> inv(n, s);  // old row of new id r
        k_inverse_perm<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, h->perm, inv.p); ++g_kl;
        const char *fr = getenv("LAP_RELABEL_TERMS");  // tests: the term-build relabel of big graphs
        const char *fs = getenv("LAP_L0_SORTED");      // 1: level 0 with sorted columns (as round 1)
        if (!(fr && fr[0] == '1')) {
            // P L P^T directly: row r = old row inv[r], columns perm[c], no duplicates,
            // nothing to sum.  The rows keep the caller's column order mapped through
            // Pi: no setup kernel needs them sorted (every setup reduction is an
            // order-free CanonSum, an argmax under a total order or a per-entry map;
            // the ordered Galerkin sorts its coarse rows itself), so the ~4 ms of
            // per-row sorts are spent only when the level is exported
            // (lap_level_export sorts a copy).  LAP_L0_SORTED=1 sorts them here.
            const bool sort0 = fs && fs[0] == '1';
            L0.cols_sorted = sort0;
            DBuf<int32_t> p32(n, s);
            k_perm_to_i32<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, h->perm, p32.p); ++g_kl;
            L0.n = n;
            L0.nnz = nnz;
            L0.row_ptr = (int64_t *)dalloc(sizeof(int64_t) * (size_t)(n + 1), s);
            L0.col = (int32_t *)dalloc(sizeof(int32_t) * (size_t)(nnz + 1), s);
            L0.w = (double *)dalloc(sizeof(double) * (size_t)(nnz + 1), s);
            permute_csr(n, nnz, inv.p, p32.p, rp, col, w, L0.row_ptr, L0.col, L0.w, sort0, INT64_MAX, s);
            tmark("  relabel: permute + row sorts");
            L0.d = (double *)dalloc(sizeof(double) * (size_t)(n > 0 ? n : 1), s);
            row_sums(n, nnz, L0.row_ptr, L0.w, L0.d, &L0.maxw, s);
            tmark("  terms: row sums");
            tr.mark("random order", 0);
        } else {
        TermSrc S;
        S.kind = SRC_RELABEL;
        S.rp = rp;
        S.col = col;
        S.w = w;
        S.vfine = inv.p;
        S.perm = h->perm;
        csr_from_source(S, n, n, cb, 0, 0, false, L0, s);
        tr.mark("random order", 0);
        }
    }
    rp_in.release();
    col_in.release();
    w_in.release();

    // Each level: setup work on its logical CSR, the next level built, then the
    // level's solve storage (build_storage needs the finer level's storage
    // order only) and -- for big levels unless params.keep_logical = 1 -- the
    // logical CSR is released (the solve runs on the storage copy; the
    // coarsest level keeps it for L^+).
    int elim_run = 0;  // consecutive elimination levels built just above (O-R21)
    LanczosStream lzs;
    const char *lza = getenv("LAP_LANCZOS_ASYNC");  // 0: in line on the setup stream
    // (under a real NCCL setup communicator the split Lanczos issues collectives:
    // in line, so that every rank enqueues them in one order on one stream)
    const bool lz_async = !(lza && lza[0] == '0') && !setup_nccl();
    double lz_host_v = 0.0, *lz_host = &lz_host_v;
    for (int l = 0;; l++) {
        Level &L = h->lev[l];
        L.maxdeg = max_degree(L.n, L.row_ptr, s);
        if (L.n + L.nnz <= p.coarse_nnz || l == p.max_levels - 1 || l == 63) {     // O-R27
            L.kind = KIND_COARSEST;
            finish_level(h, l, s);
            break;
        }
        if (p.elim_enable && elim_run < p.elim_rounds) {                            // O-R21
            DBuf<uint8_t> F;
            int64_t nF = elim_select(h, L, F, s);
            tr.mark("elim select", l);
            if (20 * nF > L.n) {                                                    // O-R20
                h->lev.emplace_back();
                Level &L2 = h->lev[l];
                build_elim_level(h, L2, F, nF, h->lev[l + 1], s);
                tr.mark("schur", l);
                F.release();
                finish_level(h, l, s);
                elim_run++;
                continue;
            }
        }
        // aggregation level: its storage first (Lanczos and the test-vector sweeps run on it)
        L.kind = KIND_AGG;
        build_storage(h, l, s);
        tr.mark("storage", l);
        if (lz_async) {
            lzs.start(l, s);
            lanczos(h, L, l, lzs.ls, lzs.lam + l);
        } else {
            lanczos(h, L, l, s, lz_host);
            LAP_CUDA(cudaStreamSynchronize(s));
            L.lambda = *lz_host;
        }
        tr.mark("lanczos", l);
        int64_t m = L.n;
        {
            DBuf<int32_t> rowof(L.nnz, s);  // row of every stored entry (entry-parallel strength kernels)
            if (L.nnz > 0) LAUNCH_G(group_size(L.n, L.nnz, L.maxdeg <= SHORT_MAX), k_rowof, L.n, s, L.n, L.row_ptr, rowof.p);
            L.rowof = rowof.p;
            DBuf<double> S(L.nnz, s);
            for (int attempt = 0; attempt < 2 && m == L.n; attempt++) m = aggregate_attempt(h, L, l, attempt, S, s);
            tr.mark("strength+votes", l);
            if (m != L.n && p.keep_strength) L.S = S.take();
            L.rowof = nullptr;
        }
        if (m == L.n) {                                                             // stalled twice (O-R28)
            if (L.agg) dfree(L.agg, s);
            L.agg = nullptr;
            L.kind = KIND_COARSEST;
            h->status = LAP_ESTALL;
            if (L.n > 8192) throw Error{LAP_ESTALL, "aggregation stalled on a level with more than 8192 vertices"};
            break;
        }
        L.m = m;
        h->lev.emplace_back();
        Level &L2 = h->lev[l];
        galerkin(h, L2, h->lev[l + 1], s);
        tr.mark("galerkin", l);
        release_logical(h, l, s);
        elim_run = 0;
    }
    coarse_pinv(h->lev.back(), s);
    tr.mark("coarsest pinv", (int)h->lev.size() - 1);
    lzs.join(h, s);
    tr.mark("lanczos join", 0);
}

// ---- test hook (lap_random_stream): the method's counter-based streams, by the
// same device functions the setup kernels use
__global__ void k_probe_hash(int64_t n, uint64_t salt2, uint64_t *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = elim_hash(i, salt2);
}
__global__ void k_probe_mix(int64_t n, uint64_t *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = mix64((uint64_t)i);
}
__global__ void k_probe_lz(int64_t n, uint64_t base, double *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = lz_start_value(base, i);
}
void random_stream(int which, uint64_t seed, int level, int attempt, int64_t n, void *out, cudaStream_t s) {
    const int64_t cnt = which == 1 ? 4 * n : n;
    DBuf<uint64_t> buf(cnt, s);
    const unsigned g = grid_for(cnt, 256, 148 * 8);
    if (which == 0) k_probe_hash<<<g, 256, 0, s>>>(n, salt_of(seed, 2), buf.p);
    else if (which == 1) k_tv_init<<<g, 256, 0, s>>>(n, mix64(salt_of(seed, 3) ^ (uint64_t)(2 * level + attempt)), (double *)buf.p);
    else if (which == 2) k_probe_lz<<<g, 256, 0, s>>>(n, mix64(salt_of(seed, 4) ^ (uint64_t)(2 * level)), (double *)buf.p);
    else k_probe_mix<<<g, 256, 0, s>>>(n, buf.p);
    LAP_CHECK_LAUNCH();
    LAP_CUDA(cudaMemcpyAsync(out, buf.p, 8 * (size_t)cnt, cudaMemcpyDeviceToHost, s));
    LAP_CUDA(cudaStreamSynchronize(s));
}

// =========================================================================
// lap_import_hierarchy: a hierarchy given as files (SURVEY §8(b) interchange
// format, written by the oracle's export): the GPU solve runs on exactly the
// operators, maps and lambda-hat of another implementation.
// =========================================================================
static std::string read_text(const std::string &fn) {
    FILE *f = fopen(fn.c_str(), "rb");
    if (!f) throw Error{LAP_EINVAL, "import: cannot open " + fn};
    std::string t;
    char buf[4096];
    size_t k;
    while ((k = fread(buf, 1, sizeof(buf), f)) > 0) t.append(buf, k);
    fclose(f);
    return t;
}
// the number after "key": in a flat JSON object
static double json_num(const std::string &js, const char *key, bool required, double dflt = 0.0) {
    const std::string k = std::string("\"") + key + "\"";
    size_t p = js.find(k);
    if (p == std::string::npos) {
        if (required) throw Error{LAP_EINVAL, std::string("import: meta.json lacks ") + key};
        return dflt;
    }
    p = js.find(':', p + k.size());
    if (p == std::string::npos) throw Error{LAP_EINVAL, std::string("import: bad value of ") + key};
    const char *c = js.c_str() + p + 1;
    char *end = nullptr;
    const double v = strtod(c, &end);
    if (end == c) throw Error{LAP_EINVAL, std::string("import: bad value of ") + key};
    return v;
}
template <class T>
static std::vector<T> read_raw(const std::string &fn, int64_t count) {
    FILE *f = fopen(fn.c_str(), "rb");
    if (!f) throw Error{LAP_EINVAL, "import: cannot open " + fn};
    fseek(f, 0, SEEK_END);
    const long long sz = ftell(f);
    fseek(f, 0, SEEK_SET);
    if (sz != (long long)(count * (int64_t)sizeof(T))) {
        fclose(f);
        throw Error{LAP_EINVAL, "import: " + fn + " has " + std::to_string(sz) + " bytes, expected " +
                                    std::to_string(count * (int64_t)sizeof(T))};
    }
    std::vector<T> v((size_t)count);
    if (count > 0 && fread(v.data(), sizeof(T), (size_t)count, f) != (size_t)count) {
        fclose(f);
        throw Error{LAP_EINVAL, "import: short read of " + fn};
    }
    fclose(f);
    return v;
}
template <class T>
static T *to_dev(const std::vector<T> &v, cudaStream_t s) {
    T *p = (T *)dalloc(sizeof(T) * (v.size() ? v.size() : 1), s);
    if (!v.empty()) h2d(p, v.data(), (int64_t)v.size(), s);
    return p;
}
__global__ void k_fmap_split(int64_t n, const int32_t *fmap, int32_t *cid, int32_t *fid, uint8_t *F) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t f = fmap[i];
        F[i] = f < 0;
        if (f < 0) fid[-1 - f] = (int32_t)i;
        else cid[f] = (int32_t)i;
    }
}

void import_hierarchy(lap_hierarchy *h, const char *dir, cudaStream_t s) {
    const std::string D(dir);
    const std::string meta = read_text(D + "/meta.json");
    if (meta.find("lap-hierarchy-v1") == std::string::npos) throw Error{LAP_EINVAL, "import: not a lap-hierarchy-v1 directory"};
    const int nlev = (int)json_num(meta, "nlev", true);
    const int64_t n0 = (int64_t)json_num(meta, "n0", true);
    if (nlev < 1 || nlev > 64 || n0 < 1 || n0 >= ((int64_t)1 << 31)) throw Error{LAP_EINVAL, "import: bad nlev / n0"};
    h->n0 = n0;
    {
        std::vector<int64_t> perm = read_raw<int64_t>(D + "/perm.i64", n0);
        std::vector<char> seen((size_t)n0, 0);
        for (int64_t i = 0; i < n0; i++) {
            if (perm[i] < 0 || perm[i] >= n0 || seen[perm[i]]) throw Error{LAP_EINVAL, "import: perm is not a permutation"};
            seen[perm[i]] = 1;
        }
        h->perm = to_dev(perm, s);
    }
    h->lev.clear();
    h->lev.reserve(64);
    int64_t expect_n = n0;
    for (int l = 0; l < nlev; l++) {
        const std::string P = D + "/L" + std::to_string(l);
        const std::string lm = read_text(P + "/meta.json");
        h->lev.emplace_back();
        Level &L = h->lev.back();
        L.kind = (int)json_num(lm, "kind", true);
        L.n = (int64_t)json_num(lm, "n", true);
        L.nnz = (int64_t)json_num(lm, "nnz", true);
        if (L.kind < 0 || L.kind > 2 || L.n != expect_n || L.nnz < 0 || (L.kind == KIND_COARSEST) != (l == nlev - 1))
            throw Error{LAP_EINVAL, "import: level " + std::to_string(l) + " has an inconsistent kind or size"};
        std::vector<int64_t> rp = read_raw<int64_t>(P + "/row_ptr.i64", L.n + 1);
        if (rp[0] != 0 || rp[L.n] != L.nnz) throw Error{LAP_EINVAL, "import: bad row_ptr at level " + std::to_string(l)};
        for (int64_t i = 0; i < L.n; i++)
            if (rp[i + 1] < rp[i]) throw Error{LAP_EINVAL, "import: row_ptr not monotone"};
        std::vector<int32_t> col = read_raw<int32_t>(P + "/col.i32", L.nnz);
        for (int64_t k = 0; k < L.nnz; k++)
            if (col[k] < 0 || col[k] >= L.n) throw Error{LAP_EINVAL, "import: column out of range"};
        L.row_ptr = to_dev(rp, s);
        L.col = to_dev(col, s);
        L.w = to_dev(read_raw<double>(P + "/w.f64", L.nnz), s);
        L.d = to_dev(read_raw<double>(P + "/d.f64", L.n), s);
        L.maxw = max_abs(L.w, L.nnz, s);
        L.maxdeg = max_degree(L.n, L.row_ptr, s);
        if (L.kind == KIND_AGG) {
            L.lambda = json_num(lm, "lambda", true);
            L.m = (int64_t)json_num(lm, "m", true);
            std::vector<int32_t> agg = read_raw<int32_t>(P + "/agg.i32", L.n);
            for (int64_t i = 0; i < L.n; i++)
                if (agg[i] < 0 || agg[i] >= L.m) throw Error{LAP_EINVAL, "import: aggregate id out of range"};
            L.agg = to_dev(agg, s);
            expect_n = L.m;
        } else if (L.kind == KIND_ELIM) {
            std::vector<int32_t> fmap = read_raw<int32_t>(P + "/fmap.i32", L.n);
            int64_t nF = 0, nc = 0;
            for (int64_t i = 0; i < L.n; i++) {
                if (fmap[i] < 0) {
                    if (-1 - fmap[i] != nF) throw Error{LAP_EINVAL, "import: F slots not in ascending order"};
                    nF++;
                } else {
                    if (fmap[i] != nc) throw Error{LAP_EINVAL, "import: C numbering not order-preserving"};
                    nc++;
                }
            }
            L.nF = nF;
            L.fmap = to_dev(fmap, s);
            L.cid = (int32_t *)dalloc(sizeof(int32_t) * (size_t)(nc + 1), s);
            L.fid = (int32_t *)dalloc(sizeof(int32_t) * (size_t)(nF + 1), s);
            DBuf<uint8_t> F(L.n, s);
            k_fmap_split<<<grid_for(L.n, 256, 148 * 8), 256, 0, s>>>(L.n, L.fmap, L.cid, L.fid, F.p); ++g_kl;
            LAP_CHECK_LAUNCH();
            build_ct_lists(L, F.p, nc, s);
            expect_n = nc;
        } else {
            L.pinv = to_dev(read_raw<double>(P + "/coarse_pinv.f64", L.n * L.n), s);
        }
    }
    for (int l = 0; l < nlev; l++) build_storage(h, l, s);
    LAP_CUDA(cudaStreamSynchronize(s));
}

}  // namespace lap
