// ktail.cu -- the K-cycle below a small level as ONE cluster kernel (N2).
//
// The K-cycle (oracle orc_kcycle / orc_kcoarse) visits level l
// 2^(number of aggregation levels above it) times per outer iteration, and
// each visit of a small level is ~10 dependent steps over a few thousand
// rows.  Launched one kernel per step (solve.cu kcoarse / cycle_rec), every
// step costs ~5 us of launch + dependent-load latency for ~0.1 us of work
// (cfg 2: ~80% of the K-cycle's ~700 launches per outer iteration are on
// levels of <= 2486 rows).
//
// Below the first level t whose sub-hierarchy is small (n_l <= KT_MAX_N,
// nnz_l <= KT_MAX_NNZ for every l >= t, and everything fits the cluster's
// shared memory), the whole coarse problem kcoarse(t) is ONE launch of a
// cluster of KT_CTAS CTAs (512 threads each) that never touches global
// memory for a vector:
//   * the host walks the same recursion as solve.cu once per hierarchy and
//     records it as a program of ops (same Chebyshev coefficients, same FCG
//     recurrence and guards);
//   * every vector of every level in the tail lives in DISTRIBUTED SHARED
//     MEMORY: level l's rows are split into KT_CTAS equal blocks, CTA c owns
//     block c of every vector of level l (uniform offsets in every CTA);
//     an op computes the rows its CTA owns from local shared memory; an op
//     that gathers (SpMV, transfers, coarsest GEMV) first pulls the whole
//     input vector from the KT_CTAS owners into a local replica with 16-byte
//     DSMEM loads, then gathers at shared-memory latency (per-element DSMEM
//     gathers measured 2-4x slower: request-rate bound);
//   * each CTA also stages its rows of every aggregation level's CSR
//     (offsets, columns, weights) and of every diagonal at launch;
//   * ops are separated by one cluster barrier (~0.2 us); dot products are
//     per-CTA block sums in shared memory, summed in CTA order by every
//     consumer (deterministic, identical in every CTA);
//   * entry: lev[t].b (and the fused step-0 x, dv) load from global;
//     exit: lev[t].x stores to global, where the launched parent reads it.
// Measured per call on cfg 2 (kcoarse(7), 67 ops): launched kernels ~335 us;
// single-CTA program ~270 us (one SM's dependent L2 round trips); cluster
// with vectors in L2 ~270 us; DSMEM per-element gathers 225-490 us; this
// design 143 us (~2.8 us per SpMV op, ~1 us per vector op, 0.2-0.3 us of it
// the cluster barrier).  A grid-wide persistent kernel was measured slower
// than launches in a graph.
//
// Arithmetic per op is that of the launched kernels (CSR-order row sums, a
// warp per row with a shuffle tree for rows longer than SHORT_MAX, the same
// epilogue formulas, FCG guards p.q = 0 -> 0); only the dot summation order
// differs, within rounding of the oracle (tests/test_gpu_kcycle.py).
#include "lap_internal.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <vector>

namespace cg = cooperative_groups;

namespace lap {

constexpr int64_t KT_MAX_N = 4096;
constexpr int64_t KT_MAX_NNZ = 131072;
constexpr int KT_THREADS = 1024;     // maximum block size (launch bound)
constexpr int KT_THREADS_DEFAULT = 512;  // measured: 1024 -> 512 threads, cfg 2 tail call 160 -> 143 us
constexpr int KT_CTAS = 8;             // portable cluster size
constexpr int KT_MAXLV = 48;           // hierarchy levels addressable by a program
constexpr int KT_MAXSTAGE = 24;        // staged matrices per program
constexpr int KT_MAXLOAD = 64;         // vectors loaded from global at entry
constexpr int KT_SLOTS = 3 * KT_MAXLV; // dot slots: 3 per level
constexpr size_t KT_SMEM_MAX = 220 * 1024;

enum KOpCode : int32_t {
    KO_CHEB_FIRST = 0,  // x = dv = (b / d) * c1
    KO_SPMV = 1,        // y = epilogue(L x), epi in {CHEB, CHEB0, RESID, FCG}; L staged (ms)
    KO_RESTRICT = 2,    // bc[a] = sum_{members} r ; optional coarse step 0
    KO_PROLONG = 3,     // x[i] += xc[agg[i]]
    KO_ERESTRICT = 4,   // bc[k] = b[cid[k]] + sum ctc * b[ctf] ; optional coarse step 0
    KO_EPROLONG = 5,    // x[i] = xc[fmap[i]] (C) ; x[f] = (b_f + sum w xc[fmap[col]]) / d_f (F)
    KO_COARSE = 6,      // x = P b  (n x n row-major)
    KO_DOT = 7,         // slot s0 = x . y
    KO_FCG_DIR = 8,     // beta = pq != 0 ? -zq/pq : 0 ; p = z + beta p      (slots s0 = pq, s2 = zq)
    KO_FCG_UPDATE = 9,  // alpha = pq != 0 ? pr/pq : 0 ; x (=|+=) alpha p ; r = rin - alpha q  (s0, s1)
};
enum KEpi : int32_t { KE_CHEB = 0, KE_CHEB0 = 1, KE_RESID = 2, KE_FCG = 3 };

// Vector operands are byte offsets into every CTA's shared memory (uniform
// layout); `lo` = level of the rows an op produces, `li` = level of the
// vector it gathers from.
struct __align__(16) KOp {
    int32_t code = 0, epi = 0, first = 0, s0 = 0, s1 = 0, s2 = 0;
    int32_t lo = 0, li = 0, ms = 0, pre0 = 0;
    uint32_t v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int64_t *rp = nullptr;  // member pointer / ct_ptr / CSR row pointer (EPROLONG)
    const int32_t *i0 = nullptr;  // members / agg / cid / fmap
    const int32_t *i1 = nullptr;  // ct_f
    const int32_t *i3 = nullptr;  // CSR columns (EPROLONG)
    const double *w = nullptr;    // ct_coef / pinv / CSR weights (EPROLONG)
    double c1 = 0, c2 = 0;
};

// one staged matrix, one CTA: its rows [r0, r1), entries [e0, e1) of the storage CSR
struct KSlice {
    int64_t e0, e1;
    uint32_t off_rp, off_col, off_w, pad;
};
struct KTailArgs {
    const KOp *prog;
    int nops;
    uint32_t prog_bytes;
    int nstage, nload;
    uint32_t part_off;                 // KT_SLOTS dot partials
    uint32_t rep_off;                  // replica of one gathered vector (largest level)
    const KSlice *slices;              // [nstage][KT_CTAS]
    const int64_t *st_rp[KT_MAXSTAGE];
    const int32_t *st_col[KT_MAXSTAGE];
    const double *st_w[KT_MAXSTAGE];
    int32_t st_lev[KT_MAXSTAGE];
    int32_t st_nshort[KT_MAXSTAGE];
    int64_t lev_n[KT_MAXLV];           // rows of each level (0 = unused)
    const double *ld_src[KT_MAXLOAD];  // entry loads: global vector -> shared offset
    uint32_t ld_off[KT_MAXLOAD];
    int32_t ld_lev[KT_MAXLOAD];
    double *out;                       // exit store: lev[t].x
    uint32_t out_off;
    int32_t out_lev;
    unsigned long long *trace;         // LAP_KTAIL_TRACE: %globaltimer after staging and after every op
};

struct KTail {
    int level = -1;
    bool pre0 = false;
    KOp *dprog = nullptr;
    KSlice *dslices = nullptr;
    KTailArgs args{};
    size_t smem = 0;
    Stats counts;  // the launched path's equivalent work (edges, bytes) per call
};

// ------------------------------------------------------------------ device
// rows of level n per CTA block (even: blocks are whole 16-byte units)
__device__ __forceinline__ int64_t kt_chunk(int64_t n) { return ((n + KT_CTAS - 1) / KT_CTAS + 1) & ~(int64_t)1; }

__device__ __forceinline__ void kt_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ double kt_block_sum(double v, double *red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double r = 0.0;
    if (wid == 0) {
        r = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    }
    __syncthreads();
    return r;  // thread 0
}

// element `local` of the vector at shared offset `off` in CTA `owner` (DSMEM; the own CTA too)
__device__ __forceinline__ double kt_dsm(uint32_t base, uint32_t off, uint32_t owner, uint32_t local) {
    uint32_t a = base + off + 8u * local, ra;
    double v;
    // not volatile, no memory clobber: the loads of a row pipeline; they cannot move above the
    // preceding cluster barrier (their addresses come from loads issued after it)
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(owner));
    asm("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra));
    return v;
}

struct KCtx {
    unsigned char *smem;
    uint32_t base;  // shared-window address of smem
    int cta;
    const int64_t *lev_n;
    cg::cluster_group cl;
    __device__ __forceinline__ double *loc(uint32_t off) const { return (double *)(smem + off); }
    // the whole vector (offset off, level l) gathered from the KT_CTAS blocks into the local
    // replica at rep (16-byte DSMEM loads); gathers then read shared memory at local latency
    __device__ __forceinline__ const double *replicate(uint32_t off, int l, uint32_t rep) const {
        const uint32_t ch2 = (uint32_t)(kt_chunk(lev_n[l]) / 2);  // 16-byte units per block
        double2 *dst = (double2 *)(smem + rep);
        for (uint32_t u = threadIdx.x; u < KT_CTAS * ch2; u += blockDim.x) {
            const uint32_t c = u / ch2, k = u - c * ch2;
            uint32_t a = base + off + 16u * k, ra;
            double2 v;
            asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(c));
            asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(ra));
            dst[u] = v;
        }
        __syncthreads();
        return (const double *)(smem + rep);
    }
    // dot slot s: the CTA partials summed in CTA order
    __device__ __forceinline__ double slot(uint32_t part_off, int s) const {
        double v[KT_CTAS];
#pragma unroll
        for (int c = 0; c < KT_CTAS; c++) v[c] = kt_dsm(base, part_off, c, s);
        double t = 0.0;
#pragma unroll
        for (int c = 0; c < KT_CTAS; c++) t += v[c];
        return t;
    }
};

__device__ __forceinline__ void kt_put_b(const KCtx &X, const KOp &o, int64_t k, int64_t lk, double s) {
    X.loc(o.v[1])[lk] = s;
    if (o.pre0) {  // fused coarse step 0: v = (s / d) / theta ; x = dv = v
        double v = (s / X.loc(o.v[2])[lk]) * o.c1;
        X.loc(o.v[4])[lk] = v;
        X.loc(o.v[3])[lk] = v;
    }
}

__global__ void __launch_bounds__(KT_THREADS, 1) k_ktail(KTailArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double red[32];
    __shared__ KSlice sl[KT_MAXSTAGE];
    pdl_begin();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    KCtx X{smem, (uint32_t)__cvta_generic_to_shared(smem), 0, A.lev_n, cg::this_cluster()};
    X.cta = (int)X.cl.block_rank();
    const int cta = X.cta;
    // ---- stage the program, this CTA's matrix rows and the entry vectors
    const KOp *prog = (const KOp *)smem;
    for (uint32_t k = tid; k < A.prog_bytes / 16; k += blockDim.x) ((int4 *)smem)[k] = ((const int4 *)A.prog)[k];
    if (tid < A.nstage) sl[tid] = A.slices[tid * KT_CTAS + cta];
    __syncthreads();
    for (int m = 0; m < A.nstage; m++) {
        const KSlice s = sl[m];
        const int64_t n = A.lev_n[A.st_lev[m]], ch = kt_chunk(n), r0 = min(n, cta * ch), r1 = min(n, r0 + ch);
        int32_t *rp = (int32_t *)(smem + s.off_rp);
        for (int64_t r = r0 + tid; r <= r1; r += blockDim.x) rp[r - r0] = (int32_t)(A.st_rp[m][r] - s.e0);
        int32_t *col = (int32_t *)(smem + s.off_col);
        double *w = (double *)(smem + s.off_w);
        for (int64_t e = s.e0 + tid; e < s.e1; e += blockDim.x) {
            col[e - s.e0] = A.st_col[m][e];
            w[e - s.e0] = A.st_w[m][e];
        }
    }
    for (int k = 0; k < A.nload; k++) {
        const int64_t n = A.lev_n[A.ld_lev[k]], ch = kt_chunk(n), r0 = min(n, cta * ch), r1 = min(n, r0 + ch);
        double *dst = X.loc(A.ld_off[k]);
        for (int64_t i = r0 + tid; i < r1; i += blockDim.x) dst[i - r0] = A.ld_src[k][i];
    }
    kt_cluster_sync();
    auto stamp = [&](int k) {
        if (A.trace && cta == 0 && tid == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            A.trace[k] = t;
        }
    };
    stamp(0);
    for (int pc = 0; pc < A.nops; pc++) {
        const KOp &o = prog[pc];
        const int64_t n = A.lev_n[o.lo], ch = kt_chunk(n), r0 = min(n, cta * ch), r1 = min(n, r0 + ch);
        switch (o.code) {
            case KO_CHEB_FIRST: {  // v0 b, v1 d, v2 x, v3 dv
                const double *b = X.loc(o.v[0]), *d = X.loc(o.v[1]);
                double *x = X.loc(o.v[2]), *dv = X.loc(o.v[3]);
                for (int64_t i = tid; i < r1 - r0; i += blockDim.x) {
                    double v = (b[i] / d[i]) * o.c1;
                    dv[i] = v;
                    x[i] = v;
                }
                break;
            }
            case KO_SPMV: {  // v0 x (gathered), v1 y, v2 b, v3 dv, v4 d ; matrix ms
                const KSlice s = sl[o.ms];
                const int32_t *rp = (const int32_t *)(smem + s.off_rp);
                const int32_t *col = (const int32_t *)(smem + s.off_col);
                const double *w = (const double *)(smem + s.off_w);
                const double *xl = X.loc(o.v[0]), *d = X.loc(o.v[4]), *b = X.loc(o.v[2]);
                const double *xr = X.replicate(o.v[0], o.li, A.rep_off);
                double *y = X.loc(o.v[1]), *dv = X.loc(o.v[3]);
                const int64_t nshort = A.st_nshort[o.ms];
                double da = 0.0, db = 0.0;
                auto epi = [&](int64_t li, double ax) {
                    const double xi = xl[li], di = d[li];
                    const double lx = di * xi - ax;
                    if (o.epi == KE_CHEB) {
                        double v = o.c1 * dv[li] + o.c2 * ((b[li] - lx) / di);
                        dv[li] = v;
                        y[li] = xi + v;
                    } else if (o.epi == KE_CHEB0) {
                        double v = o.c2 * ((b[li] - lx) / di);
                        dv[li] = v;
                        y[li] = xi + v;
                    } else if (o.epi == KE_RESID) {
                        y[li] = b[li] - lx;
                    } else {  // KE_FCG: q = L p ; p.q ; p.r
                        y[li] = lx;
                        da += xi * lx;
                        db += xi * b[li];
                    }
                };
                const int64_t rs_end = min(r1, nshort);
                for (int64_t i = r0 + tid; i < rs_end; i += blockDim.x) {  // short rows: a thread per row
                    double ax = 0.0;
                    const int32_t q1 = rp[i - r0 + 1];
#pragma unroll 4
                    for (int32_t q = rp[i - r0]; q < q1; q++) ax += w[q] * xr[col[q]];
                    epi(i - r0, ax);
                }
                for (int64_t i = max(r0, nshort) + warp; i < r1; i += nw) {  // long rows: a warp per row
                    double ax = 0.0;
                    const int32_t q1 = rp[i - r0 + 1];
                    for (int32_t q = rp[i - r0] + lane; q < q1; q += 32) ax += w[q] * xr[col[q]];
                    for (int k = 16; k > 0; k >>= 1) ax += __shfl_xor_sync(0xffffffffu, ax, k);
                    if (lane == 0) epi(i - r0, ax);
                }
                if (o.epi == KE_FCG) {
                    double t0 = kt_block_sum(da, red);
                    double t1 = kt_block_sum(db, red);
                    if (tid == 0) {
                        X.loc(A.part_off)[o.s0] = t0;
                        X.loc(A.part_off)[o.s1] = t1;
                    }
                }
                break;
            }
            case KO_RESTRICT: {  // coarse rows: v0 r (fine, gathered) ; v1 bc ; pre0: v2 d_c, v3 x_c, v4 dv_c
                const double *xr = X.replicate(o.v[0], o.li, A.rep_off);
                for (int64_t a = r0 + tid; a < r1; a += blockDim.x) {
                    double acc = 0.0;
                    const int64_t q1 = __ldg(&o.rp[a + 1]);
                    for (int64_t q = __ldg(&o.rp[a]); q < q1; q++) acc += xr[__ldg(&o.i0[q])];
                    kt_put_b(X, o, a, a - r0, acc);
                }
                break;
            }
            case KO_PROLONG: {  // fine rows: v0 xc (gathered), v1 x ; i0 = agg
                const double *xr = X.replicate(o.v[0], o.li, A.rep_off);
                double *x = X.loc(o.v[1]);
                for (int64_t i = r0 + tid; i < r1; i += blockDim.x) x[i - r0] += xr[__ldg(&o.i0[i])];
                break;
            }
            case KO_ERESTRICT: {  // coarse rows: v0 b (fine, gathered) ; v1 bc ; i0 cid, rp ct_ptr, i1 ct_f, w ct_coef
                const double *xr = X.replicate(o.v[0], o.li, A.rep_off);
                for (int64_t k = r0 + tid; k < r1; k += blockDim.x) {
                    double s = xr[__ldg(&o.i0[k])];
                    const int64_t q1 = __ldg(&o.rp[k + 1]);
                    for (int64_t q = __ldg(&o.rp[k]); q < q1; q++) s += __ldg(&o.w[q]) * xr[__ldg(&o.i1[q])];
                    kt_put_b(X, o, k, k - r0, s);
                }
                break;
            }
            case KO_EPROLONG: {  // fine rows: v0 xc (gathered), v1 x, v2 b, v3 d ; i0 fmap, CSR (rp, i3, w)
                const double *b = X.loc(o.v[2]), *d = X.loc(o.v[3]);
                const double *xr = X.replicate(o.v[0], o.li, A.rep_off);
                double *x = X.loc(o.v[1]);
                for (int64_t i = r0 + tid; i < r1; i += blockDim.x) {
                    const int32_t c = __ldg(&o.i0[i]);
                    if (c >= 0) {
                        x[i - r0] = xr[c];
                    } else {
                        double s = b[i - r0];
                        const int64_t q1 = __ldg(&o.rp[i + 1]);
                        for (int64_t q = __ldg(&o.rp[i]); q < q1; q++)
                            s += __ldg(&o.w[q]) * xr[__ldg(&o.i0[__ldg(&o.i3[q])])];
                        x[i - r0] = s / d[i - r0];
                    }
                }
                break;
            }
            case KO_COARSE: {  // rows: v0 b (gathered), v1 x ; w = P ; a warp per row (k_coarse_gemv order)
                const double *xr = X.replicate(o.v[0], o.lo, A.rep_off);
                double *x = X.loc(o.v[1]);
                for (int64_t i = r0 + warp; i < r1; i += nw) {
                    double acc = 0.0;
                    for (int64_t j = lane; j < n; j += 32) acc += __ldg(&o.w[i * n + j]) * xr[j];
                    for (int k = 16; k > 0; k >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, k);
                    if (lane == 0) x[i - r0] = acc;
                }
                break;
            }
            case KO_DOT: {  // slot s0 = v0 . v1
                const double *a = X.loc(o.v[0]), *c = X.loc(o.v[1]);
                double acc = 0.0;
                for (int64_t i = tid; i < r1 - r0; i += blockDim.x) acc += a[i] * c[i];
                double t = kt_block_sum(acc, red);
                if (tid == 0) X.loc(A.part_off)[o.s0] = t;
                break;
            }
            case KO_FCG_DIR: {  // v0 p, v1 z ; slots s0 = p.q, s2 = z.q
                const double pq = X.slot(A.part_off, o.s0), zq = X.slot(A.part_off, o.s2);
                const double beta = pq != 0.0 ? -zq / pq : 0.0;
                double *p = X.loc(o.v[0]);
                const double *z = X.loc(o.v[1]);
                for (int64_t i = tid; i < r1 - r0; i += blockDim.x) p[i] = z[i] + beta * p[i];
                break;
            }
            case KO_FCG_UPDATE: {  // v0 p, v1 q, v2 rin, v3 x, v4 rout ; slots s0 = p.q, s1 = p.r
                const double pq = X.slot(A.part_off, o.s0), pr = X.slot(A.part_off, o.s1);
                const double alpha = pq != 0.0 ? pr / pq : 0.0;
                const double *p = X.loc(o.v[0]), *q = X.loc(o.v[1]), *rin = X.loc(o.v[2]);
                double *x = X.loc(o.v[3]), *rout = X.loc(o.v[4]);
                for (int64_t i = tid; i < r1 - r0; i += blockDim.x) {
                    x[i] = o.first ? alpha * p[i] : x[i] + alpha * p[i];
                    rout[i] = rin[i] - alpha * q[i];
                }
                break;
            }
        }
        kt_cluster_sync();
        stamp(pc + 1);
    }
    {  // exit: this CTA's rows of lev[t].x
        const int64_t n = A.lev_n[A.out_lev], ch = kt_chunk(n), r0 = min(n, cta * ch), r1 = min(n, r0 + ch);
        const double *src = X.loc(A.out_off);
        for (int64_t i = r0 + tid; i < r1; i += blockDim.x) A.out[i] = src[i - r0];
    }
}

// ------------------------------------------------------------------ host: record the recursion
namespace {
struct Emitter {
    lap_hierarchy *h;
    int t;
    std::vector<KOp> ops;
    std::vector<const double *> vptr;  // registered vectors (global identity) ...
    std::vector<int> vlev;             // ... their level ...
    std::vector<uint32_t> voff;        // ... and shared-memory offset (relative to the vector region)
    uint32_t vbytes = 0;
    std::vector<int> staged;           // level of each staged matrix
    std::vector<int> loads;            // vector index loaded from global at entry
    Stats cnt;

    static int64_t chunk(int64_t n) { return ((n + KT_CTAS - 1) / KT_CTAS + 1) & ~(int64_t)1; }
    static bool fuse_on() {
        const char *e = getenv("LAP_FUSE_TRANSFERS");
        return !(e && e[0] == '0');
    }
    // shared-memory slot of vector p (level l); `load` = its entry value comes from global
    uint32_t vec(const double *p, int l, bool load = false) {
        for (size_t k = 0; k < vptr.size(); k++)
            if (vptr[k] == p) return voff[k];
        vptr.push_back(p);
        vlev.push_back(l);
        voff.push_back(vbytes);
        vbytes += (uint32_t)(8 * chunk(h->lev[l].n));
        vbytes = (vbytes + 15) & ~15u;
        if (load) loads.push_back((int)vptr.size() - 1);
        return voff.back();
    }
    uint32_t diag(int l) { return vec(h->lev[l].sd, l, true); }
    int stage(int l) {
        for (size_t k = 0; k < staged.size(); k++)
            if (staged[k] == l) return (int)k;
        staged.push_back(l);
        return (int)staged.size() - 1;
    }
    void pre0_of(KOp &o, int c) {  // fused coarse step 0 for an aggregation child (solve.cu Pre0)
        Level &C = h->lev[c];
        if (C.kind == KIND_AGG && fuse_on()) {
            o.pre0 = 1;
            o.v[2] = diag(c);
            o.v[3] = vec(C.x2, c);
            o.v[4] = vec(C.dv, c);
            o.c1 = 1.0 / C.cheb_theta;
        }
    }
    void spmv(int l, int epi, const double *x, const double *y, const double *b, const double *dv, double c1,
              double c2, int s0 = 0, int s1 = 0) {
        const Level &L = h->lev[l];
        KOp o;
        o.code = KO_SPMV;
        o.epi = epi;
        o.lo = o.li = l;
        o.ms = stage(l);
        o.v[0] = vec(x, l);
        o.v[1] = vec(y, l);
        o.v[2] = b ? vec(b, l) : 0;
        o.v[3] = dv ? vec(dv, l) : 0;
        o.v[4] = diag(l);
        o.c1 = c1;
        o.c2 = c2;
        o.s0 = s0;
        o.s1 = s1;
        ops.push_back(o);
        cnt.edges += L.nnz;
        cnt.bytes += 12 * L.nnz + 40 * L.n;
    }
    // solve.cu cycle_rec with kc = true; b and xout are level-l vectors
    void kcycle(int l, const double *b, const double *xout, bool pre0_done) {
        Level &L = h->lev[l];
        const int64_t n = L.n;
        if (L.kind == KIND_COARSEST) {
            KOp o;
            o.code = KO_COARSE;
            o.lo = o.li = l;
            o.w = L.pinv_s;
            o.v[0] = vec(b, l);
            o.v[1] = vec(xout, l);
            ops.push_back(o);
            cnt.bytes += 8 * n * n;
            return;
        }
        Level &C = h->lev[l + 1];
        if (L.kind == KIND_ELIM) {
            KOp o;
            o.code = KO_ERESTRICT;
            o.lo = l + 1;
            o.li = l;
            o.i0 = L.cid_s;
            o.rp = L.ct_ptr_s;
            o.i1 = L.ct_f_s;
            o.w = L.ct_coef_s;
            o.v[0] = vec(b, l);
            o.v[1] = vec(C.b, l + 1);
            pre0_of(o, l + 1);
            ops.push_back(o);
            kcoarse(l + 1, o.pre0 != 0);
            KOp p;
            p.code = KO_EPROLONG;
            p.lo = l;
            p.li = l + 1;
            p.i0 = L.fmap_s;
            p.rp = L.srp;
            p.i3 = L.scol;
            p.w = L.sw;
            p.v[0] = vec(C.x, l + 1);
            p.v[1] = vec(xout, l);
            p.v[2] = vec(b, l);
            p.v[3] = diag(l);
            ops.push_back(p);
            cnt.bytes += 16 * n;
            return;
        }
        const int K = h->p.cheby_degree;
        const double theta = L.cheb_theta, delta = L.cheb_delta, sigma = L.cheb_sigma;
        const double *cur = L.x2, *alt = L.t;
        if (!pre0_done) {
            KOp o;
            o.code = KO_CHEB_FIRST;
            o.lo = o.li = l;
            o.c1 = 1.0 / theta;
            o.v[0] = vec(b, l);
            o.v[1] = diag(l);
            o.v[2] = vec(cur, l);
            o.v[3] = vec(L.dv, l);
            ops.push_back(o);
        }
        cnt.bytes += 32 * n;
        double rho_old = 1.0 / sigma;
        for (int k = 1; k < K; k++) {
            double rho = 1.0 / (2.0 * sigma - rho_old);
            spmv(l, KE_CHEB, cur, alt, b, L.dv, rho * rho_old, 2.0 * rho / delta);
            std::swap(cur, alt);
            rho_old = rho;
        }
        spmv(l, KE_RESID, cur, L.r, b, nullptr, 0, 0);
        KOp r;
        r.code = KO_RESTRICT;
        r.lo = l + 1;
        r.li = l;
        r.rp = L.mem_ptr;
        r.i0 = L.members;
        r.v[0] = vec(L.r, l);
        r.v[1] = vec(C.b, l + 1);
        pre0_of(r, l + 1);
        ops.push_back(r);
        kcoarse(l + 1, r.pre0 != 0);
        KOp p;
        p.code = KO_PROLONG;
        p.lo = l;
        p.li = l + 1;
        p.i0 = L.agg_s;
        p.v[0] = vec(C.x, l + 1);
        p.v[1] = vec(cur, l);
        ops.push_back(p);
        cnt.bytes += 36 * n + 16 * L.m;
        rho_old = 1.0 / sigma;
        for (int k = 0; k < K; k++) {
            const double *dst = (k == K - 1) ? xout : alt;
            if (k == 0) {
                spmv(l, KE_CHEB0, cur, dst, b, L.dv, 0.0, 1.0 / theta);
            } else {
                double rho = 1.0 / (2.0 * sigma - rho_old);
                spmv(l, KE_CHEB, cur, dst, b, L.dv, rho * rho_old, 2.0 * rho / delta);
                rho_old = rho;
            }
            if (k < K - 1) std::swap(cur, alt);
        }
    }
    // solve.cu kcoarse
    void kcoarse(int l, bool pre0_done) {
        Level &L = h->lev[l];
        if (L.kind != KIND_AGG) {
            kcycle(l, L.b, L.x, pre0_done);
            return;
        }
        const int sq = 3 * l, sr = sq + 1, sz = sq + 2;
        for (int k = 1; k <= h->p.kcycle_inner; k++) {
            const double *rin = k == 1 ? L.b : L.kr;
            if (k == 1) {
                kcycle(l, L.b, L.kp, pre0_done);
            } else {
                kcycle(l, L.kr, L.kz, false);
                KOp d;
                d.code = KO_DOT;
                d.lo = d.li = l;
                d.v[0] = vec(L.kz, l);
                d.v[1] = vec(L.kq, l);
                d.s0 = sz;
                ops.push_back(d);
                KOp o;
                o.code = KO_FCG_DIR;
                o.lo = o.li = l;
                o.v[0] = vec(L.kp, l);
                o.v[1] = vec(L.kz, l);
                o.s0 = sq;
                o.s2 = sz;
                ops.push_back(o);
            }
            spmv(l, KE_FCG, L.kp, L.kq, rin, nullptr, 0, 0, sq, sr);
            KOp u;
            u.code = KO_FCG_UPDATE;
            u.lo = u.li = l;
            u.v[0] = vec(L.kp, l);
            u.v[1] = vec(L.kq, l);
            u.v[2] = vec(rin, l);
            u.v[3] = vec(L.x, l);
            u.v[4] = vec(L.kr, l);
            u.first = k == 1 ? 1 : 0;
            u.s0 = sq;
            u.s1 = sr;
            ops.push_back(u);
            cnt.bytes += 48 * L.n;
        }
    }
};
}  // namespace

static bool small_level(const Level &L) { return L.n <= KT_MAX_N && L.nnz <= KT_MAX_NNZ; }

static bool ktail_enabled() {  // LAP_KTAIL=0: launched kernels on every level
    const char *e = getenv("LAP_KTAIL");
    return !(e && e[0] == '0');
}

static void build_at(lap_hierarchy *h, int t, cudaStream_t s) {
    const int nl = (int)h->lev.size();
    if (nl > KT_MAXLV) return;
    Emitter em;
    em.h = h;
    em.t = t;
    Level &T = h->lev[t];
    const bool pre0 = T.kind == KIND_AGG && Emitter::fuse_on();  // what the caller of kcoarse(t) passes
    // entry vectors: b (and the fused step 0) come from the launched parent
    em.vec(T.b, t, true);
    if (pre0) {
        em.vec(T.x2, t, true);
        em.vec(T.dv, t, true);
    }
    em.kcoarse(t, pre0);
    const uint32_t out_rel = em.vec(T.x, t);
    const int nstage = (int)em.staged.size(), nload = (int)em.loads.size();
    if (nstage > KT_MAXSTAGE || nload > KT_MAXLOAD) return;
    // shared-memory layout (uniform part): program | vectors | dot partials ; then per-CTA matrix rows
    const size_t prog_bytes = sizeof(KOp) * em.ops.size();
    const uint32_t vec_base = (uint32_t)((prog_bytes + 15) & ~(size_t)15);
    const uint32_t part_off = (uint32_t)((vec_base + em.vbytes + 15) & ~15u);
    const uint32_t rep_off = (uint32_t)((part_off + 8 * KT_SLOTS + 15) & ~15u);
    const size_t uniform = rep_off + 8 * (size_t)KT_CTAS * Emitter::chunk(T.n);  // level t is the largest
    for (auto &o : em.ops)
        for (auto &v : o.v) v += vec_base;  // (unused operands point at the region start: never read)
    std::vector<KSlice> slices((size_t)nstage * KT_CTAS);
    size_t worst = uniform;
    std::vector<std::vector<int64_t>> rps(nstage);
    for (int m = 0; m < nstage; m++) {
        const Level &L = h->lev[em.staged[m]];
        rps[m].resize((size_t)L.n + 1);
        LAP_CUDA(cudaMemcpyAsync(rps[m].data(), L.srp, 8 * rps[m].size(), cudaMemcpyDeviceToHost, s));
    }
    LAP_CUDA(cudaStreamSynchronize(s));
    for (int c = 0; c < KT_CTAS; c++) {
        size_t off = uniform;
        for (int m = 0; m < nstage; m++) {
            const int64_t n = h->lev[em.staged[m]].n, ch = Emitter::chunk(n);
            const int64_t r0 = std::min<int64_t>(n, c * ch), r1 = std::min<int64_t>(n, r0 + ch);
            KSlice &q = slices[(size_t)m * KT_CTAS + c];
            q.e0 = rps[m][r0];
            q.e1 = rps[m][r1];
            off = (off + 15) & ~(size_t)15;
            q.off_rp = (uint32_t)off;
            off += 4 * (size_t)(r1 - r0 + 1);
            off = (off + 15) & ~(size_t)15;
            q.off_col = (uint32_t)off;
            off += 4 * (size_t)(q.e1 - q.e0);
            off = (off + 15) & ~(size_t)15;
            q.off_w = (uint32_t)off;
            off += 8 * (size_t)(q.e1 - q.e0);
            q.pad = 0;
        }
        worst = std::max(worst, off);
    }
    if (worst > KT_SMEM_MAX) return;  // does not fit: the caller tries a smaller tail
    KTail *kt = new KTail();
    kt->level = t;
    kt->pre0 = pre0;
    kt->counts = em.cnt;
    kt->smem = worst;
    kt->dprog = (KOp *)dalloc(prog_bytes, s);
    kt->dslices = (KSlice *)dalloc(sizeof(KSlice) * slices.size(), s);

    // pageable sources: the calls return once the data has been staged
    LAP_CUDA(cudaMemcpyAsync(kt->dprog, em.ops.data(), prog_bytes, cudaMemcpyHostToDevice, s));
    LAP_CUDA(cudaMemcpyAsync(kt->dslices, slices.data(), sizeof(KSlice) * slices.size(), cudaMemcpyHostToDevice, s));
    KTailArgs &a = kt->args;
    a.prog = kt->dprog;
    a.nops = (int)em.ops.size();
    a.prog_bytes = (uint32_t)prog_bytes;
    a.nstage = nstage;
    a.nload = nload;
    a.part_off = part_off;
    a.rep_off = rep_off;
    a.slices = kt->dslices;
    for (int m = 0; m < nstage; m++) {
        const Level &L = h->lev[em.staged[m]];
        a.st_rp[m] = L.srp;
        a.st_col[m] = L.scol;
        a.st_w[m] = L.sw;
        a.st_lev[m] = em.staged[m];
        a.st_nshort[m] = (int32_t)L.c_end[0];
    }
    for (int l = 0; l < nl; l++) a.lev_n[l] = l >= t ? h->lev[l].n : 0;
    for (int k = 0; k < nload; k++) {
        const int v = em.loads[k];
        a.ld_src[k] = em.vptr[v];
        a.ld_off[k] = vec_base + em.voff[v];
        a.ld_lev[k] = em.vlev[v];
    }
    a.out = T.x;
    a.out_off = vec_base + out_rel;
    a.out_lev = t;
    h->ktail = kt;
    if (getenv("LAP_KTAIL_INFO"))
        fprintf(stderr, "ktail: level %d (n %lld), %d ops, %d matrices, %zu B vectors, %zu B shared memory per CTA\n",
                t, (long long)T.n, a.nops, nstage, (size_t)em.vbytes, worst);
}

void build_ktail(lap_hierarchy *h, cudaStream_t s) {
    free_ktail(h, s);
    const int nl = (int)h->lev.size();
    if (h->p.cycle != 1 || !ktail_enabled() || nl < 2) return;
    int t = nl;
    while (t > 1 && small_level(h->lev[t - 1])) t--;
    // the largest tail whose program, vectors and matrix rows fit the cluster's shared memory
    for (; t < nl && h->lev[t].kind != KIND_COARSEST && !h->ktail; t++) build_at(h, t, s);
}

void free_ktail(lap_hierarchy *h, cudaStream_t s) {
    KTail *kt = (KTail *)h->ktail;
    if (!kt) return;
    dfree(kt->dprog, s);
    dfree(kt->dslices, s);
    delete kt;
    h->ktail = nullptr;
}

// kcoarse(l) as one launch when l is the program's level (and the caller's fusion matches)
bool ktail_launch(lap_hierarchy *h, int l, bool pre0_done, cudaStream_t s) {
    KTail *kt = (KTail *)h->ktail;
    if (!kt || kt->level != l || kt->pre0 != pre0_done) return false;
    static bool attr = false;
    if (!attr) {
        LAP_CUDA(cudaFuncSetAttribute(k_ktail, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)KT_SMEM_MAX));
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(KT_CTAS);
    static const int nthr = [] {  // LAP_KTAIL_THREADS: block size (multiple of 32, <= KT_THREADS)
        const char *e = getenv("LAP_KTAIL_THREADS");
        int v = e ? atoi(e) : KT_THREADS_DEFAULT;
        return (v >= 64 && v <= KT_THREADS && v % 32 == 0) ? v : KT_THREADS_DEFAULT;
    }();
    cfg.blockDim = dim3(nthr);
    cfg.dynamicSmemBytes = kt->smem;
    cfg.stream = s;
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = KT_CTAS;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    static const bool trace = getenv("LAP_KTAIL_TRACE") != nullptr;
    KTailArgs args = kt->args;
    std::vector<unsigned long long> tr;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (trace) LAP_CUDA(cudaStreamIsCapturing(s, &cap));
    if (trace && cap == cudaStreamCaptureStatusNone) {
        tr.resize((size_t)args.nops + 1);
        args.trace = (unsigned long long *)dalloc(8 * tr.size(), s);
    }
    LAP_CUDA(cudaLaunchKernelEx(&cfg, k_ktail, args));
    if (args.trace) {  // per-op device time (ns), grouped by op code
        LAP_CUDA(cudaMemcpyAsync(tr.data(), args.trace, 8 * tr.size(), cudaMemcpyDeviceToHost, s));
        LAP_CUDA(cudaStreamSynchronize(s));
        dfree(args.trace, s);
        std::vector<KOp> ops((size_t)args.nops);
        LAP_CUDA(cudaMemcpy(ops.data(), args.prog, sizeof(KOp) * ops.size(), cudaMemcpyDeviceToHost));
        double per[16] = {0};
        int cntc[16] = {0};
        for (int k = 0; k < args.nops; k++) {
            per[ops[k].code] += (double)(tr[k + 1] - tr[k]);
            cntc[ops[k].code]++;
        }
        fprintf(stderr, "ktail trace: total %.1f us over %d ops;", (tr[args.nops] - tr[0]) * 1e-3, args.nops);
        for (int c = 0; c < 10; c++)
            if (cntc[c]) fprintf(stderr, " op%d x%d %.2f us", c, cntc[c], per[c] * 1e-3 / cntc[c]);
        fprintf(stderr, "\n");
    }
    h->cur.launches++;
    h->cur.edges += kt->counts.edges;
    h->cur.bytes += kt->counts.bytes;
    LAP_CHECK_LAUNCH();
    return true;
}

}  // namespace lap
