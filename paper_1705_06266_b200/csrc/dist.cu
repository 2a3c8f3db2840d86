// dist.cu -- multi-GPU solve: the fine levels of the
// hierarchy are sharded as a 2D edge partition over a pr x pc process grid
// (the paper's CombBLAS layout, with the vectors spread over all
// ranks, P:341-342 / O-R35); coarse levels are replicated on every rank
// (O-R36).  One process per GPU; NCCL over NVLink carries
//   * the column allgather of x and the row reduce-scatter of A x per SpMV,
//   * the world reduce-scatter / allreduce of a restriction and the world
//     allgather of a prolongation source,
//   * the allreduce of every PCG dot product.
// The hierarchy itself comes from the single-GPU setup run identically on every
// rank (it is deterministic, O-R23), so every rank holds the same discrete
// data and only the solve is distributed.
//
// The same code also runs a whole pr x pc grid inside ONE process on one
// GPU ("virtual" communicator): every rank's shard lives on the device and
// the collectives are device copies and fixed-order sums.  That is how the
// 2D data path is validated on a single B200 (no kernel ever waits on another
// rank's kernel); the NCCL communicator swaps the transport only.
//
// Index spaces of a distributed level with n rows (storage order, storage.cu):
//   piece map  : storage row p -> dist index k*S + q, block-cyclic in blocks of
//                DIST_B rows over the P pieces (every piece gets every class of
//                rows: hubs are not all in the last piece); S = padded piece
//                size (NCCL collectives need equal counts), pads sit at the end
//                of a piece and stay exactly 0.
//   rank r = (gi, gj) = (r / pc, r % pc) owns piece r;
//   row block gi    = pieces [gi*pc, gi*pc + pc)  (contiguous, pc*S rows)
//   column block gj = pieces {gj, pc + gj, ...}   (pr*S columns, concatenated
//                     in grid-row order = the column-communicator rank order)
#include <nccl.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "lap_internal.cuh"

struct lap_comm {
    int pr = 1, pc = 1, P = 1;
    int virt = 1;   // 1: all P ranks emulated in this process on the current device
    int rank = 0;   // NCCL mode: this process's rank
    ncclComm_t world = nullptr, row = nullptr, col = nullptr;
};

namespace lap {

#define NCCL_CHECK(call)                                                                         \
    do {                                                                                         \
        ncclResult_t _r = (call);                                                                \
        if (_r != ncclSuccess)                                                                   \
            throw ::lap::Error{LAP_ENCCL, std::string(#call ": ") + ncclGetErrorString(_r)};     \
    } while (0)

constexpr int64_t DIST_B = 256;

struct PieceMap {
    int64_t n = 0, S = DIST_B;
    int P = 1;
    __host__ __device__ __forceinline__ int64_t dist_of(int64_t p) const {
        int64_t blk = p / DIST_B, k = blk % P, q = (blk / P) * DIST_B + p % DIST_B;
        return k * S + q;
    }
    __host__ __device__ __forceinline__ int64_t storage_of(int64_t d) const {  // -1: padding
        int64_t k = d / S, q = d % S;
        int64_t p = ((q / DIST_B) * P + k) * DIST_B + q % DIST_B;
        return p < n ? p : -1;
    }
};
static PieceMap make_map(int64_t n, int P) {
    PieceMap m;
    m.n = n;
    m.P = P;
    int64_t nb = (n + DIST_B - 1) / DIST_B;
    m.S = std::max<int64_t>(1, (nb + P - 1) / P) * DIST_B;
    return m;
}
// number of real (non-pad) slots of piece k: pads are at the end of a piece
static int64_t real_rows(const PieceMap &m, int k) {
    int64_t lo = 0, hi = m.S;  // first slot whose storage row is >= n
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (m.storage_of((int64_t)k * m.S + mid) >= 0) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

struct BlockMat {  // one part of a rank's 2D block: SELL-32 over short rows + LCHUNK chunks over long rows
    int64_t nnz = 0;
    int64_t *rp = nullptr;
    int32_t *col = nullptr;
    double *w = nullptr;
    int64_t nslices = 0;
    int64_t *slice_ptr = nullptr;
    int32_t *ell_col = nullptr;
    double *ell_w = nullptr;
    int64_t nchunks = 0;
    int32_t *crow = nullptr, *cidx = nullptr, *cslot = nullptr, *ccnt = nullptr;
    double *cpart = nullptr;
};
struct Shard {
    int r = 0, gi = 0, gj = 0;
    int64_t nreal = 0;
    // 2D block: rows = row block (nrow = pc*S), columns = column block (ncol = pr*S)
    int64_t nrow = 0, ncol = 0;
    // A_ij split by column: `own` = the columns of this rank's own x piece
    // (local ids into the piece, needs no communication), `rem` = the other
    // pieces of column block gj (ids into xcol, after the column allgather)
    BlockMat own, rem;
    // vectors: column block, row-block partial (own part, then own + remote), owned piece
    double *xcol = nullptr, *ypart = nullptr, *yown = nullptr, *ax = nullptr;
    double *d = nullptr, *b = nullptr, *x = nullptr, *x2 = nullptr, *t = nullptr, *rv = nullptr, *dv = nullptr;
    // aggregation transfer (coarse index space of the next level)
    int64_t *mem_ptr = nullptr;
    int32_t *members = nullptr, *cmap = nullptr;
    // elimination transfer
    int64_t *er_ptr = nullptr;
    int32_t *er_slot = nullptr;
    double *er_coef = nullptr;
    int32_t *ep_c = nullptr;  // owned slot -> coarse index (C rows), -1 (F rows)
    int64_t *ep_ptr = nullptr;
    int32_t *ep_col = nullptr;
    double *ep_w = nullptr;
    double *cfull = nullptr;     // coarse-space partial (restriction)
    double *xcfull = nullptr;    // coarse-space x (prolongation source, when the next level is distributed)
    // PCG (level 0)
    double *px = nullptr, *pr = nullptr, *pz = nullptr, *pp = nullptr, *pq = nullptr, *pb_in = nullptr;
    double *partials = nullptr;  // RED_BLOCKS
    double *scal = nullptr;      // 16 device scalars (local partial results)
};

struct DistLevel {
    bool dist = false;
    PieceMap map;
    int64_t mc = 0;        // length of the coarse index space of the transfer to l+1
    bool next_dist = false;
    std::vector<Shard> sh;  // one per local rank
};

struct Dist {
    lap_comm *c = nullptr;
    int D = 0;              // levels [0, D) distributed, [D, nlev) replicated
    std::vector<DistLevel> lev;
    double *gscal = nullptr;  // world-reduced scalars (16)
    double *xfull = nullptr;  // level-0 allgather target (P*S0)
    // the PCG's per-iteration preconditioner step (V-cycle + projection + z
    // dots, collectives included) as one CUDA graph, captured at the first solve
    cudaGraphExec_t pgraph = nullptr;
    int64_t pg_launches = 0, pg_edges = 0, pg_bytes = 0;
    bool use_graph = true;  // the caller's params.use_graphs
    // NCCL grids: the own-piece block SpMV runs on a side stream while the
    // column allgather is in flight (fork / join by events; captured into the graph too)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};
extern bool g_capturing_flag(bool v);
static bool dist_graph_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("LAP_DIST_GRAPH");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

static std::vector<void *> *g_owned = nullptr;
template <class T>
static T *dal(int64_t count, cudaStream_t s) {
    T *p = (T *)dalloc(sizeof(T) * (size_t)(count > 0 ? count : 1), s);
    g_owned->push_back(p);
    return p;
}

// ------------------------------------------------------------------ block extraction
// column part of an entry: 0 = not in column block gj; 1 = in this rank's own
// piece (gi of the column block); 2 = another piece of the column block
__device__ __forceinline__ int blk_part(const PieceMap &m, int pc, int gi, int gj, int32_t c) {
    const int64_t d = m.dist_of(c), piece = d / m.S;
    if (piece % pc != gj) return 0;
    return piece / pc == gi ? 1 : 2;
}
// local column id: into the column block (part 2) or into the own piece (part 1)
__device__ __forceinline__ int32_t blk_lcol(const PieceMap &m, int pc, int part, int32_t c) {
    const int64_t d = m.dist_of(c);
    return part == 1 ? (int32_t)(d % m.S) : (int32_t)((d / m.S / pc) * m.S + d % m.S);
}
template <int G>
__global__ void k_blk_count(int64_t nrow, int64_t row_d0, PieceMap m, int pc, int gi, int gj, int part,
                            const int64_t *__restrict__ srp, const int32_t *__restrict__ scol,
                            int64_t *__restrict__ cnt) {
    GROUP_LOOP_BEGIN(G, nrow)
        int64_t c = 0;
        const int64_t p = live ? m.storage_of(row_d0 + i) : -1;
        if (p >= 0)
            for (int64_t k = srp[p] + gl; k < srp[p + 1]; k += G) c += blk_part(m, pc, gi, gj, scol[k]) == part;
        c = grp_sum<G>(c);
        if (live && gl == 0) cnt[i] = c;
    GROUP_LOOP_END
}
template <int G>
__global__ void k_blk_fill(int64_t nrow, int64_t row_d0, PieceMap m, int pc, int gi, int gj, int part,
                           const int64_t *__restrict__ srp, const int32_t *__restrict__ scol,
                           const double *__restrict__ sw, const int64_t *__restrict__ rp, int32_t *__restrict__ col,
                           double *__restrict__ w) {
    GROUP_LOOP_BEGIN(G, nrow)
        const int64_t srow = live ? m.storage_of(row_d0 + i) : -1;
        const int64_t kb = srow >= 0 ? srp[srow] : 0, ke = srow >= 0 ? srp[srow + 1] : 0;
        int64_t o = live ? rp[i] : 0;
        GROUP_COMPACT_ROW(G, kb, ke, o, blk_part(m, pc, gi, gj, scol[k]) == part,
                          (col[p] = blk_lcol(m, pc, part, scol[k]), w[p] = sw[k]))
    GROUP_LOOP_END
}
// SELL-32 over all block rows; rows longer than SHORT_MAX have width 0 here
// (their chunks carry them)
__global__ void k_blk_width(int64_t nslices, int64_t nrow, const int64_t *rp, int64_t *width) {
    for (int64_t sl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sl < nslices; sl += (int64_t)gridDim.x * blockDim.x) {
        int64_t mx = 0;
        for (int64_t t = sl * 32; t < min(nrow, sl * 32 + 32); t++) {
            int64_t dg = rp[t + 1] - rp[t];
            if (dg <= SHORT_MAX) mx = max(mx, dg);
        }
        width[sl] = 32 * mx;
    }
}
__global__ void k_blk_sell_fill(int64_t nslots, int64_t nrow, const int64_t *rp, const int32_t *col, const double *w,
                                const int64_t *slice_ptr, int32_t *ell_col, double *ell_w) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nslots; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t sl = t >> 5, lane = t & 31;
        int64_t base = slice_ptr[sl] + lane, width = (slice_ptr[sl + 1] - slice_ptr[sl]) >> 5;
        int64_t a = t < nrow ? rp[t] : 0, dg = t < nrow ? rp[t + 1] - a : 0;
        if (dg > SHORT_MAX) dg = 0;
        for (int64_t k = 0; k < width; k++) {
            ell_col[base + 32 * k] = k < dg ? col[a + k] : 0;
            ell_w[base + 32 * k] = k < dg ? w[a + k] : 0.0;
        }
    }
}

// ------------------------------------------------------------------ block SpMV: ypart = A_ij xcol
__global__ void __launch_bounds__(256) k_blk_spmv(int64_t nslices, int64_t nrow, const int64_t *__restrict__ sp,
                                                  const int32_t *__restrict__ ec, const double *__restrict__ ew,
                                                  const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                                                  const double *__restrict__ w, int64_t nchunks,
                                                  const int32_t *__restrict__ crow, const int32_t *__restrict__ cidx,
                                                  const int32_t *__restrict__ cslot, double *__restrict__ cpart,
                                                  int32_t *__restrict__ ccnt, const double *__restrict__ x,
                                                  double *__restrict__ y, const double *__restrict__ yadd) {
    // y = yadd + A x (yadd: the own-piece part, NULL for 0) -- every row written once
    pdl_begin();
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = warp; t < nslices + nchunks; t += nwarps) {
        if (t < nslices) {
            const int64_t i = t * 32 + lane, beg = sp[t], end = sp[t + 1];
            double acc = 0.0;
            for (int64_t k = beg + lane; k < end; k += 32) acc += __ldg(&ew[k]) * x[__ldg(&ec[k])];
            if (i < nrow && rp[i + 1] - rp[i] <= SHORT_MAX) y[i] = (yadd ? yadd[i] : 0.0) + acc;
        } else {
            const int64_t c = t - nslices, i = crow[c], rb = rp[i], re = rp[i + 1], j = cidx[c];
            const int64_t b = rb + j * LCHUNK, e = min(re, b + LCHUNK);
            double acc = 0.0;
            for (int64_t k = b + lane; k < e; k += 32) acc += __ldg(&w[k]) * x[__ldg(&col[k])];
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            const int slot = cslot[c];
            if (slot < 0) {
                if (lane == 0) y[i] = (yadd ? yadd[i] : 0.0) + acc;
                continue;
            }
            const int nch = (int)((re - rb + LCHUNK - 1) / LCHUNK);
            int last = 0;
            if (lane == 0) {
                cpart[c] = acc;
                __threadfence();
                last = atomicAdd(&ccnt[slot], 1) == nch - 1;
            }
            last = __shfl_sync(0xffffffffu, last, 0);
            if (!last) continue;
            __threadfence();
            double s2 = 0.0;
            for (int q = lane; q < nch; q += 32) s2 += __ldcg(&cpart[c - j + q]);
            for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
            if (lane == 0) {
                ccnt[slot] = 0;
                y[i] = (yadd ? yadd[i] : 0.0) + s2;
            }
        }
    }
}

// ------------------------------------------------------------------ owned-piece kernels
enum { DE_SPMV = 0, DE_DOT = 1, DE_RESID = 2, DE_CHEB = 3, DE_CHEB0 = 5 };
__device__ __forceinline__ double blk_sum(double v, double *sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double r = 0.0;
    if (wid == 0) {
        r = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    }
    return r;
}
// the SpMV epilogue (solve.cu apply_epi) on the owned piece, A x reduced already
template <int EPI>
__global__ void __launch_bounds__(256) k_dist_epi(int64_t nreal, const double *__restrict__ ax,
                                                  const double *__restrict__ x, const double *__restrict__ d,
                                                  const double *__restrict__ b, double *__restrict__ dv,
                                                  double *__restrict__ y, double c1, double c2, double *partials) {
    pdl_begin();
    __shared__ double sh[8];
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nreal; i += (int64_t)gridDim.x * blockDim.x) {
        double xi = x[i], lx = d[i] * xi - ax[i];
        if (EPI == DE_SPMV) {
            y[i] = lx;
        } else if (EPI == DE_DOT) {
            y[i] = lx;
            acc += xi * lx;
        } else if (EPI == DE_RESID) {
            y[i] = b[i] - lx;
        } else if (EPI == DE_CHEB) {
            double v = c1 * dv[i] + c2 * ((b[i] - lx) / d[i]);
            dv[i] = v;
            y[i] = xi + v;
        } else {
            double v = c2 * ((b[i] - lx) / d[i]);
            dv[i] = v;
            y[i] = xi + v;
        }
    }
    if (EPI == DE_DOT) {
        double r = blk_sum(acc, sh);
        if (threadIdx.x == 0) partials[blockIdx.x] = r;
    }
}
__global__ void k_d_cheb_first(int64_t nreal, const double *b, const double *d, double inv_theta, double *x, double *dv) {
    pdl_begin();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nreal; i += (int64_t)gridDim.x * blockDim.x) {
        double v = (b[i] / d[i]) * inv_theta;
        dv[i] = v;
        x[i] = v;
    }
}
// coarse-space partial sums of a restriction: out[c] = sum_k coef_k v[slot_k] over the list of c
// 8 lanes per coarse index (lane-strided, fixed shuffle tree): a hub aggregate's
// members in this piece do not serialise one thread
__global__ void __launch_bounds__(256) k_d_gather_sum(int64_t mc, const int64_t *__restrict__ ptr,
                                                      const int32_t *__restrict__ slot, const double *__restrict__ coef,
                                                      const double *__restrict__ v, double *__restrict__ out) {
    pdl_begin();
    constexpr int G = 8;
    const int lane = threadIdx.x & 31, sub = lane & (G - 1);
    const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
    for (int64_t base = grp - (grp % (32 / G)); base < mc; base += ngrp) {  // a warp's groups move together
        const int64_t c = base + (grp % (32 / G));
        double s = 0.0;
        if (c < mc)
            for (int64_t k = ptr[c] + sub; k < ptr[c + 1]; k += G) s += (coef ? coef[k] : 1.0) * v[slot[k]];
        for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (sub == 0 && c < mc) out[c] = s;
    }
}
__global__ void k_d_prolong(int64_t nreal, const int32_t *__restrict__ cmap, const double *__restrict__ xc,
                            double *__restrict__ x) {
    pdl_begin();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nreal; i += (int64_t)gridDim.x * blockDim.x)
        x[i] += xc[cmap[i]];
}
__global__ void k_d_elim_prolong(int64_t nreal, const int32_t *__restrict__ ep_c, const int64_t *__restrict__ ep_ptr,
                                 const int32_t *__restrict__ ep_col, const double *__restrict__ ep_w,
                                 const double *__restrict__ b, const double *__restrict__ d,
                                 const double *__restrict__ xc, double *__restrict__ x) {
    pdl_begin();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nreal; i += (int64_t)gridDim.x * blockDim.x) {
        if (ep_c[i] >= 0) {
            x[i] = xc[ep_c[i]];
        } else {
            double s = b[i];
            for (int64_t k = ep_ptr[i]; k < ep_ptr[i + 1]; k++) s += ep_w[k] * xc[ep_col[k]];
            x[i] = s / d[i];
        }
    }
}
__global__ void k_d_dot_partial(int64_t n, const double *__restrict__ a, const double *__restrict__ b,
                                double *__restrict__ part) {
    pdl_begin();
    __shared__ double sh[8];
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += a[i] * (b ? b[i] : 1.0);
    double r = blk_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = r;
}
__global__ void k_d_reduce(const double *__restrict__ part, int64_t np, double *__restrict__ out) {
    pdl_begin();
    __shared__ double sh[8];
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < np; i += blockDim.x) acc += part[i];
    double r = blk_sum(acc, sh);
    if (threadIdx.x == 0) *out = r;
}
// fixed-order sum of up to 16 equally long device vectors (virtual collectives)
struct Ptrs {
    const double *p[16];
};
__global__ void k_sum_vecs(int64_t m, Ptrs src, int cnt, double *__restrict__ dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < cnt; r++) s += src.p[r][i];
        dst[i] = s;
    }
}
// PCG updates on the owned piece (scal: 0 rho, 1 pq, 2 rr, 3 sum z, 4 rho_new; world-reduced)
__global__ void k_d_xr(int64_t n, const double *p, const double *q, double *x, double *r, const double *g,
                       double *part) {
    pdl_begin();
    __shared__ double sh[8];
    double alpha = g[0] / g[1], acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        x[i] += alpha * p[i];
        double ri = r[i] - alpha * q[i];
        r[i] = ri;
        acc += ri * ri;
    }
    double t = blk_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}
__global__ void k_d_proj_dot(int64_t n, double inv_ntot, double *z, const double *r, const double *g, double *part) {
    pdl_begin();
    __shared__ double sh[8];
    double mean = g[3] * inv_ntot, acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double zi = z[i] - mean;
        z[i] = zi;
        acc += r[i] * zi;
    }
    double t = blk_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}
__global__ void k_d_p(int64_t n, const double *z, double *p, const double *g, int first) {
    pdl_begin();
    double beta = first ? 0.0 : g[4] / g[0];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = first ? z[i] : z[i] + beta * p[i];
}
__global__ void k_d_sub_mean(int64_t n, double inv_ntot, double *v, const double *g) {
    pdl_begin();
    double mean = g[3] * inv_ntot;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] -= mean;
}
__global__ void k_d_scatter_in(int64_t S, int k, PieceMap m, const double *__restrict__ full, double *__restrict__ own) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < S; q += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = m.storage_of((int64_t)k * S + q);
        own[q] = p >= 0 ? full[p] : 0.0;
    }
}
__global__ void k_d_gather_out(int64_t n, PieceMap m, const double *__restrict__ dfull, double *__restrict__ full) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
        full[p] = dfull[m.dist_of(p)];
}
__global__ void k_d_own_diag(int64_t S, int k, PieceMap m, const double *__restrict__ sd, double *__restrict__ d) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < S; q += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = m.storage_of((int64_t)k * S + q);
        d[q] = p >= 0 ? sd[p] : 1.0;
    }
}
// transfer pair lists: key = coarse index * S + owned slot (sorted -> CSR over the coarse space)
__global__ void k_d_agg_pairs(int64_t S, int k, PieceMap m, const int32_t *__restrict__ agg_s, PieceMap mc, int cdist,
                              uint64_t *__restrict__ key, int32_t *__restrict__ cmap) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < S; q += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = m.storage_of((int64_t)k * S + q);
        if (p < 0) {
            key[q] = ~0ULL;
            cmap[q] = 0;
            continue;
        }
        int64_t c = cdist ? mc.dist_of(agg_s[p]) : agg_s[p];
        key[q] = (uint64_t)c * (uint64_t)S + (uint64_t)q;
        cmap[q] = (int32_t)c;
    }
}
__global__ void k_d_elim_count(int64_t S, int k, PieceMap m, const int64_t *__restrict__ srp,
                               const int32_t *__restrict__ fmap_s, int64_t *__restrict__ cnt) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < S; q += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = m.storage_of((int64_t)k * S + q);
        cnt[q] = p < 0 ? 0 : fmap_s[p] >= 0 ? 1 : srp[p + 1] - srp[p];
    }
}
__global__ void k_d_elim_fill(int64_t S, int k, PieceMap m, PieceMap mc, int cdist, const int64_t *__restrict__ srp,
                              const int32_t *__restrict__ scol, const double *__restrict__ sw,
                              const double *__restrict__ sd, const int32_t *__restrict__ fmap_s,
                              const int64_t *__restrict__ off, uint64_t *__restrict__ key, double *__restrict__ coef,
                              int32_t *__restrict__ slot, int32_t *__restrict__ ep_c, int32_t *__restrict__ ep_col,
                              double *__restrict__ ep_w) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < S; q += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = m.storage_of((int64_t)k * S + q);
        if (p < 0) {
            ep_c[q] = 0;
            continue;
        }
        int64_t o = off[q];
        if (fmap_s[p] >= 0) {  // C row: its own b enters its coarse entry
            int64_t c = cdist ? mc.dist_of(fmap_s[p]) : fmap_s[p];
            ep_c[q] = (int32_t)c;
            key[o] = (uint64_t)c * (uint64_t)S + (uint64_t)q;
            coef[o] = 1.0;
            slot[o] = (int32_t)q;
        } else {  // F row: all its neighbours are C (F is independent)
            ep_c[q] = -1;
            double df = sd[p];
            for (int64_t e = srp[p]; e < srp[p + 1]; e++, o++) {
                int64_t c = cdist ? mc.dist_of(fmap_s[scol[e]]) : fmap_s[scol[e]];
                key[o] = (uint64_t)c * (uint64_t)S + (uint64_t)q;
                coef[o] = sw[e] / df;
                slot[o] = (int32_t)q;
                ep_col[o] = (int32_t)c;
                ep_w[o] = sw[e];
            }
        }
    }
}
__global__ void k_d_lower_bound(int64_t mc, int64_t cnt, const uint64_t *__restrict__ keys, int64_t S,
                                int64_t *__restrict__ ptr) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= mc; c += (int64_t)gridDim.x * blockDim.x) {
        uint64_t key = (uint64_t)c * (uint64_t)S;
        int64_t lo = 0, hi = cnt;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        ptr[c] = lo;
    }
}
__global__ void k_d_take_i32(int64_t cnt, const int64_t *__restrict__ idx, const int32_t *__restrict__ in,
                             int32_t *__restrict__ out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt; t += (int64_t)gridDim.x * blockDim.x)
        out[t] = in[idx[t]];
}
__global__ void k_d_take_f64(int64_t cnt, const int64_t *__restrict__ idx, const double *__restrict__ in,
                             double *__restrict__ out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt; t += (int64_t)gridDim.x * blockDim.x)
        out[t] = in[idx[t]];
}
__global__ void k_d_i64_to_i32(int64_t cnt, const int64_t *__restrict__ in, int32_t *__restrict__ out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt; t += (int64_t)gridDim.x * blockDim.x)
        out[t] = (int32_t)in[t];
}
__global__ void k_d_iota64(int64_t cnt, int64_t *v) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt; t += (int64_t)gridDim.x * blockDim.x) v[t] = t;
}

static inline unsigned dg(int64_t n) { return grid_for(n, 256, 148 * 8); }
static constexpr int DRED = 296;

template <class T>
static T d2h1(const T *p, cudaStream_t s) {
    T v;
    LAP_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, s));
    LAP_CUDA(cudaStreamSynchronize(s));
    return v;
}
static void sort_keys_idx(int64_t cnt, uint64_t *keys_in, uint64_t *keys_out, int64_t *idx_out, cudaStream_t s) {
    DBuf<int64_t> idx(cnt, s);
    k_d_iota64<<<dg(cnt), 256, 0, s>>>(cnt, idx.p);
    size_t bytes = 0;
    LAP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys_in, keys_out, idx.p, idx_out, cnt, 0, 64, s));
    DBuf<char> tmp((int64_t)bytes, s);
    LAP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, keys_in, keys_out, idx.p, idx_out, cnt, 0, 64, s));
}

// ------------------------------------------------------------------ shard construction
static void build_shard(lap_hierarchy *h, Dist &D, int l, Shard &sh, cudaStream_t s) {
    const Level &L = h->lev[l];
    DistLevel &DL = D.lev[l];
    const PieceMap &m = DL.map;
    lap_comm *c = D.c;
    const int pr = c->pr, pc = c->pc;
    const int64_t S = m.S;
    sh.gi = sh.r / pc;
    sh.gj = sh.r % pc;
    sh.nreal = real_rows(m, sh.r);
    sh.nrow = (int64_t)pc * S;
    sh.ncol = (int64_t)pr * S;
    const int64_t row_d0 = (int64_t)sh.gi * pc * S;
    const int G = group_size(L.n, L.nnz);
    // ---- 2D block (rows: row block gi, columns: column block gj, local ids), in
    // two parts: the own piece's columns and the rest of the column block
    auto build_part = [&](int part, BlockMat &B) {
        DBuf<int64_t> cnt(sh.nrow + 1, s);
        LAP_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int64_t) * (sh.nrow + 1), s));
        LAUNCH_G(G, k_blk_count, sh.nrow, s, sh.nrow, row_d0, m, pc, sh.gi, sh.gj, part, (const int64_t *)L.srp,
                 (const int32_t *)L.scol, cnt.p);
        B.rp = dal<int64_t>(sh.nrow + 1, s);
        size_t bytes = 0;
        LAP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, B.rp, sh.nrow + 1, s));
        DBuf<char> tmp((int64_t)bytes, s);
        LAP_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.p, B.rp, sh.nrow + 1, s));
        B.nnz = d2h1(B.rp + sh.nrow, s);
        B.col = dal<int32_t>(B.nnz + 1, s);
        B.w = dal<double>(B.nnz + 1, s);
        LAUNCH_G(G, k_blk_fill, sh.nrow, s, sh.nrow, row_d0, m, pc, sh.gi, sh.gj, part, (const int64_t *)L.srp,
                 (const int32_t *)L.scol, (const double *)L.sw, (const int64_t *)B.rp, B.col, B.w);
        LAP_CHECK_LAUNCH();
        // SELL-32 slices over the short rows, LCHUNK chunks over the long rows
        B.nslices = (sh.nrow + 31) / 32;
        DBuf<int64_t> width(B.nslices + 1, s);
        LAP_CUDA(cudaMemsetAsync(width.p + B.nslices, 0, sizeof(int64_t), s));
        k_blk_width<<<dg(B.nslices), 256, 0, s>>>(B.nslices, sh.nrow, B.rp, width.p);
        B.slice_ptr = dal<int64_t>(B.nslices + 1, s);
        bytes = 0;
        LAP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, width.p, B.slice_ptr, B.nslices + 1, s));
        DBuf<char> tmp2((int64_t)bytes, s);
        LAP_CUDA(cub::DeviceScan::ExclusiveSum(tmp2.p, bytes, width.p, B.slice_ptr, B.nslices + 1, s));
        int64_t tot = d2h1(B.slice_ptr + B.nslices, s);
        B.ell_col = dal<int32_t>(tot + 1, s);
        B.ell_w = dal<double>(tot + 1, s);
        k_blk_sell_fill<<<dg(B.nslices * 32), 256, 0, s>>>(B.nslices * 32, sh.nrow, B.rp, B.col, B.w, B.slice_ptr,
                                                             B.ell_col, B.ell_w);
        B.nchunks = build_chunks(B.rp, 0, sh.nrow, SHORT_MAX, &B.crow, &B.cidx, &B.cslot, &B.cpart, &B.ccnt, s);
        void *cs[] = {B.crow, B.cidx, B.cslot, B.cpart, B.ccnt};
        for (void *p : cs) g_owned->push_back(p);
        LAP_CHECK_LAUNCH();
    };
    build_part(1, sh.own);
    build_part(2, sh.rem);
    // ---- owned-piece vectors
    sh.xcol = dal<double>(sh.ncol, s);
    sh.ypart = dal<double>(sh.nrow, s);
    sh.yown = dal<double>(sh.nrow, s);
    sh.ax = dal<double>(S, s);
    double **vs[] = {&sh.b, &sh.x, &sh.x2, &sh.t, &sh.rv, &sh.dv};
    for (double **v : vs) {
        *v = dal<double>(S, s);
        LAP_CUDA(cudaMemsetAsync(*v, 0, sizeof(double) * S, s));
    }
    LAP_CUDA(cudaMemsetAsync(sh.xcol, 0, sizeof(double) * sh.ncol, s));
    LAP_CUDA(cudaMemsetAsync(sh.ypart, 0, sizeof(double) * sh.nrow, s));
    LAP_CUDA(cudaMemsetAsync(sh.ax, 0, sizeof(double) * S, s));
    sh.d = dal<double>(S, s);
    k_d_own_diag<<<dg(S), 256, 0, s>>>(S, sh.r, m, L.sd, sh.d);
    sh.partials = dal<double>(DRED, s);
    sh.scal = dal<double>(16, s);
    LAP_CUDA(cudaMemsetAsync(sh.scal, 0, sizeof(double) * 16, s));
    // ---- transfer to level l+1
    if (L.kind == KIND_COARSEST) return;
    const Level &C = h->lev[l + 1];
    PieceMap mcm = DL.next_dist ? D.lev[l + 1].map : PieceMap{};
    const int cdist = DL.next_dist ? 1 : 0;
    sh.cfull = dal<double>(DL.mc, s);
    if (DL.next_dist) sh.xcfull = dal<double>(DL.mc, s);
    (void)C;
    if (L.kind == KIND_AGG) {
        DBuf<uint64_t> key(S, s), key2(S, s);
        DBuf<int64_t> idx(S, s);
        sh.cmap = dal<int32_t>(S, s);
        k_d_agg_pairs<<<dg(S), 256, 0, s>>>(S, sh.r, m, L.agg_s, mcm, cdist, key.p, sh.cmap);
        sort_keys_idx(S, key.p, key2.p, idx.p, s);
        // pair t was emitted at owned slot q = idx[t]; pads (key ~0) sort last
        sh.members = dal<int32_t>(S, s);
        k_d_i64_to_i32<<<dg(S), 256, 0, s>>>(S, idx.p, sh.members);
        sh.mem_ptr = dal<int64_t>(DL.mc + 1, s);
        k_d_lower_bound<<<dg(DL.mc + 1), 256, 0, s>>>(DL.mc, sh.nreal, key2.p, S, sh.mem_ptr);
        LAP_CHECK_LAUNCH();
    } else {
        DBuf<int64_t> cnt(S + 1, s), off(S + 1, s);
        LAP_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int64_t) * (S + 1), s));
        k_d_elim_count<<<dg(S), 256, 0, s>>>(S, sh.r, m, L.srp, L.fmap_s, cnt.p);
        size_t bytes = 0;
        LAP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, off.p, S + 1, s));
        DBuf<char> tmp((int64_t)bytes, s);
        LAP_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.p, off.p, S + 1, s));
        int64_t T = d2h1(off.p + S, s);
        DBuf<uint64_t> key(T, s), key2(T, s);
        DBuf<double> coef(T, s);
        DBuf<int32_t> slot(T, s);
        DBuf<int64_t> idx(T, s);
        sh.ep_c = dal<int32_t>(S, s);
        sh.ep_col = dal<int32_t>(T + 1, s);
        sh.ep_w = dal<double>(T + 1, s);
        sh.ep_ptr = off.take();
        g_owned->push_back(sh.ep_ptr);
        k_d_elim_fill<<<dg(S), 256, 0, s>>>(S, sh.r, m, mcm, cdist, L.srp, L.scol, L.sw, L.sd, L.fmap_s, sh.ep_ptr,
                                            key.p, coef.p, slot.p, sh.ep_c, sh.ep_col, sh.ep_w);
        sort_keys_idx(T, key.p, key2.p, idx.p, s);
        sh.er_slot = dal<int32_t>(T + 1, s);
        sh.er_coef = dal<double>(T + 1, s);
        k_d_take_i32<<<dg(T), 256, 0, s>>>(T, idx.p, slot.p, sh.er_slot);
        k_d_take_f64<<<dg(T), 256, 0, s>>>(T, idx.p, coef.p, sh.er_coef);
        sh.er_ptr = dal<int64_t>(DL.mc + 1, s);
        k_d_lower_bound<<<dg(DL.mc + 1), 256, 0, s>>>(DL.mc, T, key2.p, S, sh.er_ptr);
        LAP_CHECK_LAUNCH();
    }
}


// ------------------------------------------------------------------ collectives
// Every operation acts on all local ranks; NCCL mode has exactly one.
struct Coll {
    lap_comm *c;
    cudaStream_t s;
    // recv[r] (pr*cnt) = concat over the column of send[(i, gj)]  (i = 0..pr-1)
    void allgather_col(const std::vector<const double *> &send, const std::vector<double *> &recv, int64_t cnt,
                       const std::vector<Shard> &sh) {
        if (!c->virt) {
            NCCL_CHECK(ncclAllGather(send[0], recv[0], (size_t)cnt, ncclDouble, c->col, s));
            return;
        }
        for (size_t a = 0; a < sh.size(); a++)
            for (int i = 0; i < c->pr; i++)
                LAP_CUDA(cudaMemcpyAsync(recv[a] + (int64_t)i * cnt, send[i * c->pc + sh[a].gj], sizeof(double) * cnt,
                                         cudaMemcpyDeviceToDevice, s));
    }
    // recv[r] (cnt) = sum over the row of segment gj of send[(gi, j)]
    void reduce_scatter_row(const std::vector<const double *> &send, const std::vector<double *> &recv, int64_t cnt,
                            const std::vector<Shard> &sh) {
        if (!c->virt) {
            NCCL_CHECK(ncclReduceScatter(send[0], recv[0], (size_t)cnt, ncclDouble, ncclSum, c->row, s));
            return;
        }
        for (size_t a = 0; a < sh.size(); a++) {
            Ptrs p{};
            for (int j = 0; j < c->pc; j++) p.p[j] = send[sh[a].gi * c->pc + j] + (int64_t)sh[a].gj * cnt;
            k_sum_vecs<<<dg(cnt), 256, 0, s>>>(cnt, p, c->pc, recv[a]);
        }
    }
    // recv[r] (cnt) = sum over all ranks of segment r of send (P*cnt)
    void reduce_scatter_world(const std::vector<const double *> &send, const std::vector<double *> &recv, int64_t cnt) {
        if (!c->virt) {
            NCCL_CHECK(ncclReduceScatter(send[0], recv[0], (size_t)cnt, ncclDouble, ncclSum, c->world, s));
            return;
        }
        for (int r = 0; r < c->P; r++) {
            Ptrs p{};
            for (int q = 0; q < c->P; q++) p.p[q] = send[q] + (int64_t)r * cnt;
            k_sum_vecs<<<dg(cnt), 256, 0, s>>>(cnt, p, c->P, recv[r]);
        }
    }
    // recv (cnt, one per process) = sum over all ranks of send
    void allreduce_world(const std::vector<const double *> &send, double *recv, int64_t cnt) {
        if (!c->virt) {
            NCCL_CHECK(ncclAllReduce(send[0], recv, (size_t)cnt, ncclDouble, ncclSum, c->world, s));
            return;
        }
        Ptrs p{};
        for (int q = 0; q < c->P; q++) p.p[q] = send[q];
        k_sum_vecs<<<dg(cnt), 256, 0, s>>>(cnt, p, c->P, recv);
    }
    // recv[r] (P*cnt) = concat over ranks of send
    void allgather_world(const std::vector<const double *> &send, const std::vector<double *> &recv, int64_t cnt) {
        if (!c->virt) {
            NCCL_CHECK(ncclAllGather(send[0], recv[0], (size_t)cnt, ncclDouble, c->world, s));
            return;
        }
        for (size_t a = 0; a < recv.size(); a++)
            for (int q = 0; q < c->P; q++)
                LAP_CUDA(cudaMemcpyAsync(recv[a] + (int64_t)q * cnt, send[q], sizeof(double) * cnt,
                                         cudaMemcpyDeviceToDevice, s));
    }
};

// ------------------------------------------------------------------ distributed operations
template <class F>
static std::vector<double *> each(std::vector<Shard> &sh, F f) {
    std::vector<double *> v;
    for (auto &x : sh) v.push_back(f(x));
    return v;
}
static std::vector<const double *> cnst(const std::vector<double *> &v) {
    return std::vector<const double *>(v.begin(), v.end());
}

// y = epilogue(L_l x) on the owned pieces: allgather(col) -> block SpMV -> reduce-scatter(row) -> epilogue
static void dist_spmv(lap_hierarchy *h, Dist &D, int l, int epi, const std::vector<double *> &x,
                      const std::vector<double *> &y, const std::vector<double *> &b, const std::vector<double *> &dv,
                      double c1, double c2, bool dot_partials, cudaStream_t s) {
    DistLevel &DL = D.lev[l];
    Coll co{D.c, s};
    const int64_t S = DL.map.S;
    auto part_spmv = [&](const BlockMat &B, int64_t nrow, const double *xin, double *yout, const double *yadd,
                         cudaStream_t st) {
        launch_pdl(k_blk_spmv, grid_for((B.nslices + B.nchunks) * 32, 256, 148 * 8), 256, st, B.nslices, nrow,
                   (const int64_t *)B.slice_ptr, (const int32_t *)B.ell_col, (const double *)B.ell_w,
                   (const int64_t *)B.rp, (const int32_t *)B.col, (const double *)B.w, B.nchunks,
                   (const int32_t *)B.crow, (const int32_t *)B.cidx, (const int32_t *)B.cslot, B.cpart, B.ccnt, xin,
                   yout, yadd);
        h->cur.launches++;
    };
    // own-piece columns first: they need no communication, so on an NCCL grid this
    // part runs on the side stream while the column allgather is in flight
    const bool fork = D.side != nullptr;
    if (fork) {
        LAP_CUDA(cudaEventRecord(D.ev_fork, s));
        LAP_CUDA(cudaStreamWaitEvent(D.side, D.ev_fork, 0));
    }
    for (size_t k = 0; k < DL.sh.size(); k++)
        part_spmv(DL.sh[k].own, DL.sh[k].nrow, x[k], DL.sh[k].yown, nullptr, fork ? D.side : s);
    if (fork) LAP_CUDA(cudaEventRecord(D.ev_join, D.side));
    co.allgather_col(cnst(x), each(DL.sh, [](Shard &a) { return a.xcol; }), S, DL.sh);
    if (fork) LAP_CUDA(cudaStreamWaitEvent(s, D.ev_join, 0));
    // the rest of the column block, added to the own part (fixed order: own + remote)
    for (auto &a : DL.sh) part_spmv(a.rem, a.nrow, a.xcol, a.ypart, a.yown, s);
    co.reduce_scatter_row(cnst(each(DL.sh, [](Shard &a) { return a.ypart; })), each(DL.sh, [](Shard &a) { return a.ax; }),
                          S, DL.sh);
    for (size_t k = 0; k < DL.sh.size(); k++) {
        Shard &a = DL.sh[k];
        const double *bb = b.empty() ? nullptr : b[k];
        double *dd = dv.empty() ? nullptr : dv[k];
        unsigned g = dot_partials ? DRED : dg(a.nreal);
        switch (epi) {
            case DE_SPMV: launch_pdl(k_dist_epi<DE_SPMV>, g, 256, s, a.nreal, (const double *)a.ax, (const double *)x[k], (const double *)a.d, bb, dd, y[k], c1, c2, a.partials); break;
            case DE_DOT: launch_pdl(k_dist_epi<DE_DOT>, g, 256, s, a.nreal, (const double *)a.ax, (const double *)x[k], (const double *)a.d, bb, dd, y[k], c1, c2, a.partials); break;
            case DE_RESID: launch_pdl(k_dist_epi<DE_RESID>, g, 256, s, a.nreal, (const double *)a.ax, (const double *)x[k], (const double *)a.d, bb, dd, y[k], c1, c2, a.partials); break;
            case DE_CHEB: launch_pdl(k_dist_epi<DE_CHEB>, g, 256, s, a.nreal, (const double *)a.ax, (const double *)x[k], (const double *)a.d, bb, dd, y[k], c1, c2, a.partials); break;
            default: launch_pdl(k_dist_epi<DE_CHEB0>, g, 256, s, a.nreal, (const double *)a.ax, (const double *)x[k], (const double *)a.d, bb, dd, y[k], c1, c2, a.partials); break;
        }
        h->cur.launches++;
    }
    h->cur.edges += h->lev[l].nnz;
    h->cur.bytes += 12 * h->lev[l].nnz + 56 * h->lev[l].n;
    LAP_CHECK_LAUNCH();
}

// world-reduced dot: every local rank reduces its piece, then the ranks' partial scalars are summed
// (fixed order); the result lands in D.gscal[slot] (one copy per process)
static void dist_dot(lap_hierarchy *h, Dist &D, std::vector<Shard> &sh, const std::vector<double *> &a,
                     const std::vector<double *> &b, int slot, bool partials_ready, cudaStream_t s) {
    Coll co{D.c, s};
    for (size_t k = 0; k < sh.size(); k++) {
        if (!partials_ready) launch_pdl(k_d_dot_partial, DRED, 256, s, sh[k].nreal, (const double *)a[k],
                                        b.empty() ? (const double *)nullptr : (const double *)b[k], sh[k].partials);
        launch_pdl(k_d_reduce, 1, 256, s, (const double *)sh[k].partials, (int64_t)DRED, sh[k].scal + slot);
        h->cur.launches += 2;
    }
    co.allreduce_world(cnst(each(sh, [slot](Shard &x) { return x.scal + slot; })), D.gscal + slot, 1);
}

static void dist_vcycle(lap_hierarchy *h, Dist &D, int l, const std::vector<double *> &b,
                        const std::vector<double *> &xout, cudaStream_t s);

// transfer from distributed level l: partial restriction sums over the coarse space, then
// reduce-scatter into the next level's pieces or allreduce into its replicated vector
static void dist_restrict_finish(lap_hierarchy *h, Dist &D, int l, cudaStream_t s) {
    DistLevel &DL = D.lev[l];
    Coll co{D.c, s};
    auto parts = cnst(each(DL.sh, [](Shard &a) { return a.cfull; }));
    if (DL.next_dist) {
        DistLevel &N = D.lev[l + 1];
        co.reduce_scatter_world(parts, each(N.sh, [](Shard &a) { return a.b; }), N.map.S);
    } else {
        co.allreduce_world(parts, h->lev[l + 1].b, DL.mc);
    }
}
// coarse x for the prolongation: allgather of the next level's pieces, or its replicated vector
static std::vector<const double *> dist_coarse_x(lap_hierarchy *h, Dist &D, int l, cudaStream_t s) {
    DistLevel &DL = D.lev[l];
    Coll co{D.c, s};
    if (DL.next_dist) {
        DistLevel &N = D.lev[l + 1];
        co.allgather_world(cnst(each(N.sh, [](Shard &a) { return a.x; })), each(DL.sh, [](Shard &a) { return a.xcfull; }),
                           N.map.S);
        return cnst(each(DL.sh, [](Shard &a) { return a.xcfull; }));
    }
    std::vector<const double *> v(DL.sh.size(), h->lev[l + 1].x);
    return v;
}

static void dist_vcycle(lap_hierarchy *h, Dist &D, int l, const std::vector<double *> &b,
                        const std::vector<double *> &xout, cudaStream_t s) {
    Level &L = h->lev[l];
    DistLevel &DL = D.lev[l];
    auto next = [&]() {
        if (D.lev[l + 1].dist) {
            dist_vcycle(h, D, l + 1, each(D.lev[l + 1].sh, [](Shard &a) { return a.b; }),
                        each(D.lev[l + 1].sh, [](Shard &a) { return a.x; }), s);
        } else {
            vcycle(h, l + 1, s);  // replicated: the single-GPU V-cycle below (same on every rank)
        }
    };
    if (L.kind == KIND_ELIM) {
        for (size_t k = 0; k < DL.sh.size(); k++) {
            Shard &a = DL.sh[k];
            launch_pdl(k_d_gather_sum, dg(DL.mc * 8), 256, s, DL.mc, (const int64_t *)a.er_ptr, (const int32_t *)a.er_slot,
                       (const double *)a.er_coef, (const double *)b[k], a.cfull);
        }
        dist_restrict_finish(h, D, l, s);
        next();
        auto xc = dist_coarse_x(h, D, l, s);
        for (size_t k = 0; k < DL.sh.size(); k++) {
            Shard &a = DL.sh[k];
            launch_pdl(k_d_elim_prolong, dg(a.nreal), 256, s, a.nreal, (const int32_t *)a.ep_c,
                       (const int64_t *)a.ep_ptr, (const int32_t *)a.ep_col, (const double *)a.ep_w,
                       (const double *)b[k], (const double *)a.d, xc[k], xout[k]);
        }
        LAP_CHECK_LAUNCH();
        return;
    }
    // aggregation level (O-S6 / O-S7; same recurrence as solve.cu vcycle_rec)
    const int K = h->p.cheby_degree;
    const double theta = L.cheb_theta, delta = L.cheb_delta, sigma = L.cheb_sigma;
    std::vector<double *> cur = each(DL.sh, [](Shard &a) { return a.x2; }), alt = each(DL.sh, [](Shard &a) { return a.t; });
    auto dv = each(DL.sh, [](Shard &a) { return a.dv; });
    for (size_t k = 0; k < DL.sh.size(); k++)
        launch_pdl(k_d_cheb_first, dg(DL.sh[k].nreal), 256, s, DL.sh[k].nreal, (const double *)b[k],
                   (const double *)DL.sh[k].d, 1.0 / theta, cur[k], dv[k]);
    double rho_old = 1.0 / sigma;
    for (int k = 1; k < K; k++) {
        double rho = 1.0 / (2.0 * sigma - rho_old);
        dist_spmv(h, D, l, DE_CHEB, cur, alt, b, dv, rho * rho_old, 2.0 * rho / delta, false, s);
        std::swap(cur, alt);
        rho_old = rho;
    }
    auto rv = each(DL.sh, [](Shard &a) { return a.rv; });
    dist_spmv(h, D, l, DE_RESID, cur, rv, b, {}, 0, 0, false, s);
    for (size_t k = 0; k < DL.sh.size(); k++) {
        Shard &a = DL.sh[k];
        launch_pdl(k_d_gather_sum, dg(DL.mc * 8), 256, s, DL.mc, (const int64_t *)a.mem_ptr, (const int32_t *)a.members,
                   (const double *)nullptr, (const double *)rv[k], a.cfull);
    }
    dist_restrict_finish(h, D, l, s);
    next();
    auto xc = dist_coarse_x(h, D, l, s);
    for (size_t k = 0; k < DL.sh.size(); k++)
        launch_pdl(k_d_prolong, dg(DL.sh[k].nreal), 256, s, DL.sh[k].nreal, (const int32_t *)DL.sh[k].cmap, xc[k], cur[k]);
    rho_old = 1.0 / sigma;
    for (int k = 0; k < K; k++) {
        auto dst = (k == K - 1) ? xout : alt;
        if (k == 0) {
            dist_spmv(h, D, l, DE_CHEB0, cur, dst, b, dv, 0.0, 1.0 / theta, false, s);
        } else {
            double rho = 1.0 / (2.0 * sigma - rho_old);
            dist_spmv(h, D, l, DE_CHEB, cur, dst, b, dv, rho * rho_old, 2.0 * rho / delta, false, s);
            rho_old = rho;
        }
        if (k < K - 1) std::swap(cur, alt);
    }
    LAP_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ PCG (O-S8) over the pieces of level 0
void dist_run_pcg(lap_hierarchy *h, double tol, int32_t *iters, double *relres, int *conv, cudaStream_t s) {
    Dist &D = *(Dist *)h->dist;
    DistLevel &L0 = D.lev[0];
    auto &sh = L0.sh;
    const int64_t n0 = h->lev[0].n;
    const double inv_n = 1.0 / (double)n0;
    Coll co{D.c, s};
    auto V = [&](double *Shard::*m) { return each(sh, [m](Shard &a) { return a.*m; }); };
    auto px = V(&Shard::px), pr = V(&Shard::pr), pz = V(&Shard::pz), pp = V(&Shard::pp), pq = V(&Shard::pq);
    double *g = D.gscal;
    auto read = [&](int slot) {
        double v;
        LAP_CUDA(cudaMemcpyAsync(&v, g + slot, sizeof(double), cudaMemcpyDeviceToHost, s));
        LAP_CUDA(cudaStreamSynchronize(s));
        return v;
    };
    // the projected b (storage order, h->pb) into the pieces
    for (auto &a : sh) {
        LAP_CUDA(cudaMemsetAsync(a.px, 0, sizeof(double) * L0.map.S, s));
        k_d_scatter_in<<<dg(L0.map.S), 256, 0, s>>>(L0.map.S, a.r, L0.map, h->pb, a.pb_in);
    }
    auto pbin = V(&Shard::pb_in);
    *conv = 0;
    dist_dot(h, D, sh, pbin, pbin, 5, false, s);
    double bn = std::sqrt(read(5));
    if (bn == 0.0) {
        *iters = 0;
        *relres = 0.0;
        *conv = 1;
        return;
    }
    auto precond_body = [&](bool first, cudaStream_t st) {
        dist_vcycle(h, D, 0, pr, pz, st);
        dist_dot(h, D, sh, pz, {}, 3, false, st);  // sum z
        for (auto &a : sh)
            launch_pdl(k_d_proj_dot, DRED, 256, st, a.nreal, inv_n, a.pz, (const double *)a.pr, (const double *)g, a.partials);
        dist_dot(h, D, sh, {}, {}, first ? 0 : 4, true, st);
        for (auto &a : sh) launch_pdl(k_d_p, dg(a.nreal), 256, st, a.nreal, (const double *)a.pz, a.pp, (const double *)g, first ? 1 : 0);
        if (!first) LAP_CUDA(cudaMemcpyAsync(g + 0, g + 4, sizeof(double), cudaMemcpyDeviceToDevice, st));
    };
    // the per-iteration step is the same launch sequence every time: replay it as
    // one CUDA graph (NCCL collectives are captured with it), captured once
    auto precond = [&](bool first) {
        h->stats.vcycles++;
        if (first || !D.use_graph || !dist_graph_enabled()) {
            precond_body(first, s);
            return;
        }
        if (!D.pgraph) {
            cudaStream_t cs;
            LAP_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
            Stats save = h->cur;
            h->cur = Stats{};
            cudaGraph_t gr;
            LAP_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
            g_capturing_flag(true);
            try {
                precond_body(false, cs);
            } catch (...) {
                g_capturing_flag(false);
                cudaStreamEndCapture(cs, &gr);
                cudaStreamDestroy(cs);
                throw;
            }
            g_capturing_flag(false);
            LAP_CUDA(cudaStreamEndCapture(cs, &gr));
            LAP_CUDA(cudaGraphInstantiate(&D.pgraph, gr, 0));
            LAP_CUDA(cudaGraphDestroy(gr));
            LAP_CUDA(cudaStreamDestroy(cs));
            D.pg_launches = h->cur.launches;
            D.pg_edges = h->cur.edges;
            D.pg_bytes = h->cur.bytes;
            h->cur = save;
        }
        LAP_CUDA(cudaGraphLaunch(D.pgraph, s));
        h->cur.launches += D.pg_launches;
        h->cur.edges += D.pg_edges;
        h->cur.bytes += D.pg_bytes;
    };
    auto true_ok = [&]() {
        dist_spmv(h, D, 0, DE_RESID, px, pq, pbin, {}, 0, 0, false, s);
        dist_dot(h, D, sh, pq, pq, 6, false, s);
        return std::sqrt(read(6)) / bn <= tol;
    };
    for (auto &a : sh) LAP_CUDA(cudaMemcpyAsync(a.pr, a.pb_in, sizeof(double) * L0.map.S, cudaMemcpyDeviceToDevice, s));
    precond(true);
    const int maxit = h->p.max_iters;
    int k;
    for (k = 1; k <= maxit; k++) {
        dist_spmv(h, D, 0, DE_DOT, pp, pq, {}, {}, 0, 0, true, s);
        dist_dot(h, D, sh, {}, {}, 1, true, s);
        for (auto &a : sh)
            launch_pdl(k_d_xr, DRED, 256, s, a.nreal, (const double *)a.pp, (const double *)a.pq, a.px, a.pr, (const double *)g, a.partials);
        dist_dot(h, D, sh, {}, {}, 2, true, s);
        double rr = read(2);
        if (std::sqrt(rr) / bn <= tol) {
            if (true_ok()) {
                *conv = 1;
                break;
            }
            for (auto &a : sh) LAP_CUDA(cudaMemcpyAsync(a.pr, a.pq, sizeof(double) * L0.map.S, cudaMemcpyDeviceToDevice, s));
        }
        if (k == maxit) break;
        precond(false);
    }
    if (k > maxit) k = maxit;
    *iters = k;
    // x -= mean(x); true residual
    dist_dot(h, D, sh, px, {}, 3, false, s);
    for (auto &a : sh) launch_pdl(k_d_sub_mean, dg(a.nreal), 256, s, a.nreal, inv_n, a.px, (const double *)g);
    dist_spmv(h, D, 0, DE_RESID, px, pq, pbin, {}, 0, 0, false, s);
    dist_dot(h, D, sh, pq, pq, 6, false, s);
    *relres = std::sqrt(read(6)) / bn;
    // pieces -> full storage-order x (h->px)
    co.allgather_world(cnst(px), std::vector<double *>(1, D.xfull), L0.map.S);
    k_d_gather_out<<<dg(n0), 256, 0, s>>>(n0, L0.map, D.xfull, h->px);
    LAP_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ construction
void build_dist(lap_hierarchy *h, lap_comm *c, cudaStream_t s, bool use_graph) {
    Dist *D = new Dist();
    D->use_graph = use_graph;
    h->dist = D;
    h->dist_owned = new std::vector<void *>();
    g_owned = (std::vector<void *> *)h->dist_owned;
    D->c = c;
    const int P = c->P;
    const int nl = (int)h->lev.size();
    int64_t thr = h->p.replicate_nnz > 0 ? h->p.replicate_nnz : std::max<int64_t>(1, h->lev[0].nnz / (32 * (int64_t)P));
    int Dn = 0;
    while (Dn < nl - 1 && h->lev[Dn].kind != KIND_COARSEST && h->lev[Dn].nnz >= thr) Dn++;
    if (Dn == 0) Dn = 1;  // level 0 is always sharded (the PCG vectors live in its pieces)
    if (h->lev[0].kind == KIND_COARSEST) Dn = 0;
    D->D = Dn;
    D->lev.resize(nl);
    std::vector<int> ranks;
    if (c->virt) for (int r = 0; r < P; r++) ranks.push_back(r);
    else ranks.push_back(c->rank);
    for (int l = 0; l < Dn; l++) {
        D->lev[l].dist = true;
        D->lev[l].map = make_map(h->lev[l].n, P);
    }
    for (int l = 0; l < Dn; l++) {
        DistLevel &DL = D->lev[l];
        DL.next_dist = (l + 1 < Dn);
        if (h->lev[l].kind != KIND_COARSEST) {
            DL.mc = DL.next_dist ? (int64_t)P * D->lev[l + 1].map.S : h->lev[l + 1].n;
        }
        for (int r : ranks) {
            Shard sh;
            sh.r = r;
            DL.sh.push_back(sh);
        }
        for (auto &sh : DL.sh) build_shard(h, *D, l, sh, s);
    }
    // PCG vectors of level 0 (pieces)
    if (Dn > 0) {
        for (auto &a : D->lev[0].sh) {
            double **vs[] = {&a.px, &a.pr, &a.pz, &a.pp, &a.pq, &a.pb_in};
            for (double **v : vs) {
                *v = dal<double>(D->lev[0].map.S, s);
                LAP_CUDA(cudaMemsetAsync(*v, 0, sizeof(double) * D->lev[0].map.S, s));
            }
        }
        D->xfull = dal<double>((int64_t)P * D->lev[0].map.S, s);
    }
    D->gscal = dal<double>(16, s);
    LAP_CUDA(cudaMemsetAsync(D->gscal, 0, sizeof(double) * 16, s));
    if (!c->virt) {  // overlap of the own-piece SpMV with the column allgather (also 1x1: tested there)
        LAP_CUDA(cudaStreamCreateWithFlags(&D->side, cudaStreamNonBlocking));
        LAP_CUDA(cudaEventCreateWithFlags(&D->ev_fork, cudaEventDisableTiming));
        LAP_CUDA(cudaEventCreateWithFlags(&D->ev_join, cudaEventDisableTiming));
    }
    LAP_CUDA(cudaStreamSynchronize(s));
    g_owned = nullptr;
}

void free_dist(lap_hierarchy *h) {
    if (!h->dist) return;
    Dist *Dd = (Dist *)h->dist;
    if (Dd->pgraph) cudaGraphExecDestroy(Dd->pgraph);
    if (Dd->side) cudaStreamDestroy(Dd->side);
    if (Dd->ev_fork) cudaEventDestroy(Dd->ev_fork);
    if (Dd->ev_join) cudaEventDestroy(Dd->ev_join);
    auto *own = (std::vector<void *> *)h->dist_owned;
    if (own) {
        for (void *p : *own) dfree(p, nullptr);
        delete own;
    }
    delete (Dist *)h->dist;
    h->dist = nullptr;
    h->dist_owned = nullptr;
}

}  // namespace lap

namespace lap {

// ------------------------------------------------------------------ distributed setup
// The coarse-operator term builds (Galerkin R L P, the Schur complement, the
// level-0 relabel of a big graph) are split by output rows over the ranks of
// the setup communicator (setup.cu build_split); here the ranges are gathered
// into the whole operator on every rank: per root rank, an ncclBroadcast of its
// rows' row_ptr / col / w pieces (grouped: NCCL has no allgatherv), then the
// row_ptr pieces are shifted by their entry offsets.  On a virtual grid (one
// process) the pieces are device copies.  Only discrete data and final CanonSum
// values move: the result is the single-GPU operator bit for bit.
static thread_local lap_comm *g_setup_comm = nullptr;

SetupCommScope::SetupCommScope(lap_comm *c) { g_setup_comm = c; }
SetupCommScope::~SetupCommScope() { g_setup_comm = nullptr; }

int setup_nranks() { return g_setup_comm ? g_setup_comm->P : 1; }
bool setup_has_comm() { return g_setup_comm != nullptr; }
std::vector<int> setup_local_ranks() {
    std::vector<int> r;
    if (!g_setup_comm) {
        r.push_back(0);
    } else if (g_setup_comm->virt) {
        for (int q = 0; q < g_setup_comm->P; q++) r.push_back(q);
    } else {
        r.push_back(g_setup_comm->rank);
    }
    return r;
}
__global__ void k_shift_rows(int64_t nr, const int64_t *__restrict__ in, int64_t off, int64_t *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nr; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[i] + off;
}
__global__ void k_shift_rows_inplace(int64_t nr, int64_t *__restrict__ v, int64_t off) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nr; i += (int64_t)gridDim.x * blockDim.x)
        v[i] += off;
}
void setup_gather(std::vector<Level> &pieces, const std::vector<int> &mine, const std::vector<int64_t> &bounds,
                  Level &out, cudaStream_t s) {
    const int P = (int)bounds.size() - 1;
    const int64_t nout = bounds[P];
    std::vector<int64_t> cnt(P, 0);
    lap_comm *c = g_setup_comm;
    const bool nccl = c && !c->virt;
    if (nccl) {  // entry counts of every rank's range
        int64_t *dc = (int64_t *)dalloc(8 * (size_t)(P + 1), s);
        LAP_CUDA(cudaMemcpyAsync(dc + P, &pieces[0].nnz, 8, cudaMemcpyHostToDevice, s));
        NCCL_CHECK(ncclAllGather(dc + P, dc, 1, ncclInt64, c->world, s));
        LAP_CUDA(cudaMemcpyAsync(cnt.data(), dc, 8 * P, cudaMemcpyDeviceToHost, s));
        LAP_CUDA(cudaStreamSynchronize(s));
        dfree(dc, s);
    } else {
        for (size_t q = 0; q < mine.size(); q++) cnt[mine[q]] = pieces[q].nnz;
    }
    std::vector<int64_t> off(P + 1, 0);
    for (int r = 0; r < P; r++) off[r + 1] = off[r] + cnt[r];
    out.n = nout;
    out.nnz = off[P];
    out.row_ptr = (int64_t *)dalloc(sizeof(int64_t) * (size_t)(nout + 1), s);
    out.col = (int32_t *)dalloc(sizeof(int32_t) * (size_t)(out.nnz + 1), s);
    out.w = (double *)dalloc(sizeof(double) * (size_t)(out.nnz + 1), s);
    if (nccl) {
        const Level &me = pieces[0];
        NCCL_CHECK(ncclGroupStart());
        for (int r = 0; r < P; r++) {
            const bool root = r == c->rank;
            const int64_t nr = bounds[r + 1] - bounds[r];
            if (nr > 0)
                NCCL_CHECK(ncclBroadcast(root ? (const void *)me.row_ptr : nullptr, out.row_ptr + bounds[r], (size_t)nr,
                                         ncclInt64, r, c->world, s));
            if (cnt[r] > 0) {
                NCCL_CHECK(ncclBroadcast(root ? (const void *)me.col : nullptr, out.col + off[r], (size_t)cnt[r],
                                         ncclInt32, r, c->world, s));
                NCCL_CHECK(ncclBroadcast(root ? (const void *)me.w : nullptr, out.w + off[r], (size_t)cnt[r],
                                         ncclFloat64, r, c->world, s));
            }
        }
        NCCL_CHECK(ncclGroupEnd());
        for (int r = 1; r < P; r++) {
            const int64_t nr = bounds[r + 1] - bounds[r];
            if (nr > 0 && off[r])
                k_shift_rows_inplace<<<dg(nr), 256, 0, s>>>(nr, out.row_ptr + bounds[r], off[r]);
        }
    } else {
        for (size_t q = 0; q < mine.size(); q++) {
            const int r = mine[q];
            const Level &pc = pieces[q];
            const int64_t nr = bounds[r + 1] - bounds[r];
            if (nr > 0) k_shift_rows<<<dg(nr), 256, 0, s>>>(nr, pc.row_ptr, off[r], out.row_ptr + bounds[r]);
            if (cnt[r] > 0) {
                LAP_CUDA(cudaMemcpyAsync(out.col + off[r], pc.col, 4 * (size_t)cnt[r], cudaMemcpyDeviceToDevice, s));
                LAP_CUDA(cudaMemcpyAsync(out.w + off[r], pc.w, 8 * (size_t)cnt[r], cudaMemcpyDeviceToDevice, s));
            }
        }
    }
    LAP_CHECK_LAUNCH();
    const int64_t tot = out.nnz;
    LAP_CUDA(cudaMemcpyAsync(out.row_ptr + nout, &tot, 8, cudaMemcpyHostToDevice, s));
    LAP_CUDA(cudaStreamSynchronize(s));  // (the host value above) before the pieces go
    for (Level &pc : pieces) {
        dfree(pc.row_ptr, s);
        dfree(pc.col, s);
        dfree(pc.w, s);
        pc.row_ptr = nullptr;
        pc.col = nullptr;
        pc.w = nullptr;
    }
}

// Row-split setup passes (elimination select, affinity, vote rounds; setup.cu
// RowSplit): every rank computed bytes [bb[r], bb[r+1]) of buf for its own
// rows; afterwards every rank holds the whole array.  NCCL: one broadcast per
// root, grouped, in place (the root's range is already in buf).  Virtual grid
// or no communicator: every range was computed into the same buffer, nothing
// moves.  Only exact per-row results move (states, indices, flags, the C_ij
// and M_i of a row): bit-identical to one GPU.
bool setup_nccl() { return g_setup_comm && !g_setup_comm->virt; }
void setup_share(void *buf, const std::vector<int64_t> &bb, cudaStream_t s) {
    if (!setup_nccl()) return;
    lap_comm *c = g_setup_comm;
    const int P = (int)bb.size() - 1;
    uint8_t *b = (uint8_t *)buf;
    NCCL_CHECK(ncclGroupStart());
    for (int r = 0; r < P; r++) {
        const int64_t cnt = bb[r + 1] - bb[r];
        if (cnt > 0) NCCL_CHECK(ncclBroadcast(b + bb[r], b + bb[r], (size_t)cnt, ncclUint8, r, c->world, s));
    }
    NCCL_CHECK(ncclGroupEnd());
}
// K4: the votes of a round = sum over ranks of each rank's own votes
// (integer sums: exact, order-free); NCCL only
void setup_sum_i32(const int32_t *in, int32_t *out, int64_t n, cudaStream_t s) {
    if (!setup_nccl() || n <= 0) return;
    NCCL_CHECK(ncclAllReduce(in, out, (size_t)n, ncclInt32, ncclSum, g_setup_comm->world, s));
}
// the Lanczos max |y| (bit patterns of non-negative doubles order like the
// values): an exact max over the ranks; NCCL only
void setup_max_u64(unsigned long long *v, cudaStream_t s) {
    if (!setup_nccl()) return;
    NCCL_CHECK(ncclAllReduce(v, v, 1, ncclUint64, ncclMax, g_setup_comm->world, s));
}
void setup_sum_u64(unsigned long long *v, int64_t n, cudaStream_t s) {
    if (!setup_nccl() || n <= 0) return;
    NCCL_CHECK(ncclAllReduce(v, v, (size_t)n, ncclUint64, ncclSum, g_setup_comm->world, s));
}
}  // namespace lap

// ------------------------------------------------------------------ C ABI (multi-GPU)
extern "C" {

lap_status lap_nccl_unique_id(uint8_t id[128]) {
    if (!id) return LAP_EINVAL;
    ncclUniqueId u;
    if (ncclGetUniqueId(&u) != ncclSuccess) {
        lap::set_error("ncclGetUniqueId failed");
        return LAP_ENCCL;
    }
    std::memcpy(id, &u, sizeof(u) < 128 ? sizeof(u) : 128);
    return LAP_OK;
}

lap_status lap_comm_create(const uint8_t nccl_id[128], int32_t rank, int32_t nranks, int32_t grid_rows,
                           int32_t grid_cols, lap_comm **out) {
    if (out) *out = nullptr;
    if (!nccl_id || !out || nranks < 1 || grid_rows < 1 || grid_cols < 1 || grid_rows * grid_cols != nranks ||
        rank < 0 || rank >= nranks || nranks > 16) {
        lap::set_error("lap_comm_create: invalid arguments");
        return LAP_EINVAL;
    }
    lap_comm *c = new lap_comm();
    c->pr = grid_rows;
    c->pc = grid_cols;
    c->P = nranks;
    c->virt = 0;
    c->rank = rank;
    ncclUniqueId u;
    std::memcpy(&u, nccl_id, sizeof(u));
    ncclResult_t r = ncclCommInitRank(&c->world, nranks, u, rank);
    if (r == ncclSuccess) r = ncclCommSplit(c->world, rank / grid_cols, rank % grid_cols, &c->row, nullptr);
    if (r == ncclSuccess) r = ncclCommSplit(c->world, rank % grid_cols, rank / grid_cols, &c->col, nullptr);
    if (r != ncclSuccess) {
        lap::set_error(std::string("lap_comm_create: ") + ncclGetErrorString(r));
        if (c->col) ncclCommDestroy(c->col);
        if (c->row) ncclCommDestroy(c->row);
        if (c->world) ncclCommDestroy(c->world);
        delete c;
        return LAP_ENCCL;
    }
    *out = c;
    return LAP_OK;
}

lap_status lap_comm_create_virtual(int32_t grid_rows, int32_t grid_cols, lap_comm **out) {
    if (out) *out = nullptr;
    if (!out || grid_rows < 1 || grid_cols < 1 || grid_rows * grid_cols > 16) {
        lap::set_error("lap_comm_create_virtual: invalid arguments (1 <= pr*pc <= 16)");
        return LAP_EINVAL;
    }
    lap_comm *c = new lap_comm();
    c->pr = grid_rows;
    c->pc = grid_cols;
    c->P = grid_rows * grid_cols;
    c->virt = 1;
    *out = c;
    return LAP_OK;
}

void lap_comm_free(lap_comm *c) {
    if (!c) return;
    if (c->col) ncclCommDestroy(c->col);
    if (c->row) ncclCommDestroy(c->row);
    if (c->world) ncclCommDestroy(c->world);
    delete c;
}

lap_status lap_comm_info(const lap_comm *c, int32_t *rank, int32_t *nranks, int32_t *grid_rows, int32_t *grid_cols,
                         int32_t *is_virtual) {
    if (!c) return LAP_EINVAL;
    if (rank) *rank = c->rank;
    if (nranks) *nranks = c->P;
    if (grid_rows) *grid_rows = c->pr;
    if (grid_cols) *grid_cols = c->pc;
    if (is_virtual) *is_virtual = c->virt;
    return LAP_OK;
}

lap_status lap_dist_index(int64_t n, int32_t nranks, int64_t m, const int64_t *rows, int64_t *dist,
                          int64_t *piece_size) {
    if (n < 0 || nranks < 1 || (m > 0 && (!rows || !dist))) return LAP_EINVAL;
    lap::PieceMap pm = lap::make_map(n, nranks);
    if (piece_size) *piece_size = pm.S;
    for (int64_t t = 0; t < m; t++) {
        if (rows[t] < 0 || rows[t] >= n) return LAP_EINVAL;
        dist[t] = pm.dist_of(rows[t]);
    }
    return LAP_OK;
}

lap_status lap_setup_split(int64_t nout, const int64_t *cum, int32_t nranks, int64_t *bounds) {
    if (nout < 0 || !cum || !bounds || nranks < 1) return LAP_EINVAL;
    for (int64_t o = 0; o < nout; o++)
        if (cum[o + 1] < cum[o] || cum[o] < 0) return LAP_EINVAL;
    for (int r = 0; r <= nranks; r++) bounds[r] = lap::split_bound(r, nranks, nout, [&](int64_t o) { return cum[o]; });
    return LAP_OK;
}

}  // extern "C"
