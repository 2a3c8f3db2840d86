// lap_internal.cuh -- internal structures and device helpers of liblap.so.
// B200 (sm_100a) only.  Not part of the ABI (see include/lap.h).
#pragma once
#include <cuda_runtime.h>
#include <cub/cub.cuh>
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/lap.h"

namespace lap {

extern int64_t g_kl;  // setup-phase kernel launch counter (setup.cu)

// ---------------------------------------------------------------- errors
struct Error {
    lap_status code;
    std::string msg;
};
void set_error(const std::string &m);

#define LAP_STR2(x) #x
#define LAP_STR(x) LAP_STR2(x)
#define LAP_CUDA(call)                                                                          \
    do {                                                                                        \
        cudaError_t _e = (call);                                                                \
        if (_e != cudaSuccess)                                                                  \
            throw ::lap::Error{_e == cudaErrorMemoryAllocation ? LAP_ENOMEM : LAP_ECUDA,        \
                               std::string(__FILE__ ":" LAP_STR(__LINE__) " ") + #call + ": " + \
                                   cudaGetErrorString(_e)};                                     \
    } while (0)

// LAP_DEBUG_SYNC=1 in the environment: synchronise after every launch check
bool debug_sync();
#define LAP_CHECK_LAUNCH()                                   \
    do {                                                     \
        LAP_CUDA(cudaGetLastError());                        \
        if (::lap::debug_sync()) LAP_CUDA(cudaDeviceSynchronize()); \
    } while (0)

// ---------------------------------------------------------------- memory
// Stream-ordered device allocation (cudaMallocAsync pool).
void *dalloc(size_t bytes, cudaStream_t s);
cudaMemPool_t lib_pool();
void dfree(void *p, cudaStream_t s);

template <class T>
struct DBuf {
    T *p = nullptr;
    int64_t n = 0;
    cudaStream_t s = nullptr;
    DBuf() = default;
    DBuf(int64_t count, cudaStream_t st) { alloc(count, st); }
    void alloc(int64_t count, cudaStream_t st) {
        release();
        s = st;
        n = count;
        p = (T *)dalloc(sizeof(T) * (size_t)(count > 0 ? count : 1), st);
    }
    void release() {
        if (p) dfree(p, s);
        p = nullptr;
        n = 0;
    }
    T *take() {
        T *q = p;
        p = nullptr;
        n = 0;
        return q;
    }
    ~DBuf() { release(); }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
};

// ---------------------------------------------------------------- levels
enum { KIND_AGG = 0, KIND_ELIM = 1, KIND_COARSEST = 2 };

// Solve-phase storage (H0).  The hierarchy's logical ids are fixed by the
// method (random order, aggregate numbering: bit-identical to the oracle);
// the solve kernels run on a per-level STORAGE ORDER chosen for the GPU:
//   key(level 0)   = caller's vertex id (undoes Pi_rand for locality)
//   key(aggregate) = min storage position of its members
//   key(C vertex)  = its storage position on the finer level
// sorted by (degree class, key), so each class is a contiguous row range:
//   class 0: deg <= 64        SELL-32 slices (warp per 32-row slice, thread per row,
//                             column-major padded to the slice's max degree; rows
//                             degree-sorted first when natural order pads > 20%)
//   classes 1-3: deg 65..1024, 1025..16384, > 16384 (grouped by magnitude);
//                all long rows are cut into LCHUNK-entry chunks, one warp per
//                chunk, combined in chunk order by the last-arriving warp
// The SpMV is one launch over the work list [SELL slices | long-row chunks].
constexpr int NCLASS = 4;
constexpr int64_t SHORT_MAX = 64;
constexpr int64_t HUB_CHUNK = 16384;  // class 2/3 boundary (storage grouping only)
constexpr int64_t LCHUNK = 1024;      // long-row chunk (entries per warp work item)
constexpr int64_t SETUP_LONG = 4096;   // setup row kernels: longer rows go to LCHUNK warp chunks
constexpr int64_t RESTRICT_SHORT = 64;  // restriction: aggregates with more members are chunked
constexpr int64_t ELIM_SHORT = 32;    // elimination restriction: longer coarse lists are chunked
constexpr int64_t DTAIL_MAX_N = 3072;  // the V-cycle below the first level this small is one dense operator (tail.cu)
constexpr int64_t NB4_MIN_NNZ = 4000000;  // SELL batch width 4 for levels this big with avg degree <= 8
constexpr int64_t SMEM_X_MAX = 26624;   // levels with n <= this (208 KB of x) ...
constexpr int64_t SMEM_X_MIN_DEG = 256; // ... and average degree >= this gather x from shared memory

struct Level {
    int kind = KIND_COARSEST;
    int64_t n = 0, nnz = 0;
    // logical CSR (setup numbering, bit-identical to the oracle)
    int64_t *row_ptr = nullptr;
    int32_t *col = nullptr;
    double *w = nullptr;
    double *d = nullptr;
    double maxw = 0.0;
    int64_t maxdeg = 0;             // longest row (setup kernels' hub handling; known before storage)
    bool logical_released = false;  // logical row_ptr/col/w freed after storage (params.keep_logical)
    bool cols_sorted = true;        // logical rows in ascending column order (level 0: not by default)
    int32_t *rowof = nullptr;       // setup only: row of every stored entry (not owned)
    // aggregation (logical)
    double lambda = 0.0;
    int64_t m = 0;
    int32_t *agg = nullptr;
    double *S = nullptr;          // optional (keep_strength)
    // elimination (logical)
    int64_t nF = 0;
    int32_t *fmap = nullptr;      // n: C -> coarse index, F -> -1-slot
    int32_t *cid = nullptr;       // nC: logical fine id of coarse index
    int32_t *fid = nullptr;       // nF
    int64_t *ct_ptr = nullptr;    // nC+1: transposed L_FC (coarse -> F neighbours)
    int32_t *ct_f = nullptr;
    double *ct_coef = nullptr;    // w_fc / d_f
    // coarsest (logical)
    double *pinv = nullptr;
    // ---- solve storage (see above)
    int32_t *sid = nullptr;       // storage -> logical
    int32_t *spos = nullptr;      // logical -> storage
    int64_t *srp = nullptr;
    int32_t *scol = nullptr;
    double *sw = nullptr, *sd = nullptr;
    int64_t c_end[NCLASS] = {0, 0, 0, 0};
    int64_t nslices = 0;            // SELL-32 slices over the short class
    int64_t *slice_ptr = nullptr;   // nslices+1 offsets into ell_* (multiples of 32)
    int32_t *ell_col = nullptr;     // padded entries: column (own row for padding)
    double *ell_w = nullptr;        // padded entries: weight (0 for padding)
    bool sell_sorted = false;       // short rows degree-sorted
    bool smem_x = false;            // small dense-ish level: k_spmv_smem (x in shared memory, 16-bit columns)
    int spmv_nb = 8;                // SELL batch width of k_spmv (8, or 4 for mid-size levels)
    bool unit = false;              // every stored weight is 1 (level 0 of a unit-weight graph): the
                                    // solve SpMV reads the pattern only, 4 instead of 12 B per entry (N4)
    int spmv_vec = 0;               // > 0: k_spmv_vec, G lanes per row over the CSR (solve.cu)
    uint16_t *ell_col16 = nullptr;  // smem_x: 16-bit copies of ell_col / scol
    uint16_t *scol16 = nullptr;
    int64_t nchunks = 0;            // LCHUNK chunks over the long rows [c_end[0], n)
    int32_t *chunk_row = nullptr;   // chunk -> storage row
    int32_t *chunk_idx = nullptr;   // chunk -> index within its row
    int32_t *chunk_slot = nullptr;  // chunk -> arrival counter slot (-1: one-chunk row)
    int32_t *chunk_cnt = nullptr;   // n - c_end[0] arrival counters (kept at 0 between launches)
    double *chunk_part = nullptr;
    int64_t nmulti = 0;             // rows of several chunks (slots 0..nmulti-1)
    double *mdot = nullptr;         // their dot-epilogue terms, 3 per slot
    int *mdone = nullptr;           // block-arrival counter of the dot fix-up (kept at 0)
    // column-tiled "x-stationary" layout (xt.cu): dense-ish levels too big for x
    // in shared memory; a CTA owns a row block and sweeps x tile by tile
    bool xt = false;
    int xt_nb = 0, xt_T = 0, xt_W = 0, xt_rmax = 0;  // row blocks, tiles, tile width (doubles), max rows per block
    int64_t *xt_rb = nullptr;       // nb+1 storage-row boundaries of the row blocks
    int64_t *xt_seg = nullptr;      // nb*T+1 start of segment (block, tile) (global entry index)
    int32_t *xt_wo = nullptr;       // nb*T*(XT_NW+1) warp offsets inside each segment
    uint32_t *xt_rc = nullptr;      // nnz: (local row << 16) | local column
    double *xt_w = nullptr;         // nnz
    // transfer maps in storage space
    int32_t *agg_s = nullptr;       // agg: coarse storage index of each fine storage row
    int64_t *mem_ptr = nullptr;     // agg: coarse storage index -> members (m+1)
    int32_t *members = nullptr;     // agg: fine storage rows, ascending
    int32_t *cid_s = nullptr;       // elim: fine storage row of each coarse storage index
    int32_t *flist = nullptr;       // elim: fine storage rows of F (ascending), nF
    int64_t *ct_ptr_s = nullptr;    // elim: coarse storage -> F neighbours (storage), coef
    int32_t *ct_f_s = nullptr;
    double *ct_coef_s = nullptr;
    int64_t rs_nchunks = 0;         // agg: LCHUNK chunks of the aggregates with more than RESTRICT_SHORT members
    int32_t *rs_crow = nullptr, *rs_cidx = nullptr, *rs_cslot = nullptr, *rs_ccnt = nullptr;
    double *rs_cpart = nullptr;
    int64_t ct_nchunks = 0;         // elim: LCHUNK chunks of the coarse lists longer than ELIM_SHORT
    int32_t *ct_crow = nullptr, *ct_cidx = nullptr, *ct_cslot = nullptr, *ct_ccnt = nullptr;
    double *ct_cpart = nullptr;
    int32_t *fmap_s = nullptr;      // elim: coarse storage index of a C storage row, -1 for F
    double *pinv_s = nullptr;       // coarsest: L^+ in storage order
    double *dense = nullptr;        // dense-tail level: M = [V(l, e_j)] (n x n, column-major; tail.cu)
    double *dense_part = nullptr;   // dense-tail GEMV: split partials, per-tile arrival counters
    int *dense_cnt = nullptr;
    // Chebyshev constants (O-S6), host
    double cheb_theta = 0, cheb_delta = 0, cheb_sigma = 0;
    // solve work vectors (storage order, length n >= 1)
    double *b = nullptr, *x = nullptr, *x2 = nullptr, *t = nullptr, *r = nullptr, *dv = nullptr;
    // K-cycle inner FCG(1) (aggregation levels l >= 1; solve.cu): direction,
    // L*direction, preconditioned residual, residual; 8 device scalars
    double *kp = nullptr, *kq = nullptr, *kz = nullptr, *kr = nullptr, *ksc = nullptr;
};

struct Stats {
    int64_t launches = 0;
    int64_t edges = 0;
    int64_t bytes = 0;
};

}  // namespace lap

struct lap_hierarchy {
    lap_params p;
    int64_t n0 = 0;
    int64_t *perm = nullptr;       // device: perm[i] = internal id of caller vertex i
    int64_t *cmap = nullptr;       // device: caller vertex -> level-0 storage row
    std::vector<lap::Level> lev;
    lap_status status = LAP_OK;
    // PCG workspaces (level 0, internal numbering)
    double *pb = nullptr, *px = nullptr, *pr = nullptr, *pz = nullptr, *pp = nullptr, *pq = nullptr;
    double *scal = nullptr;        // device scalars
    double *partials = nullptr;    // reduction partials
    int64_t npartials = 0;
    double *host_scal = nullptr;   // pinned
    // caller-buffer staging
    double *stage_in = nullptr, *stage_out = nullptr;
    // graph of the V-cycle
    cudaGraphExec_t vgraph = nullptr;
    cudaStream_t vgraph_stream = nullptr;
    // the whole PCG loop as resident graphs (WHILE conditional node, solve.cu)
    cudaGraphExec_t pcg_start = nullptr, pcg_resume = nullptr;
    void *pcg_counts = nullptr;
    int dtail_level = -1;          // level whose V-cycle is the dense operator lev[].dense (tail.cu)
    void *ktail = nullptr;         // K-cycle below a small level as one cluster program (ktail.cu)
    std::vector<void *> blk;       // block (many right-hand sides) workspaces per width (block.cu)
    // multi-GPU shards (dist.cu), NULL for a single-GPU hierarchy
    void *dist = nullptr;
    void *dist_owned = nullptr;
    lap_stats stats{};
    lap::Stats cur;
    int device = 0;
};

namespace lap {

// ---------------------------------------------------------------- distributed setup (dist.cu)
// The communicator of the setup in progress (lap_setup_dist), else none: the
// coarse-operator term builds are then split over its ranks (setup.cu
// build_split) and gathered here.
int setup_nranks();                   // 1 without a setup communicator
bool setup_has_comm();
std::vector<int> setup_local_ranks(); // ranks this process builds: {rank} (NCCL) or 0..P-1 (virtual grid)
// pieces[q] = rows [bounds[r], bounds[r+1]) of the operator for r = mine[q]
// (local row_ptr from 0); out <- the whole operator's row_ptr / col / w / nnz
void setup_gather(std::vector<Level> &pieces, const std::vector<int> &mine, const std::vector<int64_t> &bounds,
                  Level &out, cudaStream_t s);
// row-split setup passes: a real NCCL setup communicator?; bytes [bb[r], bb[r+1])
// of buf broadcast from rank r to all (in place; no-op without NCCL); integer
// sums over the ranks (no-op without NCCL)
bool setup_nccl();
void setup_share(void *buf, const std::vector<int64_t> &bb, cudaStream_t s);
void setup_sum_i32(const int32_t *in, int32_t *out, int64_t n, cudaStream_t s);
void setup_sum_u64(unsigned long long *v, int64_t n, cudaStream_t s);
void setup_max_u64(unsigned long long *v, cudaStream_t s);
// the split rule of a term build over P ranks (device: setup.cu k_split_bounds;
// host: lap_setup_split): bounds[r] = the first output row o with
// cum(o) * P >= r * cum(nout), cum(o) = terms of the rows before o
template <class Cum>
__host__ __device__ inline int64_t split_bound(int r, int P, int64_t nout, Cum cum) {
    if (r <= 0) return 0;
    if (r >= P) return nout;
    const __int128 want = (__int128)r * cum(nout);
    int64_t lo = 0, hi = nout;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((__int128)cum(mid) * P >= want) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}
struct SetupCommScope {  // lap_setup_dist: the setup runs under this communicator
    explicit SetupCommScope(lap_comm *c);
    ~SetupCommScope();
};

// ---------------------------------------------------------------- kernels (host launchers)
// setup (setup.cu)
void build_hierarchy(lap_hierarchy *h, const lap_graph *g, cudaStream_t s);
void import_hierarchy(lap_hierarchy *h, const char *dir, cudaStream_t s);
void finalize_solve_structures(lap_hierarchy *h, cudaStream_t s);

// solve (solve.cu)
enum EpiKind { EPI_SPMV = 0, EPI_SPMV_DOT = 1, EPI_RESID = 2, EPI_CHEB = 3, EPI_LANCZOS = 4 };
struct EpiArgs {
    const double *x = nullptr;    // input vector (gathered)
    double *y = nullptr;          // output (SPMV / RESID r / CHEB x_out)
    const double *b = nullptr;    // rhs (RESID / CHEB)
    double *dv = nullptr;         // Chebyshev direction (in/out)
    const double *rs = nullptr;   // Lanczos: D^-1/2 (y_i = rs_i (L (rs o v))_i - beta_prev vp_i)
    const double *v = nullptr, *vp = nullptr, *lz = nullptr;  // Lanczos: v, v_prev, device scalars
    double c1 = 0, c2 = 0;        // CHEB: dv = c1 dv + c2 D^-1 r
    double *partials = nullptr;   // SPMV_DOT partial sums (one per block per bin)
};
void spmv_level(lap_hierarchy *h, const Level &L, EpiKind kind, const EpiArgs &a, cudaStream_t s);
// storage (storage.cu)
void build_storage(lap_hierarchy *h, int l, cudaStream_t s);
size_t device_free_estimate();  // lap_api.cu
void trace_mark(const char *what);  // LAP_SETUP_TRACE phase mark (setup.cu)
// every row of a CSR sorted by column (distinct columns < 2^cbits): kin/vin -> kout/vout
void sort_rows(int64_t n, const int64_t *rp, int64_t nnz, int cbits, const int32_t *kin, const double *vin,
               int32_t *kout, double *vout, cudaStream_t s);
// P A P^T with sorted rows: new row p = old row sid[p], column c -> spos[c]; writes srp (n+1),
// scol / sw (nnz); w NULL = unit weights
void permute_csr(int64_t n, int64_t nnz, const int32_t *sid, const int32_t *spos, const int64_t *rp,
                 const int32_t *col, const double *w, int64_t *srp, int32_t *scol, double *sw, bool sort_cols,
                 int64_t maxlen, cudaStream_t s);
// the same rows sorted into scol / sw with srp already built; maxlen bounds the row length
// (rows of sort_max < len <= band_hi are permuted but keep their column order)
void permute_sorted_rows(int64_t n, int64_t nnz, const int32_t *sid, const int32_t *spos, const int64_t *rp,
                         const int32_t *col, const double *w, const int64_t *srp, int32_t *scol, double *sw,
                         int64_t maxlen, cudaStream_t s, int64_t sort_max = INT64_MAX,
                         int64_t band_hi = INT64_MAX);
void build_transfers(lap_hierarchy *h, cudaStream_t s);
// column-tiled SpMV layout (xt.cu)
constexpr int XT_NW = 16;             // warps per CTA (512 threads)
constexpr size_t XT_SMEM_MAX = 220 * 1024;  // dynamic shared memory of k_spmv_xt: 8 (2 W + rows per block)
bool xt_eligible(const Level &L, int l);
void build_xt(Level &L, cudaStream_t s);
// LCHUNK work items over the rows [row0, row0+nrows) of a CSR longer than minlen
int64_t build_chunks(const int64_t *rp, int64_t row0, int64_t nrows, int64_t minlen, int32_t **crow, int32_t **cidx,
                     int32_t **cslot, double **cpart, int32_t **ccnt, cudaStream_t s, int64_t *nmulti = nullptr);
int64_t spmv_partial_slots(const Level &L);
void vcycle(lap_hierarchy *h, int l, cudaStream_t s);   // x_l = V(l, b_l)
void run_pcg(lap_hierarchy *h, double tol, int32_t *iters, double *relres, int *conv, cudaStream_t s);
void capture_pcg(lap_hierarchy *h);
// dense tail (tail.cu)
void build_dense_tail(lap_hierarchy *h, cudaStream_t s);
void launch_dense_gemv(const Level &L, const double *b, double *x, cudaStream_t s);
void kcycle_level(lap_hierarchy *h, int l, bool with_fcg, cudaStream_t s);  // N2 (solve.cu)
void build_ktail(lap_hierarchy *h, cudaStream_t s);                          // N2 (ktail.cu)
void free_ktail(lap_hierarchy *h, cudaStream_t s);
bool ktail_launch(lap_hierarchy *h, int l, bool pre0_done, cudaStream_t s);
void solve_block(lap_hierarchy *h, int k, const double *B, double *X, double tol, int32_t *iters, double *relres,
                 int *conv, cudaStream_t s);                                   // N4 (block.cu)
void free_block(lap_hierarchy *h);
void random_stream(int which, uint64_t seed, int level, int attempt, int64_t n, void *out, cudaStream_t s);
// multi-GPU (dist.cu)
void build_dist(lap_hierarchy *h, lap_comm *c, cudaStream_t s, bool use_graph = true);
void free_dist(lap_hierarchy *h);
void dist_run_pcg(lap_hierarchy *h, double tol, int32_t *iters, double *relres, int *conv, cudaStream_t s);
void free_pcg(lap_hierarchy *h);

// small shared reductions (solve.cu)
void dot(lap_hierarchy *h, const double *a, const double *b, int64_t n, double *out, cudaStream_t s);
void reduce_partials(lap_hierarchy *h, const double *partials, int64_t np, double *out, cudaStream_t s);

inline unsigned grid_for(int64_t work, int threads, int64_t cap = 148 * 32) {
    int64_t g = (work + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

// ---------------------------------------------------------------- row groups
// Row groups: a row is handled by G lanes (G | 32, chosen per level from the
// average degree, group_size()), so low-degree levels do not idle 80% of a
// warp and long rows still get several lanes.  Every lane of a warp runs the
// same number of outer iterations (rows past n are empty), so the group
// shuffles below always see converged warps.  All reductions done this way
// are exact (integer / int128 / max / total-order arg-max), so the result is
// independent of G.
#define GROUP_LOOP_BEGIN(G, n)                                                         \
    const int lane = threadIdx.x & 31, gl = lane & ((G)-1);                            \
    (void)gl;                                                                          \
    const int64_t _gpw = 32 / (G);                                                     \
    const int64_t _stride = (((int64_t)gridDim.x * blockDim.x) >> 5) * _gpw;           \
    for (int64_t _base = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * _gpw; \
         _base < (n); _base += _stride) {                                              \
        const int64_t i = _base + lane / (G);                                          \
        const bool live = i < (n);                                                     \
        (void)live;
#define GROUP_LOOP_END }
// the same over rows [r0, r1) (row-split setup passes)
#define GROUP_LOOP_RANGE_BEGIN(G, r0, r1)                                              \
    const int lane = threadIdx.x & 31, gl = lane & ((G)-1);                            \
    (void)gl;                                                                          \
    const int64_t _gpw = 32 / (G);                                                     \
    const int64_t _stride = (((int64_t)gridDim.x * blockDim.x) >> 5) * _gpw;           \
    for (int64_t _base = (r0) + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * _gpw; \
         _base < (r1); _base += _stride) {                                             \
        const int64_t i = _base + lane / (G);                                          \
        const bool live = i < (r1);                                                    \
        (void)live;

template <int G, class T>
__device__ __forceinline__ T grp_sum(T v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
int group_shift();  // LAP_GSHIFT (lap_api.cu): experiments with narrower groups
// Lanes per row.  all_short: the level has no row longer than SHORT_MAX
// (known once its storage is built), so narrow groups cannot serialise a hub
// and the per-row group reductions become the cost (3D grid: setup 24 -> 21
// ms at one lane per row); with hubs keep G near the average degree.
inline int group_size(int64_t n, int64_t nnz, bool all_short = false) {
    double avg = n > 0 ? (double)nnz / (double)n : 0.0;
    int g = all_short ? (avg <= 8.0 ? 1 : avg <= 16.0 ? 2 : 4)
                      : (avg <= 4.0 ? 4 : avg <= 8.0 ? 8 : avg <= 16.0 ? 16 : 32);
    g >>= group_shift();
    return g < 1 ? 1 : g;
}
#define LAUNCH_G(G, kern, rows, s, ...)                                                                 \
    do {                                                                                                \
        switch (G) {                                                                                    \
            case 1: kern<1><<<grid_for((rows) * 1, 256, 148 * 16), 256, 0, s>>>(__VA_ARGS__); break;    \
            case 2: kern<2><<<grid_for((rows) * 2, 256, 148 * 16), 256, 0, s>>>(__VA_ARGS__); break;    \
            case 4: kern<4><<<grid_for((rows) * 4, 256, 148 * 16), 256, 0, s>>>(__VA_ARGS__); break;    \
            case 8: kern<8><<<grid_for((rows) * 8, 256, 148 * 16), 256, 0, s>>>(__VA_ARGS__); break;    \
            case 16: kern<16><<<grid_for((rows) * 16, 256, 148 * 16), 256, 0, s>>>(__VA_ARGS__); break; \
            default: kern<32><<<grid_for((rows) * 32, 256, 148 * 16), 256, 0, s>>>(__VA_ARGS__); break; \
        }                                                                                               \
        ++g_kl;                                                                                         \
    } while (0)

// ballot-compacted emission over a row in ascending column order: entries k of
// row i with pred(k) go to out[o + rank]; the warp loops to the longest row
// (EMIT sees the entry index k and its output position p)
#define GROUP_COMPACT_ROW(G, kb, ke, o, PRED, EMIT)                                                   \
    {                                                                                                 \
        const unsigned _gmask = ((G) == 32 ? 0xffffffffu : ((1u << (G)) - 1u)) << (lane & ~((G)-1)); \
        int64_t _len = (ke) - (kb);                                                                   \
        for (int _sh = 16; _sh > 0; _sh >>= 1) {                                                      \
            int64_t _t2 = __shfl_xor_sync(0xffffffffu, _len, _sh);                                    \
            _len = _t2 > _len ? _t2 : _len;                                                           \
        }                                                                                             \
        for (int64_t _q = 0; _q < _len; _q += (G)) {                                                  \
            int64_t k = (kb) + _q + gl;                                                               \
            bool _take = k < (ke) && (PRED);                                                          \
            unsigned _bal = __ballot_sync(0xffffffffu, _take) & _gmask;                               \
            if (_take) {                                                                              \
                int64_t p = (o) + __popc(_bal & ((1u << lane) - 1));                                  \
                EMIT;                                                                                 \
            }                                                                                         \
            (o) += __popc(_bal);                                                                      \
        }                                                                                             \
    }
// ---------------------------------------------------------------- entry-parallel helpers
// row of stored entry t of a CSR with n rows: the largest i with rp[i] <= t
// (empty rows are skipped).  Consecutive t of a warp follow the same path, so
// the search runs out of L1.
__device__ __forceinline__ int64_t row_of(const int64_t *__restrict__ rp, int64_t n, int64_t t) {
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) >> 1;
        if (rp[mid] <= t) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}
// Entry-parallel filtered emission: a 256-thread block claims contiguous
// output space with ONE atomicAdd on *cursor per 256 entries (block prefix
// sum of the predicate).  The output ORDER depends on block scheduling, so
// this is only used where the emitted terms are sorted by key and combined
// by an order-independent CanonSum afterwards (Galerkin, Schur): the level
// built from them is bitwise deterministic.
#define ENTRY_EMIT_LOOP(nent, cursor, TAKE, EMIT)                                                   \
    {                                                                                              \
        typedef cub::BlockScan<int, 256> _BS;                                                      \
        __shared__ typename _BS::TempStorage _ts;                                                  \
        __shared__ unsigned long long _boff;                                                       \
        for (int64_t _b0 = (int64_t)blockIdx.x * 256; _b0 < (nent); _b0 += (int64_t)gridDim.x * 256) { \
            const int64_t t = _b0 + threadIdx.x;                                                   \
            bool take = false;                                                                     \
            if (t < (nent)) { TAKE; }                                                              \
            int _rk, _tot;                                                                         \
            _BS(_ts).ExclusiveSum(take ? 1 : 0, _rk, _tot);                                        \
            if (threadIdx.x == 0) _boff = _tot ? atomicAdd((cursor), (unsigned long long)_tot) : 0ULL; \
            __syncthreads();                                                                       \
            if (take) {                                                                            \
                const int64_t p = (int64_t)_boff + _rk;                                            \
                EMIT;                                                                              \
            }                                                                                      \
            __syncthreads();                                                                       \
        }                                                                                          \
    }

// ---------------------------------------------------------------- programmatic dependent launch
// Solve-phase kernels are chained with programmatic dependent launch (PDL,
// sm_90+): each kernel is launched with programmatic stream serialization,
// lets its dependents launch as soon as all of its CTAs are resident
// (griddepcontrol.launch_dependents) and waits for its predecessor's memory
// (griddepcontrol.wait) before touching any input.  Inside the captured
// V-cycle / PCG graphs this hides the ~2-4 us launch + ramp latency of every
// small coarse-level kernel behind its predecessor's tail.  Without the
// launch attribute both instructions are no-ops.  LAP_PDL=0 disables it.
bool pdl_enabled();
__device__ __forceinline__ void pdl_begin() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    LAP_CUDA(cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...));
}
template <typename... KArgs, typename... Args>
inline void launch_pdl_smem(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                            Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    LAP_CUDA(cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...));
}

}  // namespace lap
