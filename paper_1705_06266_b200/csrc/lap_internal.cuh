// lap_internal.cuh -- internal structures and device helpers of liblap.so.
// B200 (sm_100a) only.  Not part of the ABI (see include/lap.h).
#pragma once
#include <cuda_runtime.h>
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

// Degree-binned row schedule for the SpMV (H0).  Bins by stored degree:
//   0: deg <= 8      -> 8 lanes per row
//   1: 9..32         -> 32 lanes (warp) per row
//   2: 33..1024      -> warp per row, unrolled
//   3: 1025..16384   -> one 256-thread block per row
//   4: > 16384       -> split into 16384-entry chunks (block per chunk) + ordered combine
constexpr int NBINS = 5;
constexpr int64_t HUB_CHUNK = 16384;

struct RowBins {
    int64_t cnt[NBINS] = {0, 0, 0, 0, 0};
    int64_t off[NBINS + 1] = {0, 0, 0, 0, 0, 0};
    int32_t *rows = nullptr;       // permutation of rows grouped by bin (nullptr: identity, single bin)
    bool identity = false;
    int identity_bin = 0;
    // hub chunks (bin 4)
    int64_t nchunks = 0;
    int64_t *chunk_row_first = nullptr;  // per hub row: first chunk index (nhub+1)
    double *chunk_partial = nullptr;     // per chunk partial sum
};

struct Level {
    int kind = KIND_COARSEST;
    int64_t n = 0, nnz = 0;
    int64_t *row_ptr = nullptr;
    int32_t *col = nullptr;
    double *w = nullptr;
    double *d = nullptr;
    double *dinv = nullptr;
    double maxw = 0.0;
    RowBins bins;
    // aggregation
    double lambda = 0.0;
    int64_t m = 0;
    int32_t *agg = nullptr;
    int64_t *mem_ptr = nullptr;   // aggregate -> members (m+1)
    int32_t *members = nullptr;   // n, ascending within each aggregate
    double *S = nullptr;          // optional (keep_strength)
    // Chebyshev constants (O-S6), host
    double cheb_theta = 0, cheb_delta = 0, cheb_sigma = 0;
    // elimination
    int64_t nF = 0;
    int32_t *fmap = nullptr;      // n
    int32_t *cid = nullptr;       // nC: fine id of coarse index
    int32_t *fid = nullptr;       // nF: fine id of F slot
    int64_t *ct_ptr = nullptr;    // nC+1: transposed L_FC (coarse -> F neighbours)
    int32_t *ct_f = nullptr;      // fine id of the F neighbour
    double *ct_coef = nullptr;    // w_fc / d_f
    // coarsest
    double *pinv = nullptr;       // n*n
    // solve work vectors (length n, n >= 1)
    double *b = nullptr, *x = nullptr, *x2 = nullptr, *t = nullptr, *r = nullptr, *dv = nullptr;
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
    lap_stats stats{};
    lap::Stats cur;
    int device = 0;
};

namespace lap {

// ---------------------------------------------------------------- kernels (host launchers)
// setup (setup.cu)
void build_hierarchy(lap_hierarchy *h, const lap_graph *g, cudaStream_t s);
void finalize_solve_structures(lap_hierarchy *h, cudaStream_t s);

// solve (solve.cu)
enum EpiKind { EPI_SPMV = 0, EPI_SPMV_DOT = 1, EPI_RESID = 2, EPI_CHEB = 3, EPI_LANCZOS = 4 };
struct EpiArgs {
    const double *x = nullptr;    // input vector (gathered)
    double *y = nullptr;          // output (SPMV / RESID r / CHEB x_out)
    const double *b = nullptr;    // rhs (RESID / CHEB)
    double *dv = nullptr;         // Chebyshev direction (in/out)
    const double *rs = nullptr;   // Lanczos: D^-1/2 (y_i = rs_i (L (rs o v))_i)
    double c1 = 0, c2 = 0;        // CHEB: dv = c1 dv + c2 D^-1 r
    double *partials = nullptr;   // SPMV_DOT partial sums (one per block per bin)
};
void spmv_level(lap_hierarchy *h, const Level &L, EpiKind kind, const EpiArgs &a, cudaStream_t s);
void build_row_bins(Level &L, cudaStream_t s);
int64_t spmv_partial_slots(const Level &L);
void vcycle(lap_hierarchy *h, int l, cudaStream_t s);   // x_l = V(l, b_l)
void run_pcg(lap_hierarchy *h, double tol, int32_t *iters, double *relres, int *conv, cudaStream_t s);

// small shared reductions (solve.cu)
void dot(lap_hierarchy *h, const double *a, const double *b, int64_t n, double *out, cudaStream_t s);
void reduce_partials(lap_hierarchy *h, const double *partials, int64_t np, double *out, cudaStream_t s);

inline unsigned grid_for(int64_t work, int threads, int64_t cap = 148 * 32) {
    int64_t g = (work + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

}  // namespace lap
