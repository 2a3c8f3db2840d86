// lap_api.cu -- the extern "C" boundary of liblap.so (include/lap.h) and the
// host-side sequencing of setup/solve.  No C++ exception crosses the ABI.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "lap_internal.cuh"
#include "canon.cuh"

namespace lap {
void vcycle_apply(lap_hierarchy *h, const double *r, double *z, cudaStream_t s);

static thread_local std::string g_err;
void set_error(const std::string &m) { g_err = m; }
static bool g_capturing = false;
bool g_capturing_flag(bool v) {
    g_capturing = v;
    return v;
}
bool debug_sync() {
    if (g_capturing) return false;
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("LAP_DEBUG_SYNC");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

int group_shift() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("LAP_GSHIFT");
        v = e ? std::max(0, std::min(5, atoi(e))) : 0;
    }
    return v;
}

bool pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("LAP_PDL");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

// liblap's own stream-ordered pool, one per device (never the device's default
// pool: memory a pool holds is invisible to other allocators of the process --
// PyTorch's caching allocator, NCCL -- so the library keeps its reservation in
// a pool of its own and trims it when the last hierarchy is freed).
static cudaMemPool_t g_pool[64];
static bool g_pool_ok[64];
static int g_live = 0;  // hierarchies alive (lap_setup .. lap_free)
static uint64_t g_retain = 0;  // bytes the pool keeps reserved when idle (lap_pool_retain)
cudaMemPool_t lib_pool() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) throw Error{LAP_ECUDA, "device ordinal out of range"};
    if (!g_pool_ok[dev]) {
        cudaMemPoolProps pr;
        std::memset(&pr, 0, sizeof(pr));
        pr.allocType = cudaMemAllocationTypePinned;
        pr.handleTypes = cudaMemHandleTypeNone;
        pr.location.type = cudaMemLocationTypeDevice;
        pr.location.id = dev;
        cudaError_t e = cudaMemPoolCreate(&g_pool[dev], &pr);
        if (e != cudaSuccess) throw Error{LAP_ECUDA, std::string("cudaMemPoolCreate: ") + cudaGetErrorString(e)};
        uint64_t thr = UINT64_MAX;  // keep freed memory reserved between setups (no re-mapping stalls)
        cudaMemPoolSetAttribute(g_pool[dev], cudaMemPoolAttrReleaseThreshold, &thr);
        g_pool_ok[dev] = true;
    }
    return g_pool[dev];
}
void live_add(int d) { g_live += d; }
// return the pool's reservation to the device once no hierarchy is alive
void pool_trim_if_idle() {
    if (g_live > 0) return;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && g_pool_ok[dev]) cudaMemPoolTrimTo(g_pool[dev], (size_t)g_retain);
}
void *dalloc(size_t bytes, cudaStream_t s) {
    cudaMemPool_t pool = lib_pool();
    void *p = nullptr;
    cudaError_t e = cudaMallocFromPoolAsync(&p, bytes ? bytes : 1, pool, s);
    if (e != cudaSuccess)
        throw Error{e == cudaErrorMemoryAllocation ? LAP_ENOMEM : LAP_ECUDA,
                    std::string("cudaMallocFromPoolAsync: ") + cudaGetErrorString(e)};
    static int poison = -1;  // LAP_POISON=1: fill new allocations with NaN bytes (tests)
    if (poison < 0) {
        const char *v = getenv("LAP_POISON");
        poison = (v && v[0] == '1') ? 1 : 0;
    }
    if (poison) cudaMemsetAsync(p, 0xFF, bytes ? bytes : 1, s);
    return p;
}
void dfree(void *p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

// ---------------------------------------------------------------- members CSR
__global__ void k_iota(int64_t n, int32_t *v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (int32_t)i;
}
__global__ void k_lower_bound_i32(int64_t m, int64_t n, const int32_t *keys, int64_t *ptr) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a <= m; a += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < a) lo = mid + 1;
            else hi = mid;
        }
        ptr[a] = lo;
    }
}
__global__ void k_scatter_perm(int64_t n, const int64_t *perm, const double *in, double *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[perm[i]] = in[i];
}
__global__ void k_gather_perm(int64_t n, const int64_t *perm, const double *in, double *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[perm[i]];
}
__global__ void k_sub_mean2(int64_t n, double *v, const double *sum) {
    double mean = *sum / (double)n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] -= mean;
}

__global__ void k_gather_i32map(int64_t n, const int32_t *map, const double *in, double *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[map[i]];
}
__global__ void k_scatter_i32map(int64_t n, const int32_t *map, const double *in, double *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[map[i]] = in[i];
}

void finalize_solve_structures(lap_hierarchy *h, cudaStream_t s) {
    for (size_t l = 0; l < h->lev.size(); l++) {
        Level &L = h->lev[l];
        int64_t n = L.n > 0 ? L.n : 1;
        L.b = (double *)dalloc(8 * n, s);
        L.x = (double *)dalloc(8 * n, s);
        L.x2 = (double *)dalloc(8 * n, s);
        L.t = (double *)dalloc(8 * n, s);
        L.r = (double *)dalloc(8 * n, s);
        L.dv = (double *)dalloc(8 * n, s);
        if (L.kind == KIND_AGG && l > 0) {  // K-cycle inner FCG vectors (small: coarse levels)
            L.kp = (double *)dalloc(8 * n, s);
            L.kq = (double *)dalloc(8 * n, s);
            L.kz = (double *)dalloc(8 * n, s);
            L.kr = (double *)dalloc(8 * n, s);
            L.ksc = (double *)dalloc(8 * 8, s);
        }
        if (L.kind == KIND_AGG) {
            double a = h->p.cheby_lo * L.lambda, b = h->p.cheby_hi * L.lambda;
            L.cheb_theta = 0.5 * (b + a);
            L.cheb_delta = 0.5 * (b - a);
            L.cheb_sigma = L.cheb_theta / L.cheb_delta;
        }
    }
    build_transfers(h, s);
    int64_t n0 = h->lev[0].n;
    double **vecs[] = {&h->pb, &h->px, &h->pr, &h->pz, &h->pp, &h->pq, &h->stage_in, &h->stage_out};
    for (double **v : vecs) *v = (double *)dalloc(8 * (n0 > 0 ? n0 : 1), s);
    h->scal = (double *)dalloc(8 * 16, s);
    LAP_CUDA(cudaMemsetAsync(h->scal, 0, 8 * 16, s));
    int64_t np = std::max<int64_t>(148 * 8, spmv_partial_slots(h->lev[0]));  // >= XR_BLOCKS (solve.cu)
    for (auto &L : h->lev) np = std::max<int64_t>(np, 2 * spmv_partial_slots(L));  // E_FCG: two dots
    np = std::max<int64_t>(np, 3 * spmv_partial_slots(h->lev[0]));                  // E_CHEBZ: three sums
    if (np > h->npartials) {
        dfree(h->partials, s);
        h->partials = (double *)dalloc(8 * np, s);
        h->npartials = np;
    }
    // pageable (not pinned): every read of it is followed by a stream sync, and a
    // cudaMallocHost / cudaFreeHost pair per hierarchy costs milliseconds
    h->host_scal = (double *)calloc(16, sizeof(double));
    if (!h->host_scal) throw Error{LAP_ENOMEM, "host scalars"};
}

static void free_level(Level &L, cudaStream_t s) {
    void *ps[] = {L.row_ptr, L.col, L.w, L.d, L.agg, L.S, L.fmap, L.cid, L.fid, L.ct_ptr, L.ct_f, L.ct_coef,
                  L.pinv, L.sid, L.spos, L.srp, L.scol, L.sw, L.sd, L.slice_ptr, L.ell_col, L.ell_w, L.chunk_row, L.chunk_idx, L.chunk_slot, L.chunk_cnt,
                  L.chunk_part, L.ell_col16, L.scol16, L.xt_rb, L.xt_seg, L.xt_wo, L.xt_rc, L.xt_w,
                  L.agg_s, L.mem_ptr, L.members, L.cid_s, L.flist, L.ct_ptr_s, L.ct_f_s, L.ct_coef_s, L.fmap_s,
                  L.ct_crow, L.ct_cidx, L.ct_cslot, L.ct_ccnt, L.ct_cpart,
                  L.pinv_s, L.dense, L.dense_part, L.dense_cnt, L.b, L.x, L.x2, L.t, L.r, L.dv, L.kp, L.kq, L.kz,
                  L.kr, L.ksc, L.mdot, L.mdone, L.rs_crow, L.rs_cidx, L.rs_cslot, L.rs_ccnt, L.rs_cpart};
    for (void *p : ps) dfree(p, s);
}

// V-cycle launch (graph when captured)
struct VcCounts {
    int64_t launches = 0, edges = 0, bytes = 0;
};
static std::vector<std::pair<lap_hierarchy *, VcCounts>> g_vc;  // per-hierarchy V-cycle counts (captured graph)
static VcCounts &vc_of(lap_hierarchy *h) {
    for (auto &e : g_vc)
        if (e.first == h) return e.second;
    g_vc.push_back({h, VcCounts{}});
    return g_vc.back().second;
}
static void vc_forget(lap_hierarchy *h) {
    for (size_t i = 0; i < g_vc.size(); i++)
        if (g_vc[i].first == h) {
            g_vc.erase(g_vc.begin() + i);
            return;
        }
}

void launch_vcycle(lap_hierarchy *h, cudaStream_t s) {
    if (h->vgraph) {
        LAP_CUDA(cudaGraphLaunch(h->vgraph, s));
        VcCounts &c = vc_of(h);
        h->cur.launches += c.launches;
        h->cur.edges += c.edges;
        h->cur.bytes += c.bytes;
    } else {
        vcycle_apply(h, h->pr, h->pz, s);
    }
}

static void capture_vcycle(lap_hierarchy *h) {
    cudaStream_t cs;
    LAP_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    Stats save = h->cur;
    h->cur = Stats{};
    cudaGraph_t g;
    LAP_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    g_capturing = true;
    try {
        vcycle_apply(h, h->pr, h->pz, cs);
        g_capturing = false;
    } catch (...) {
        g_capturing = false;
        cudaStreamEndCapture(cs, &g);
        cudaStreamDestroy(cs);
        throw;
    }
    LAP_CUDA(cudaStreamEndCapture(cs, &g));
    LAP_CUDA(cudaGraphInstantiate(&h->vgraph, g, 0));
    LAP_CUDA(cudaGraphDestroy(g));
    LAP_CUDA(cudaStreamDestroy(cs));
    VcCounts &c = vc_of(h);
    c.launches = h->cur.launches;
    c.edges = h->cur.edges;
    c.bytes = h->cur.bytes;
    h->cur = save;
}

// Stream-ordered pool warm-up: the pool's physical memory only grows when a
// request does not fit its free chunks, and growing it (mapping GBs) stalls a
// setup by 30-500 ms at cfg 4 sizes.  Before each setup, make sure the pool
// holds one chunk twice as large as the biggest setup peak seen so far in this
// process: allocate it once and free it back to the pool.
static size_t g_peak = 0;
// device memory total (cached) minus what liblap's pool has in use: a free-memory
// estimate for batch sizing that avoids cudaMemGetInfo on the setup path (that
// call measured 0.5-29 ms, at random -- the source of the setup-time outliers)
size_t device_free_estimate() {
    static size_t total = 0;
    if (!total) {
        size_t fr = 0;
        if (cudaMemGetInfo(&fr, &total) != cudaSuccess) total = (size_t)80 << 30;
    }
    uint64_t used = 0;
    cudaMemPoolGetAttribute(lib_pool(), cudaMemPoolAttrUsedMemCurrent, &used);
    return total > used ? total - (size_t)used : 0;
}
void pool_warm(cudaStream_t s) {
    cudaMemPool_t pool = lib_pool();
    uint64_t zero = 0, reserved = 0, used = 0;
    if (g_peak) {
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
        size_t want = 2 * g_peak;  // headroom against fragmentation (1.1x still grew now and then)
        size_t fr = 0, tot = 0;
        // (cudaMemGetInfo only when the pool must grow: it is slow at random)
        if (reserved < used + want && cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
            // never reserve beyond what the device has free (leave 5% for other allocators)
            const size_t cap = (size_t)((double)(fr + (reserved - used)) * 0.95);
            want = std::min(want, cap);
        }
        if (want > 0 && reserved < used + want) {
            void *p = nullptr;
            if (cudaMallocFromPoolAsync(&p, want, pool, s) == cudaSuccess) cudaFreeAsync(p, s);
            else cudaGetLastError();
        }
    }
    // the setup's own high-water mark (not the warm-up block's): reset after the warm-up
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &zero);
}
void pool_note_peak() {
    cudaMemPool_t pool = lib_pool();
    uint64_t hi = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &hi);
    if (hi > g_peak) g_peak = hi;
    if (getenv("LAP_SETUP_TRACE") || getenv("LAP_POOL_TRACE")) {
        uint64_t reserved = 0;
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
        fprintf(stderr, "[lap setup] pool: peak used %.2f GB, reserved %.2f GB\n", hi / 1e9, reserved / 1e9);
    }
}

static bool is_device_ptr(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace lap

// =========================================================================
// extern "C"
// =========================================================================

#define LAP_API_BEGIN try {
#define LAP_API_END                                 \
    }                                               \
    catch (const lap::Error &e) {                   \
        lap::set_error(e.msg);                      \
        return e.code;                              \
    }                                               \
    catch (const std::exception &e) {               \
        lap::set_error(e.what());                   \
        return LAP_ECUDA;                           \
    }                                               \
    catch (...) {                                   \
        lap::set_error("unknown error");            \
        return LAP_ECUDA;                           \
    }

extern "C" {

void lap_params_default(lap_params *p) {
    std::memset(p, 0, sizeof(*p));
    p->tol = 1e-8;
    p->max_iters = 500;
    p->cheby_degree = 2;
    p->cheby_lo = 0.3;
    p->cheby_hi = 1.1;
    p->lanczos_steps = 10;
    p->elim_max_degree = 4;
    p->elim_enable = 1;
    p->n_test_vectors = 4;
    p->tv_sweeps = 3;
    p->tv_omega = 2.0 / 3.0;
    p->vote_rounds = 10;
    p->vote_threshold = 8;
    p->coarse_nnz = 1000;
    p->max_levels = 40;
    p->seed = 0;
    p->random_order = 1;
    p->affinity_power = 1;
    p->keep_strength = 0;
    p->cycle = 0;
    p->kcycle_inner = 2;
    p->use_graphs = 1;
    p->replicate_nnz = 0;
    p->elim_rounds = 1;
    p->keep_logical = -1;
}

const char *lap_last_error(void) { return lap::g_err.c_str(); }

lap_status lap_random_stream(int32_t which, uint64_t seed, int32_t level, int32_t attempt, int64_t n, void *out,
                             void *stream) {
    if (which < 0 || which > 3 || n < 0 || level < 0 || attempt < 0 || (n > 0 && !out)) {
        lap::set_error("lap_random_stream: invalid arguments");
        return LAP_EINVAL;
    }
    LAP_API_BEGIN
    if (n > 0) lap::random_stream(which, seed, level, attempt, n, out, (cudaStream_t)stream);
    return LAP_OK;
    LAP_API_END
}

void lap_pool_retain(uint64_t bytes) {
    lap::g_retain = bytes;
    lap::pool_trim_if_idle();
}
const char *lap_version(void) { return "liblap 0.1 (sm_100a)"; }

static lap_status setup_common(const lap_graph *g, const char *dir, const lap_params *pp, void *stream,
                               lap_hierarchy **out);

lap_status lap_setup(const lap_graph *g, const lap_params *pp, void *stream, lap_hierarchy **out) {
    if (out) *out = nullptr;
    if (!g || !out || g->n < 1 || !g->row_ptr || (g->row_ptr && !g->col && g->n > 1)) {
        lap::set_error("lap_setup: invalid arguments");
        return LAP_EINVAL;
    }
    return setup_common(g, nullptr, pp, stream, out);
}

lap_status lap_import_hierarchy(const char *dir, const lap_params *pp, void *stream, lap_hierarchy **out) {
    if (out) *out = nullptr;
    if (!dir || !out) {
        lap::set_error("lap_import_hierarchy: invalid arguments");
        return LAP_EINVAL;
    }
    return setup_common(nullptr, dir, pp, stream, out);
}

static lap_status setup_common(const lap_graph *g, const char *dir, const lap_params *pp, void *stream,
                               lap_hierarchy **out) {
    lap_params p;
    if (pp) p = *pp;
    else lap_params_default(&p);
    if (p.n_test_vectors != 4 || p.cheby_degree < 1 || p.tv_sweeps < 0 || p.vote_rounds < 0 ||
        p.lanczos_steps < 1 || p.lanczos_steps > 64 || !(p.cheby_hi > p.cheby_lo) || !(p.cheby_lo > 0) ||
        p.max_levels < 1 || p.cycle < 0 || p.cycle > 1 || p.kcycle_inner < 1 || p.kcycle_inner > 8 ||
        p.elim_rounds < 1 || p.elim_rounds > 64 || p.keep_logical < -1 || p.keep_logical > 1) {
        lap::set_error("lap_setup: unsupported parameter values");
        return LAP_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    lap_hierarchy *h = new lap_hierarchy();
    lap::live_add(1);
    h->p = p;
    cudaGetDevice(&h->device);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    try {
        LAP_CUDA(cudaEventCreate(&e0));
        LAP_CUDA(cudaEventCreate(&e1));
        lap::pool_warm(s);
        LAP_CUDA(cudaEventRecord(e0, s));
        h->cur = lap::Stats{};
        int64_t kl0 = lap::g_kl;
        h->npartials = 1024;  // reduction scratch used during setup (Lanczos dots)
        h->partials = (double *)lap::dalloc(8 * h->npartials, s);
        if (g) lap::build_hierarchy(h, g, s);
        else lap::import_hierarchy(h, dir, s);
        lap::finalize_solve_structures(h, s);
        lap::build_dense_tail(h, s);
        lap::build_ktail(h, s);
        LAP_CUDA(cudaEventRecord(e1, s));
        LAP_CUDA(cudaStreamSynchronize(s));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        h->stats.setup_ms = ms;
        h->stats.kernel_launches = h->cur.launches + (lap::g_kl - kl0);
        h->stats.spmv_edges = h->cur.edges;
        h->stats.spmv_bytes = h->cur.bytes;
        lap::pool_note_peak();
        if (p.use_graphs) {
            lap::capture_vcycle(h);
            lap::capture_pcg(h);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    } catch (const lap::Error &e) {
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        lap::set_error(e.msg);
        cudaStreamSynchronize(s);
        lap_free(h);
        cudaGetLastError();
        return e.code;
    } catch (...) {
        lap::set_error("lap_setup: unexpected exception");
        lap_free(h);
        return LAP_ECUDA;
    }
    *out = h;
    return h->status;
}

lap_status lap_setup_dist(const lap_graph *g, const lap_params *pp, lap_comm *c, void *stream, lap_hierarchy **out) {
    if (out) *out = nullptr;
    if (!c) {
        lap::set_error("lap_setup_dist: NULL communicator");
        return LAP_EINVAL;
    }
    lap_params p;
    if (pp) p = *pp;
    else lap_params_default(&p);
    const int want_graphs = p.use_graphs;
    p.use_graphs = 0;  // no single-GPU solve graphs: the sharded solve captures its own (dist.cu)
    if (p.cycle != 0) {
        lap::set_error("lap_setup_dist: the K-cycle (params.cycle = 1) is single-GPU only");
        return LAP_EINVAL;
    }
    lap_hierarchy *h = nullptr;
    lap_status st;
    {
        lap::SetupCommScope scope(c);  // the coarse-operator term builds split over the ranks
        st = lap_setup(g, &p, stream, &h);
    }
    if (st != LAP_OK && st != LAP_ESTALL) return st;
    try {
        if (h->lev[0].kind != lap::KIND_COARSEST) lap::build_dist(h, c, (cudaStream_t)stream, want_graphs != 0);
    } catch (const lap::Error &e) {
        lap::set_error(e.msg);
        lap_free(h);
        return e.code;
    } catch (...) {
        lap::set_error("lap_setup_dist: unexpected exception");
        lap_free(h);
        return LAP_ECUDA;
    }
    *out = h;
    return st;
}

void lap_free(lap_hierarchy *h) {
    if (!h) return;
    cudaStream_t s = nullptr;
    cudaDeviceSynchronize();
    if (h->vgraph) cudaGraphExecDestroy(h->vgraph);
    lap::free_dist(h);
    lap::free_pcg(h);
    lap::free_ktail(h, s);
    lap::free_block(h);
    for (auto &L : h->lev) lap::free_level(L, s);
    void *ps[] = {h->perm, h->cmap, h->pb, h->px, h->pr, h->pz, h->pp, h->pq, h->scal, h->partials, h->stage_in,
                  h->stage_out};
    for (void *p : ps) lap::dfree(p, s);
    free(h->host_scal);
    cudaStreamSynchronize(s);
    lap::vc_forget(h);
    delete h;
    lap::live_add(-1);
    lap::pool_trim_if_idle();
}

lap_status lap_solve(lap_hierarchy *h, const double *b, double *x, double tol, int32_t *iters, double *rel_residual,
                     void *stream) {
    if (!h || !b || !x) {
        lap::set_error("lap_solve: invalid arguments");
        return LAP_EINVAL;
    }
    LAP_API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    int64_t n = h->n0;
    if (tol <= 0) tol = h->p.tol;
    cudaEvent_t e0, e1;
    LAP_CUDA(cudaEventCreate(&e0));
    LAP_CUDA(cudaEventCreate(&e1));
    h->cur = lap::Stats{};
    LAP_CUDA(cudaEventRecord(e0, s));
    const double *bd = b;
    if (!lap::is_device_ptr(b)) {
        LAP_CUDA(cudaMemcpyAsync(h->stage_in, b, 8 * n, cudaMemcpyHostToDevice, s));
        bd = h->stage_in;
    }
    unsigned g = lap::grid_for(n, 256, 148 * 8);
    lap::k_scatter_perm<<<g, 256, 0, s>>>(n, h->cmap, bd, h->pb);            // b' = Pi b (storage order)
    lap::dot(h, h->pb, nullptr, n, h->scal + 7, s);
    lap::k_sub_mean2<<<g, 256, 0, s>>>(n, h->pb, h->scal + 7);               // project out 1
    h->cur.launches += 2;
    LAP_CHECK_LAUNCH();
    int32_t it = 0;
    double rr = 0;
    int conv = 0;
    if (h->dist) lap::dist_run_pcg(h, tol, &it, &rr, &conv, s);
    else lap::run_pcg(h, tol, &it, &rr, &conv, s);
    bool xdev = lap::is_device_ptr(x);
    double *xd = xdev ? x : h->stage_out;
    lap::k_gather_perm<<<g, 256, 0, s>>>(n, h->cmap, h->px, xd);             // x = Pi^T x'
    h->cur.launches++;
    LAP_CHECK_LAUNCH();
    if (!xdev) LAP_CUDA(cudaMemcpyAsync(x, xd, 8 * n, cudaMemcpyDeviceToHost, s));
    LAP_CUDA(cudaEventRecord(e1, s));
    LAP_CUDA(cudaStreamSynchronize(s));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    h->stats.solve_ms = ms;
    h->stats.kernel_launches = h->cur.launches;
    h->stats.spmv_edges = h->cur.edges;
    h->stats.spmv_bytes = h->cur.bytes;
    if (iters) *iters = it;
    if (rel_residual) *rel_residual = rr;
    return conv ? LAP_OK : LAP_ENOCONV;
    LAP_API_END
}

lap_status lap_solve_block(lap_hierarchy *h, int32_t k, const double *B, double *X, double tol, int32_t *iters,
                           double *rel_residual, void *stream) {
    if (!h || !B || !X || !iters || !rel_residual || k < 1 || k > 32 || h->dist) {
        lap::set_error("lap_solve_block: invalid arguments (1 <= k <= 32, single-GPU hierarchy)");
        return LAP_EINVAL;
    }
    LAP_API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = h->n0;
    cudaEvent_t e0, e1;
    LAP_CUDA(cudaEventCreate(&e0));
    LAP_CUDA(cudaEventCreate(&e1));
    h->cur = lap::Stats{};
    const bool bdev = lap::is_device_ptr(B), xdev = lap::is_device_ptr(X);
    lap::DBuf<double> bin, xout;
    if (!bdev) bin.alloc(n * k, s);
    if (!xdev) xout.alloc(n * k, s);
    LAP_CUDA(cudaEventRecord(e0, s));
    if (!bdev) LAP_CUDA(cudaMemcpyAsync(bin.p, B, 8 * (size_t)(n * k), cudaMemcpyHostToDevice, s));
    int conv = 0;
    lap::solve_block(h, k, bdev ? B : bin.p, xdev ? X : xout.p, tol > 0 ? tol : h->p.tol, iters, rel_residual, &conv,
                     s);
    if (!xdev) LAP_CUDA(cudaMemcpyAsync(X, xout.p, 8 * (size_t)(n * k), cudaMemcpyDeviceToHost, s));
    LAP_CUDA(cudaEventRecord(e1, s));
    LAP_CUDA(cudaStreamSynchronize(s));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    h->stats.solve_ms = ms;
    h->stats.kernel_launches = h->cur.launches;
    h->stats.spmv_edges = h->cur.edges;
    h->stats.spmv_bytes = h->cur.bytes;
    return conv ? LAP_OK : LAP_ENOCONV;
    LAP_API_END
}

lap_status lap_num_levels(const lap_hierarchy *h, int32_t *nlev) {
    if (!h || !nlev) return LAP_EINVAL;
    *nlev = (int32_t)h->lev.size();
    return LAP_OK;
}

lap_status lap_level_info(const lap_hierarchy *h, int32_t l, int32_t *kind, int64_t *n, int64_t *nnz,
                          double *lambda_hat) {
    if (!h || l < 0 || l >= (int32_t)h->lev.size()) return LAP_EINVAL;
    const lap::Level &L = h->lev[l];
    if (kind) *kind = L.kind;
    if (n) *n = L.n;
    if (nnz) *nnz = L.nnz;
    if (lambda_hat) *lambda_hat = L.lambda;
    return LAP_OK;
}

lap_status lap_level_export(const lap_hierarchy *h, int32_t l, int64_t *row_ptr, int32_t *col, double *w, double *d,
                            int32_t *map) {
    if (!h || l < 0 || l >= (int32_t)h->lev.size()) return LAP_EINVAL;
    LAP_API_BEGIN
    const lap::Level &L = h->lev[l];
    if (L.logical_released && (row_ptr || col || w)) {
        lap::set_error("lap_level_export: the logical CSR of this level was released (params.keep_logical); "
                       "use lap_level_rows");
        return LAP_EINVAL;
    }
    if (row_ptr) LAP_CUDA(cudaMemcpy(row_ptr, L.row_ptr, 8 * (L.n + 1), cudaMemcpyDeviceToHost));
    if ((col || w) && L.nnz) {
        const int32_t *cs = L.col;
        const double *ws = L.w;
        lap::DBuf<int32_t> c2;
        lap::DBuf<double> w2;
        if (!L.cols_sorted) {  // the logical CSR as the method defines it: each row in ascending column order
            c2.alloc(L.nnz, nullptr);
            w2.alloc(L.nnz, nullptr);
            lap::sort_rows(L.n, L.row_ptr, L.nnz, lap::bitlen_u64((uint64_t)(L.n > 0 ? L.n : 1)), L.col, L.w, c2.p,
                           w2.p, nullptr);
            LAP_CUDA(cudaStreamSynchronize(nullptr));
            cs = c2.p;
            ws = w2.p;
        }
        if (col) LAP_CUDA(cudaMemcpy(col, cs, 4 * L.nnz, cudaMemcpyDeviceToHost));
        if (w) LAP_CUDA(cudaMemcpy(w, ws, 8 * L.nnz, cudaMemcpyDeviceToHost));
    }
    if (d) LAP_CUDA(cudaMemcpy(d, L.d, 8 * L.n, cudaMemcpyDeviceToHost));
    if (map) {
        if (L.kind == lap::KIND_AGG) LAP_CUDA(cudaMemcpy(map, L.agg, 4 * L.n, cudaMemcpyDeviceToHost));
        else if (L.kind == lap::KIND_ELIM) LAP_CUDA(cudaMemcpy(map, L.fmap, 4 * L.n, cudaMemcpyDeviceToHost));
    }
    return LAP_OK;
    LAP_API_END
}

lap_status lap_level_rows(const lap_hierarchy *h, int32_t l, int64_t k, const int64_t *rows, int64_t *row_ptr,
                          int32_t *col, double *w) {
    if (!h || l < 0 || l >= (int32_t)h->lev.size() || k < 0 || (k > 0 && !rows) || !row_ptr) return LAP_EINVAL;
    LAP_API_BEGIN
    const lap::Level &L = h->lev[l];
    std::vector<int32_t> spos(L.n), sid(L.n);
    std::vector<int64_t> srp(L.n + 1);
    LAP_CUDA(cudaMemcpy(spos.data(), L.spos, 4 * L.n, cudaMemcpyDeviceToHost));
    LAP_CUDA(cudaMemcpy(srp.data(), L.srp, 8 * (L.n + 1), cudaMemcpyDeviceToHost));
    row_ptr[0] = 0;
    for (int64_t t = 0; t < k; t++) {
        if (rows[t] < 0 || rows[t] >= L.n) throw lap::Error{LAP_EINVAL, "lap_level_rows: row out of range"};
        const int64_t p = spos[rows[t]];
        row_ptr[t + 1] = row_ptr[t] + (srp[p + 1] - srp[p]);
    }
    if (!col) return LAP_OK;
    LAP_CUDA(cudaMemcpy(sid.data(), L.sid, 4 * L.n, cudaMemcpyDeviceToHost));
    std::vector<std::pair<int32_t, double>> row;
    for (int64_t t = 0; t < k; t++) {
        const int64_t p = spos[rows[t]], a = srp[p], len = srp[p + 1] - a;
        std::vector<int32_t> c(len);
        std::vector<double> v(len);
        if (len) {
            LAP_CUDA(cudaMemcpy(c.data(), L.scol + a, 4 * len, cudaMemcpyDeviceToHost));
            LAP_CUDA(cudaMemcpy(v.data(), L.sw + a, 8 * len, cudaMemcpyDeviceToHost));
        }
        row.resize(len);
        for (int64_t q = 0; q < len; q++) row[q] = {sid[c[q]], v[q]};  // storage column -> logical id
        std::sort(row.begin(), row.end(), [](const std::pair<int32_t, double> &x, const std::pair<int32_t, double> &y) {
            return x.first < y.first;
        });
        for (int64_t q = 0; q < len; q++) {
            col[row_ptr[t] + q] = row[q].first;
            if (w) w[row_ptr[t] + q] = row[q].second;
        }
    }
    return LAP_OK;
    LAP_API_END
}

lap_status lap_level_strength(const lap_hierarchy *h, int32_t l, double *S) {
    if (!h || l < 0 || l >= (int32_t)h->lev.size() || !S) return LAP_EINVAL;
    const lap::Level &L = h->lev[l];
    if (!L.S) {
        lap::set_error("strength not retained (set keep_strength)");
        return LAP_EINVAL;
    }
    LAP_API_BEGIN
    if (L.nnz && !L.cols_sorted && L.col) {  // S in the logical entry order of sorted rows (as exported)
        lap::DBuf<int32_t> c2(L.nnz, nullptr);
        lap::DBuf<double> s2(L.nnz, nullptr);
        lap::sort_rows(L.n, L.row_ptr, L.nnz, lap::bitlen_u64((uint64_t)(L.n > 0 ? L.n : 1)), L.col, L.S, c2.p, s2.p,
                       nullptr);
        LAP_CUDA(cudaMemcpy(S, s2.p, 8 * L.nnz, cudaMemcpyDeviceToHost));
    } else if (L.nnz) {
        LAP_CUDA(cudaMemcpy(S, L.S, 8 * L.nnz, cudaMemcpyDeviceToHost));
    }
    return LAP_OK;
    LAP_API_END
}

lap_status lap_coarse_pinv(const lap_hierarchy *h, double *pinv) {
    if (!h || !pinv) return LAP_EINVAL;
    LAP_API_BEGIN
    const lap::Level &L = h->lev.back();
    LAP_CUDA(cudaMemcpy(pinv, L.pinv, 8 * L.n * L.n, cudaMemcpyDeviceToHost));
    return LAP_OK;
    LAP_API_END
}

lap_status lap_perm(const lap_hierarchy *h, int64_t *perm) {
    if (!h || !perm) return LAP_EINVAL;
    LAP_API_BEGIN
    LAP_CUDA(cudaMemcpy(perm, h->perm, 8 * h->n0, cudaMemcpyDeviceToHost));
    return LAP_OK;
    LAP_API_END
}

lap_status lap_spmv(const lap_hierarchy *hc, int32_t l, const double *x, double *y, void *stream) {
    lap_hierarchy *h = const_cast<lap_hierarchy *>(hc);
    if (!h || l < 0 || l >= (int32_t)h->lev.size() || !x || !y) return LAP_EINVAL;
    LAP_API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    const lap::Level &L = h->lev[l];
    int64_t n = L.n;
    lap::DBuf<double> xin, yout;
    const double *xd = x;
    double *yd = y;
    bool xdev = lap::is_device_ptr(x), ydev = lap::is_device_ptr(y);
    if (!xdev) {
        xin.alloc(n, s);
        LAP_CUDA(cudaMemcpyAsync(xin.p, x, 8 * n, cudaMemcpyHostToDevice, s));
        xd = xin.p;
    }
    if (!ydev) {
        yout.alloc(n, s);
        yd = yout.p;
    }
    lap::DBuf<double> xs(n, s), ys(n, s);  // logical <-> storage order
    unsigned g = lap::grid_for(n, 256, 148 * 8);
    lap::k_gather_i32map<<<g, 256, 0, s>>>(n, L.sid, xd, xs.p);
    lap::EpiArgs a;
    a.x = xs.p;
    a.y = ys.p;
    lap::spmv_level(h, L, lap::EPI_SPMV, a, s);
    lap::k_scatter_i32map<<<g, 256, 0, s>>>(n, L.sid, ys.p, yd);
    LAP_CHECK_LAUNCH();
    if (!ydev) LAP_CUDA(cudaMemcpyAsync(y, yd, 8 * n, cudaMemcpyDeviceToHost, s));
    LAP_CUDA(cudaStreamSynchronize(s));
    return LAP_OK;
    LAP_API_END
}

lap_status lap_vcycle(lap_hierarchy *h, const double *r, double *z, void *stream) {
    if (!h || !r || !z) return LAP_EINVAL;
    LAP_API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    int64_t n = h->lev[0].n;
    bool rdev = lap::is_device_ptr(r), zdev = lap::is_device_ptr(z);
    const lap::Level &L0 = h->lev[0];
    unsigned g = lap::grid_for(n, 256, 148 * 8);
    LAP_CUDA(cudaMemcpyAsync(h->stage_in, r, 8 * n, rdev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    lap::k_gather_i32map<<<g, 256, 0, s>>>(n, L0.sid, h->stage_in, h->pr);      // logical -> storage
    lap::launch_vcycle(h, s);
    lap::k_scatter_i32map<<<g, 256, 0, s>>>(n, L0.sid, h->pz, h->stage_out);    // storage -> logical
    LAP_CHECK_LAUNCH();
    LAP_CUDA(cudaMemcpyAsync(z, h->stage_out, 8 * n, zdev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    LAP_CUDA(cudaStreamSynchronize(s));
    return LAP_OK;
    LAP_API_END
}

lap_status lap_kcycle(lap_hierarchy *h, int32_t l, int32_t with_fcg, const double *r, double *z, void *stream) {
    if (!h || !r || !z || l < 0 || l >= (int32_t)h->lev.size() || h->dist) return LAP_EINVAL;
    if (with_fcg && l == 0 && h->lev[0].kind == lap::KIND_AGG) return LAP_EINVAL;  // level 0: the outer FCG
    LAP_API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    lap::Level &L = h->lev[l];
    int64_t n = L.n;
    bool rdev = lap::is_device_ptr(r), zdev = lap::is_device_ptr(z);
    unsigned g = lap::grid_for(n, 256, 148 * 8);
    LAP_CUDA(cudaMemcpyAsync(h->stage_in, r, 8 * n, rdev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    lap::k_gather_i32map<<<g, 256, 0, s>>>(n, L.sid, h->stage_in, L.b);       // logical -> storage
    lap::kcycle_level(h, l, with_fcg != 0, s);
    lap::k_scatter_i32map<<<g, 256, 0, s>>>(n, L.sid, L.x, h->stage_out);     // storage -> logical
    LAP_CHECK_LAUNCH();
    LAP_CUDA(cudaMemcpyAsync(z, h->stage_out, 8 * n, zdev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    LAP_CUDA(cudaStreamSynchronize(s));
    return LAP_OK;
    LAP_API_END
}

lap_status lap_get_stats(const lap_hierarchy *h, lap_stats *st) {
    if (!h || !st) return LAP_EINVAL;
    *st = h->stats;
    return LAP_OK;
}

lap_status lap_bench_op(lap_hierarchy *h, int32_t which, int32_t l, int32_t reps, void *stream, double *ms,
                        double *bytes, int64_t *edges) {
    if (!h || reps < 1 || which < 0 || which > 2) return LAP_EINVAL;
    if (which < 2 && (l < 0 || l >= (int32_t)h->lev.size() || h->lev[l].kind == lap::KIND_COARSEST)) return LAP_EINVAL;
    if (which == 1 && h->lev[l].kind != lap::KIND_AGG) return LAP_EINVAL;
    LAP_API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<cudaEvent_t> ev(reps + 1);
    for (auto &e : ev) LAP_CUDA(cudaEventCreate(&e));
    lap::Stats save = h->cur;
    h->cur = lap::Stats{};
    double by = 0;
    int64_t ed = 0;
    auto run = [&](bool count) {
        if (which == 2) {
            lap::launch_vcycle(h, s);
        } else {
            lap::Level &L = h->lev[l];
            lap::EpiArgs a;
            a.x = L.x2;
            a.y = L.t;
            a.b = L.b;
            a.dv = L.dv;
            a.c1 = 0.5;
            a.c2 = 0.5;
            lap::spmv_level(h, L, which == 0 ? lap::EPI_SPMV : lap::EPI_CHEB, a, s);
        }
        if (count) {
            by = (double)h->cur.bytes;
            ed = h->cur.edges;
        }
        h->cur = lap::Stats{};
    };
    if (which < 2) {
        lap::Level &L = h->lev[l];
        double *vs[] = {L.x2, L.t, L.b, L.dv};
        for (double *v : vs) LAP_CUDA(cudaMemsetAsync(v, 0, 8 * (L.n > 0 ? L.n : 1), s));
    } else {
        LAP_CUDA(cudaMemsetAsync(h->pr, 0, 8 * h->lev[0].n, s));
    }
    for (int i = 0; i < 3; i++) run(i == 0);  // warm-up
    if (which == 2) {
        // one graph launch per V-cycle, an event between consecutive launches
        for (int i = 0; i < reps; i++) {
            LAP_CUDA(cudaEventRecord(ev[i], s));
            run(false);
        }
        LAP_CUDA(cudaEventRecord(ev[reps], s));
        LAP_CUDA(cudaEventSynchronize(ev[reps]));
        for (int i = 0; i < reps; i++) {
            float t = 0;
            cudaEventElapsedTime(&t, ev[i], ev[i + 1]);
            if (ms) ms[i] = t;
        }
    } else {
        // single kernels are too short to time one by one from the host (the
        // host-side launch rate would be measured): capture the `reps`
        // launches into one graph, as the solve runs them, and time 5 graph
        // launches; every entry of ms[] is the mean per launch of one of them
        cudaStream_t cs;
        LAP_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        cudaGraph_t g;
        lap::g_capturing_flag(true);
        LAP_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        cudaStream_t keep = s;
        s = cs;
        for (int i = 0; i < reps; i++) run(false);
        s = keep;
        LAP_CUDA(cudaStreamEndCapture(cs, &g));
        lap::g_capturing_flag(false);
        cudaGraphExec_t ge;
        LAP_CUDA(cudaGraphInstantiate(&ge, g, 0));
        LAP_CUDA(cudaGraphDestroy(g));
        LAP_CUDA(cudaStreamDestroy(cs));
        LAP_CUDA(cudaGraphLaunch(ge, s));  // warm
        int nt = reps < 5 ? reps : 5;
        for (int i = 0; i < nt; i++) {
            LAP_CUDA(cudaEventRecord(ev[i], s));
            LAP_CUDA(cudaGraphLaunch(ge, s));
        }
        LAP_CUDA(cudaEventRecord(ev[nt], s));
        LAP_CUDA(cudaEventSynchronize(ev[nt]));
        for (int i = 0; i < reps; i++) {
            float t = 0;
            cudaEventElapsedTime(&t, ev[i % nt], ev[i % nt + 1]);
            if (ms) ms[i] = t / reps;
        }
        cudaGraphExecDestroy(ge);
    }
    for (auto &e : ev) cudaEventDestroy(e);
    h->cur = save;
    if (which == 1) by = 12.0 * h->lev[l].nnz + 56.0 * h->lev[l].n;  // SURVEY M3, H2 with SpMV
    if (bytes) *bytes = by;
    if (edges) *edges = ed;
    return LAP_OK;
    LAP_API_END
}

}  // extern "C"
