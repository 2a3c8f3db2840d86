// ktail.cu -- the K-cycle below a small level as ONE single-CTA kernel (N2).
//
// The K-cycle (oracle orc_kcycle / orc_kcoarse) visits level l
// 2^(number of aggregation levels above it) times per outer iteration, and
// each visit of a small level is ~10 dependent steps of a few hundred rows:
// launched one kernel per step (solve.cu kcoarse / cycle_rec) every step
// costs ~5 us of launch + dependent-load latency while doing ~0.1 us of work
// (cfg 2: ~80% of the K-cycle's 700 launches per iteration are on levels of
// <= 1865 rows).  Below the first level t whose sub-hierarchy is small
// (n_l <= KT_MAX_N and nnz_l <= KT_MAX_NNZ for every l >= t), the whole
// coarse problem kcoarse(t) runs inside one CTA of 1024 threads: the host
// walks the same recursion as solve.cu once per hierarchy and records it as a
// program of ops (same operands, same Chebyshev coefficients, same FCG
// recurrence); the kernel executes the ops in order with a __syncthreads()
// between them, keeping the FCG scalars in shared memory.  Vectors stay in
// global memory (L2-resident at these sizes).
//
// It is not a grid-wide persistent kernel: a grid barrier costs more than a
// kernel boundary inside a CUDA graph (measured), while a CTA
// barrier costs tens of nanoseconds; one SM is enough for levels this small.
//
// Arithmetic per op is the launched kernels' (solve.cu): row sums in CSR
// order (a warp per row for rows longer than SHORT_MAX, lane-strided with a
// shuffle tree), the same epilogue formulas, FCG guards p.q = 0 -> 0.  Dot
// products are single-CTA fixed-order reductions: deterministic, and within
// rounding of the launched path and of the oracle (tests/test_gpu_kcycle.py).
#include "lap_internal.cuh"

#include <vector>

namespace lap {

constexpr int64_t KT_MAX_N = 4096;
constexpr int64_t KT_MAX_NNZ = 131072;
constexpr int KT_THREADS = 1024;

enum KOpCode : int32_t {
    KO_CHEB_FIRST = 0,  // x = dv = (b / d) * c1
    KO_SPMV = 1,        // y = epilogue(L x), epi in {CHEB, CHEB0, RESID, FCG}
    KO_RESTRICT = 2,    // bc[a] = sum_{members} r ; optional coarse step 0
    KO_PROLONG = 3,     // x[i] += xc[agg[i]]
    KO_ERESTRICT = 4,   // bc[k] = b[cid[k]] + sum ctc * b[ctf] ; optional coarse step 0
    KO_EPROLONG = 5,    // x[cid[k]] = xc[k] ; x[f] = (b_f + sum w xc[fmap]) / d_f
    KO_COARSE = 6,      // x = P b  (n x n row-major)
    KO_DOT = 7,         // slot = a . b
    KO_FCG_DIR = 8,     // beta = slot(pq) != 0 ? -slot(zq)/slot(pq) : 0 ; p = z + beta p
    KO_FCG_UPDATE = 9,  // alpha = slot(pq) != 0 ? slot(pr)/slot(pq) : 0 ; x (=|+=) alpha p ; r = rin - alpha q
};
enum KEpi : int32_t { KE_CHEB = 0, KE_CHEB0 = 1, KE_RESID = 2, KE_FCG = 3 };

struct __align__(16) KOp {
    int32_t code = 0, epi = 0, first = 0, s0 = 0, s1 = 0, s2 = 0;
    int64_t n = 0, n2 = 0;
    const int64_t *rp = nullptr;  // CSR row pointer / member pointer / ct_ptr
    const int32_t *i0 = nullptr;  // CSR columns / members / agg / cid
    const int32_t *i1 = nullptr;  // ct_f / flist
    const int32_t *i2 = nullptr;  // fmap
    const int32_t *i3 = nullptr;  // CSR columns (KO_EPROLONG)
    const double *w = nullptr;    // CSR weights / ct_coef / pinv
    const double *d = nullptr;    // diagonal
    double *x = nullptr, *y = nullptr, *b = nullptr, *dv = nullptr, *z = nullptr, *q = nullptr;
    double c1 = 0, c2 = 0;
    const double *pd = nullptr;   // fused coarse step 0: coarse diagonal (null = none)
    double pinv_theta = 0;
    double *px = nullptr, *pdv = nullptr;
};

struct KTail {
    int level = -1;
    bool pre0 = false;
    KOp *dprog = nullptr;
    int nops = 0;
    Stats counts;  // the launched path's equivalent work (edges, bytes) per call
};

// ------------------------------------------------------------------ device
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

__device__ __forceinline__ void kt_epi(const KOp &o, int64_t i, double ax, double &da, double &db) {
    const double xi = o.x[i], di = o.d[i];
    const double lx = di * xi - ax;
    if (o.epi == KE_CHEB) {
        double dv = o.c1 * o.dv[i] + o.c2 * ((o.b[i] - lx) / di);
        o.dv[i] = dv;
        o.y[i] = xi + dv;
    } else if (o.epi == KE_CHEB0) {
        double dv = o.c2 * ((o.b[i] - lx) / di);
        o.dv[i] = dv;
        o.y[i] = xi + dv;
    } else if (o.epi == KE_RESID) {
        o.y[i] = o.b[i] - lx;
    } else {  // KE_FCG: q = L p ; p.q ; p.r
        o.y[i] = lx;
        da += xi * lx;
        db += xi * o.b[i];
    }
}

__device__ __forceinline__ void kt_put_b(const KOp &o, int64_t k, double s) {
    o.y[k] = s;
    if (o.pd) {
        double v = (s / o.pd[k]) * o.pinv_theta;
        o.pdv[k] = v;
        o.px[k] = v;
    }
}

__global__ void __launch_bounds__(KT_THREADS, 1) k_ktail(const KOp *__restrict__ prog, int nops) {
    pdl_begin();
    __shared__ double slots[64];
    __shared__ double red[32];
    __shared__ __align__(16) KOp op;  // the current op, staged once for the CTA
    static_assert(sizeof(KOp) % 16 == 0, "KOp staging copies int4 words");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    for (int k = tid; k < 64; k += blockDim.x) slots[k] = 0.0;
    for (int pc = 0; pc < nops; pc++) {
        if (tid < (int)(sizeof(KOp) / 16)) ((int4 *)&op)[tid] = ((const int4 *)(prog + pc))[tid];
        __syncthreads();
        const KOp &o = op;
        switch (o.code) {
            case KO_CHEB_FIRST:
                for (int64_t i = tid; i < o.n; i += blockDim.x) {
                    double v = (o.b[i] / o.d[i]) * o.c1;
                    o.dv[i] = v;
                    o.x[i] = v;
                }
                break;
            case KO_SPMV: {
                double da = 0.0, db = 0.0;
                const int64_t nshort = o.n2;
                for (int64_t i = tid; i < nshort; i += blockDim.x) {  // short rows: a thread per row
                    double ax = 0.0;
#pragma unroll 4
                    for (int64_t q = o.rp[i]; q < o.rp[i + 1]; q++) ax += __ldg(&o.w[q]) * o.x[__ldg(&o.i0[q])];
                    kt_epi(o, i, ax, da, db);
                }
                for (int64_t i = nshort + warp; i < o.n; i += nw) {  // long rows: a warp per row
                    double ax = 0.0;
                    for (int64_t q = o.rp[i] + lane; q < o.rp[i + 1]; q += 32) ax += __ldg(&o.w[q]) * o.x[__ldg(&o.i0[q])];
                    for (int s = 16; s > 0; s >>= 1) ax += __shfl_xor_sync(0xffffffffu, ax, s);
                    if (lane == 0) kt_epi(o, i, ax, da, db);
                }
                if (o.epi == KE_FCG) {
                    double t0 = kt_block_sum(da, red);
                    double t1 = kt_block_sum(db, red);
                    if (tid == 0) {
                        slots[o.s0] = t0;
                        slots[o.s1] = t1;
                    }
                }
                break;
            }
            case KO_RESTRICT:  // o.n = m aggregates, rp = member ptr, i0 = members, x = r, y = bc
                for (int64_t a = tid; a < o.n; a += blockDim.x) {
                    double acc = 0.0;
                    for (int64_t q = o.rp[a]; q < o.rp[a + 1]; q++) acc += o.x[o.i0[q]];
                    kt_put_b(o, a, acc);
                }
                break;
            case KO_PROLONG:  // o.n fine rows, i0 = agg, x = xc, y = x
                for (int64_t i = tid; i < o.n; i += blockDim.x) o.y[i] += o.x[o.i0[i]];
                break;
            case KO_ERESTRICT:  // o.n = nc, i0 = cid, rp = ct_ptr, i1 = ct_f, w = ct_coef, b = fine b, y = bc
                for (int64_t k = tid; k < o.n; k += blockDim.x) {
                    double s = o.b[o.i0[k]];
                    for (int64_t q = o.rp[k]; q < o.rp[k + 1]; q++) s += o.w[q] * o.b[o.i1[q]];
                    kt_put_b(o, k, s);
                }
                break;
            case KO_EPROLONG:  // o.n = nc, o.n2 = nF, i0 = cid, i1 = flist, i2 = fmap, CSR (rp, i3, w, d)
                for (int64_t t = tid; t < o.n + o.n2; t += blockDim.x) {
                    if (t < o.n) {
                        o.y[o.i0[t]] = o.x[t];
                    } else {
                        const int64_t f = o.i1[t - o.n];
                        double s = o.b[f];
                        for (int64_t q = o.rp[f]; q < o.rp[f + 1]; q++) s += o.w[q] * o.x[o.i2[o.i3[q]]];
                        o.y[f] = s / o.d[f];
                    }
                }
                break;
            case KO_COARSE:  // o.n rows, w = P, b = rhs, y = x ; a warp per row (k_coarse_gemv order)
                for (int64_t i = warp; i < o.n; i += nw) {
                    double acc = 0.0;
                    for (int64_t j = lane; j < o.n; j += 32) acc += o.w[i * o.n + j] * o.b[j];
                    for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
                    if (lane == 0) o.y[i] = acc;
                }
                break;
            case KO_DOT: {  // slot s0 = x . y
                double acc = 0.0;
                for (int64_t i = tid; i < o.n; i += blockDim.x) acc += o.x[i] * o.y[i];
                double t = kt_block_sum(acc, red);
                if (tid == 0) slots[o.s0] = t;
                break;
            }
            case KO_FCG_DIR: {  // z, p = x ; slots: s0 = p.q, s2 = z.q
                const double pq = slots[o.s0], zq = slots[o.s2];
                const double beta = pq != 0.0 ? -zq / pq : 0.0;
                for (int64_t i = tid; i < o.n; i += blockDim.x) o.x[i] = o.z[i] + beta * o.x[i];
                break;
            }
            case KO_FCG_UPDATE: {  // p = z, q, rin = b, x, rout = y ; slots s0 = p.q, s1 = p.r
                const double pq = slots[o.s0], pr = slots[o.s1];
                const double alpha = pq != 0.0 ? pr / pq : 0.0;
                for (int64_t i = tid; i < o.n; i += blockDim.x) {
                    o.x[i] = o.first ? alpha * o.z[i] : o.x[i] + alpha * o.z[i];
                    o.y[i] = o.b[i] - alpha * o.q[i];
                }
                break;
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ host: record the recursion
namespace {
struct Emitter {
    lap_hierarchy *h;
    std::vector<KOp> ops;
    Stats cnt;
    int slot_base(int l) const { return 3 * l; }  // pq, pr, zq per level

    static bool fuse_on() {
        const char *e = getenv("LAP_FUSE_TRANSFERS");
        return !(e && e[0] == '0');
    }
    void pre0_of(KOp &o, int c) {  // fused coarse step 0 for an aggregation child (solve.cu Pre0)
        Level &C = h->lev[c];
        if (C.kind == KIND_AGG && fuse_on()) {
            o.pd = C.sd;
            o.pinv_theta = 1.0 / C.cheb_theta;
            o.px = C.x2;
            o.pdv = C.dv;
        }
    }
    void spmv(const Level &L, int epi, double *x, double *y, double *b, double *dv, double c1, double c2, int s0 = 0,
              int s1 = 0) {
        KOp o;
        o.code = KO_SPMV;
        o.epi = epi;
        o.n = L.n;
        o.n2 = L.c_end[0];
        o.rp = L.srp;
        o.i0 = L.scol;
        o.w = L.sw;
        o.d = L.sd;
        o.x = x;
        o.y = y;
        o.b = b;
        o.dv = dv;
        o.c1 = c1;
        o.c2 = c2;
        o.s0 = s0;
        o.s1 = s1;
        ops.push_back(o);
        cnt.edges += L.nnz;
        cnt.bytes += 12 * L.nnz + 40 * L.n;
    }
    // solve.cu cycle_rec with kc = true
    void kcycle(int l, double *b, double *xout, bool pre0_done) {
        Level &L = h->lev[l];
        const int64_t n = L.n;
        if (L.kind == KIND_COARSEST) {
            KOp o;
            o.code = KO_COARSE;
            o.n = n;
            o.w = L.pinv_s;
            o.b = b;
            o.y = xout;
            ops.push_back(o);
            cnt.bytes += 8 * n * n;
            return;
        }
        Level &C = h->lev[l + 1];
        if (L.kind == KIND_ELIM) {
            KOp o;
            o.code = KO_ERESTRICT;
            o.n = C.n;
            o.i0 = L.cid_s;
            o.rp = L.ct_ptr_s;
            o.i1 = L.ct_f_s;
            o.w = L.ct_coef_s;
            o.b = b;
            o.y = C.b;
            pre0_of(o, l + 1);
            const bool fuse0 = o.pd != nullptr;
            ops.push_back(o);
            kcoarse(l + 1, fuse0);
            KOp p;
            p.code = KO_EPROLONG;
            p.n = C.n;
            p.n2 = L.nF;
            p.i0 = L.cid_s;
            p.i1 = L.flist;
            p.i2 = L.fmap_s;
            p.rp = L.srp;
            p.i3 = L.scol;
            p.w = L.sw;
            p.d = L.sd;
            p.b = b;
            p.x = C.x;
            p.y = xout;
            ops.push_back(p);
            cnt.bytes += 16 * n;
            return;
        }
        const int K = h->p.cheby_degree;
        const double theta = L.cheb_theta, delta = L.cheb_delta, sigma = L.cheb_sigma;
        double *cur = L.x2, *alt = L.t;
        if (!pre0_done) {
            KOp o;
            o.code = KO_CHEB_FIRST;
            o.n = n;
            o.b = b;
            o.d = L.sd;
            o.c1 = 1.0 / theta;
            o.x = cur;
            o.dv = L.dv;
            ops.push_back(o);
        }
        cnt.bytes += 32 * n;
        double rho_old = 1.0 / sigma;
        for (int k = 1; k < K; k++) {
            double rho = 1.0 / (2.0 * sigma - rho_old);
            spmv(L, KE_CHEB, cur, alt, b, L.dv, rho * rho_old, 2.0 * rho / delta);
            std::swap(cur, alt);
            rho_old = rho;
        }
        spmv(L, KE_RESID, cur, L.r, b, nullptr, 0, 0);
        KOp r;
        r.code = KO_RESTRICT;
        r.n = L.m;
        r.rp = L.mem_ptr;
        r.i0 = L.members;
        r.x = L.r;
        r.y = C.b;
        pre0_of(r, l + 1);
        const bool fuse0 = r.pd != nullptr;
        ops.push_back(r);
        kcoarse(l + 1, fuse0);
        KOp p;
        p.code = KO_PROLONG;
        p.n = n;
        p.i0 = L.agg_s;
        p.x = C.x;
        p.y = cur;
        ops.push_back(p);
        cnt.bytes += 36 * n + 16 * L.m;
        rho_old = 1.0 / sigma;
        for (int k = 0; k < K; k++) {
            double *dst = (k == K - 1) ? xout : alt;
            if (k == 0) {
                spmv(L, KE_CHEB0, cur, dst, b, L.dv, 0.0, 1.0 / theta);
            } else {
                double rho = 1.0 / (2.0 * sigma - rho_old);
                spmv(L, KE_CHEB, cur, dst, b, L.dv, rho * rho_old, 2.0 * rho / delta);
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
        const int sq = slot_base(l), sr = sq + 1, sz = sq + 2;
        for (int k = 1; k <= h->p.kcycle_inner; k++) {
            double *rin = k == 1 ? L.b : L.kr;
            if (k == 1) {
                kcycle(l, L.b, L.kp, pre0_done);
            } else {
                kcycle(l, L.kr, L.kz, false);
                KOp d;
                d.code = KO_DOT;
                d.n = L.n;
                d.x = L.kz;
                d.y = L.kq;
                d.s0 = sz;
                ops.push_back(d);
                KOp o;
                o.code = KO_FCG_DIR;
                o.n = L.n;
                o.z = L.kz;
                o.x = L.kp;
                o.s0 = sq;
                o.s2 = sz;
                ops.push_back(o);
            }
            spmv(L, KE_FCG, L.kp, L.kq, rin, nullptr, 0, 0, sq, sr);
            KOp u;
            u.code = KO_FCG_UPDATE;
            u.n = L.n;
            u.z = L.kp;
            u.q = L.kq;
            u.b = rin;
            u.x = L.x;
            u.y = L.kr;
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

void build_ktail(lap_hierarchy *h, cudaStream_t s) {
    free_ktail(h, s);
    const int nl = (int)h->lev.size();
    if (h->p.cycle != 1 || !ktail_enabled() || nl < 2 || 3 * nl > 64) return;
    int t = nl;
    while (t > 1 && small_level(h->lev[t - 1])) t--;
    if (t >= nl || h->lev[t].kind == KIND_COARSEST) return;  // nothing worth a program
    Emitter em{h, {}, {}};
    const bool pre0 = h->lev[t].kind == KIND_AGG && Emitter::fuse_on();  // what the caller of kcoarse(t) passes
    em.kcoarse(t, pre0);
    KTail *kt = new KTail();
    kt->level = t;
    kt->pre0 = pre0;
    kt->nops = (int)em.ops.size();
    kt->counts = em.cnt;
    kt->dprog = (KOp *)dalloc(sizeof(KOp) * em.ops.size(), s);
    // pageable source: the call returns once em.ops has been staged
    LAP_CUDA(cudaMemcpyAsync(kt->dprog, em.ops.data(), sizeof(KOp) * em.ops.size(), cudaMemcpyHostToDevice, s));
    h->ktail = kt;
}

void free_ktail(lap_hierarchy *h, cudaStream_t s) {
    KTail *kt = (KTail *)h->ktail;
    if (!kt) return;
    dfree(kt->dprog, s);
    delete kt;
    h->ktail = nullptr;
}

// kcoarse(l) as one launch when l is the program's level (and the caller's fusion matches)
bool ktail_launch(lap_hierarchy *h, int l, bool pre0_done, cudaStream_t s) {
    KTail *kt = (KTail *)h->ktail;
    if (!kt || kt->level != l || kt->pre0 != pre0_done) return false;
    launch_pdl(k_ktail, 1, KT_THREADS, s, (const KOp *)kt->dprog, kt->nops);
    h->cur.launches++;
    h->cur.edges += kt->counts.edges;
    h->cur.bytes += kt->counts.bytes;
    LAP_CHECK_LAUNCH();
    return true;
}

}  // namespace lap
