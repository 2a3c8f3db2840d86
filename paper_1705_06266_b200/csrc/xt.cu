// xt.cu -- column-tiled ("x-stationary") layout of dense-ish levels.
//
// On a random-ordered power-law level every x gather of the SpMV is one 32-byte
// L2 sector request, and the L1TEX request rate -- not HBM -- bounds the CSR/SELL
// kernel (lap_bench_gather: ~2.5e11 random gathers/s on a B200, an SpMV-
// equivalent 0.45-0.5 of the HBM copy bandwidth).  The coarse levels produced
// by the first aggregation of R-MAT / BA graphs (cfg 3 level 1: 343K rows x 90
// entries; cfg 4 level 1: 720K x 79; cfg 5 level 3: 331K x 5400) are too big
// for the whole x in shared memory (k_spmv_smem) but dense enough that
// STREAMING x through shared memory is cheaper than gathering it:
//
//   * the rows are cut into nb row blocks of about equal work (one CTA each,
//     one CTA per SM), the columns into T tiles of W entries of x;
//   * the entries of (block b, tile t) form one segment, sorted by (row, col),
//     stored as a 32-bit (local row << 16 | local column) word + the fp64 weight
//     -- 12 B per entry, as the CSR;
//   * a CTA sweeps the tiles in order: x[tile] arrives in shared memory by a TMA
//     bulk copy (cp.async.bulk + mbarrier, double-buffered so tile t+1 loads
//     while tile t is consumed), its 16 warps read their segment entries with
//     coalesced loads (4 chunks of 32 in flight per warp) and gather x from
//     shared memory; each warp takes an equal share of the segment's entries,
//     adds segmented (row-run) warp sums into a shared-memory y, and hands the
//     run of its first row (which may continue the previous warp's) to a carry
//     that one thread adds after the tile in warp order -- a fixed summation
//     order, bitwise reproducible, no atomics, hub rows spread over all warps;
//   * the fused epilogue (diagonal, Chebyshev, residual, dots) runs per row.
//
// Traffic per SpMV: 12 B/entry + the epilogue vectors from HBM, plus nb * 8n
// bytes of x tiles from L2 (bulk, one request per 16 KB instead of one per
// entry).  Chosen per level by xt_eligible(); the CSR/SELL storage stays for
// the other consumers (block SpMM, sharded solve, export).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "lap_internal.cuh"

namespace lap {

constexpr int XT_RMAX = 6144;        // rows per block (8 B each in shared memory)
constexpr int XT_W_DEFAULT = 10240;  // x entries per tile (80 KB; two buffers)

static int env_int(const char *name, int dflt) {
    const char *e = getenv(name);
    return e ? atoi(e) : dflt;
}

bool xt_eligible(const Level &L, int l) {
    // Off by default: measured no faster than the SELL/chunk kernel (dense random
    // level n = 100K x 1980: 861 vs 873 us; cfg 5 level 3 slower).
    // LAP_XT=1 applies the rule below, LAP_XT=force any level (tests).
    const char *e = getenv("LAP_XT");
    if (!e || e[0] == '0') return false;
    const bool force = e[0] == 'f';  // tests: any level with a few hundred rows
    if (L.smem_x || L.n < 2 || L.nnz == 0) return false;
    if (force) return L.n >= 256 && L.nnz >= 4 * L.n;
    if (L.spmv_vec) return false;
    if (L.kind == KIND_ELIM && l > 0) return false;  // no SpMV on an elimination level below 0 in the solve
    // dense enough that streaming x (nb * 8n bytes from L2) beats one sector per
    // entry (32 B): average degree >= 32; tiles bounded (T < 4096)
    if (!(L.n > SMEM_X_MAX && L.nnz >= 32 * L.n && L.n < (int64_t)XT_W_DEFAULT * 4000)) return false;
    // a row's entries inside one tile must form long runs (>= 8 on average) or the
    // per-chunk segmented scans cost more issue slots than the gathers they save
    // (cfg 3 / 4 level 1: 1-3 entries per row and tile, measured slower than SELL)
    const double run = (double)L.nnz / (double)L.n * std::min<double>(1.0, (double)XT_W_DEFAULT / (double)L.n);
    if (run < env_int("LAP_XT_MIN_RUN", 8)) return false;
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    uint64_t rsv = 0, used = 0;  // memory liblap's pool holds but does not use is free for us too
    cudaMemPoolGetAttribute(lib_pool(), cudaMemPoolAttrReservedMemCurrent, &rsv);
    cudaMemPoolGetAttribute(lib_pool(), cudaMemPoolAttrUsedMemCurrent, &used);
    const double avail = (double)fr + (double)(rsv - used);
    return avail > 1.5 * 12.0 * (double)L.nnz + 8e9;  // the copy + its build buffers, with headroom
}

// row-block boundaries: equal shares of (entries + XT_ROWCOST * rows)
constexpr int64_t XT_ROWCOST = 8;
__global__ void k_xt_bounds(int64_t n, int nb, const int64_t *__restrict__ srp, int64_t *__restrict__ rb) {
    const int64_t total = srp[n] + XT_ROWCOST * n;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += gridDim.x * blockDim.x) {
        const int64_t target = (int64_t)((double)total * b / nb);
        int64_t lo = 0, hi = n;  // first p with srp[p] + c p >= target
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (srp[mid] + XT_ROWCOST * mid < target) lo = mid + 1;
            else hi = mid;
        }
        rb[b] = b == 0 ? 0 : (b == nb ? n : lo);
    }
}
// sort keys of the entries [E0, E1) (rows [p0, p0 + nrows) = blocks [b0, b1)):
//   (block - b0) << 39 | tile << 27 | local row << 14 | local column
// G lanes per row (hub rows stream), the row's block by one small search
template <int G>
__global__ void k_xt_keys(int64_t nrows, int64_t p0, int64_t E0, int b0, int b1, int W, const int64_t *__restrict__ rb,
                          const int64_t *__restrict__ srp, const int32_t *__restrict__ scol, uint64_t *__restrict__ key,
                          int32_t *__restrict__ idx) {
    GROUP_LOOP_BEGIN(G, nrows)
    if (live) {
        const int64_t p = p0 + i;
        int blo = b0, bhi = b1 - 1;
        while (blo < bhi) {
            const int mid = (blo + bhi + 1) >> 1;
            if (rb[mid] <= p) blo = mid;
            else bhi = mid - 1;
        }
        const uint64_t hi = ((uint64_t)(blo - b0) << 39) | ((uint64_t)(p - rb[blo]) << 14);
        for (int64_t k = srp[p] + gl; k < srp[p + 1]; k += G) {
            const int64_t c = scol[k];
            const uint64_t t = (uint64_t)(c / W);
            key[k - E0] = hi | (t << 27) | (uint64_t)(c - (int64_t)t * W);
            idx[k - E0] = (int32_t)(k - E0);
        }
    }
    GROUP_LOOP_END
}
__global__ void k_xt_fill(int64_t cnt, int64_t E0, const uint64_t *__restrict__ key, const int32_t *__restrict__ idx,
                          const double *__restrict__ sw, uint32_t *__restrict__ rc, double *__restrict__ w) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = key[q];
        rc[E0 + q] = (uint32_t)((((k >> 14) & 0x1FFF) << 16) | (k & 0x3FFF));
        w[E0 + q] = sw[E0 + idx[q]];
    }
}
__device__ __forceinline__ int64_t xt_lower(const uint64_t *__restrict__ key, int64_t cnt, uint64_t v) {
    int64_t lo = 0, hi = cnt;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (key[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
// segment starts of blocks [b0, b1): first entry of (block, tile) in sorted order
__global__ void k_xt_segs(int64_t cnt, int64_t E0, int b0, int b1, int T, const uint64_t *__restrict__ key,
                          int64_t *__restrict__ seg) {
    const int64_t npairs = (int64_t)(b1 - b0) * T;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < npairs; q += (int64_t)gridDim.x * blockDim.x) {
        const int bl = (int)(q / T), t = (int)(q % T), b = b0 + bl;
        seg[(int64_t)b * T + t] = E0 + xt_lower(key, cnt, ((uint64_t)bl << 39) | ((uint64_t)t << 27));
    }
}

void build_xt(Level &L, cudaStream_t s) {
    const int64_t n = L.n, nnz = L.nnz;
    int W = env_int("LAP_XT_W", XT_W_DEFAULT);
    W = std::max(2, std::min(11264, W & ~1));  // 2 W + XT_RMAX doubles <= XT_SMEM_MAX
    const int64_t T = (n + W - 1) / W;
    if (T >= 4096) return;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int nb = env_int("LAP_XT_NB", sms);
    nb = std::max(1, nb);
    std::vector<int64_t> hrb;
    DBuf<int64_t> rb;
    for (;;) {  // rows per block <= XT_RMAX (and < 2^13 for the 13-bit local row of the sort key)
        rb.alloc(nb + 1, s);
        k_xt_bounds<<<grid_for(nb + 1, 128, 64), 128, 0, s>>>(n, nb, L.srp, rb.p);
        LAP_CHECK_LAUNCH();
        hrb.resize(nb + 1);
        LAP_CUDA(cudaMemcpyAsync(hrb.data(), rb.p, 8 * (nb + 1), cudaMemcpyDeviceToHost, s));
        LAP_CUDA(cudaStreamSynchronize(s));
        int64_t rmax = 0;
        for (int b = 0; b < nb; b++) rmax = std::max(rmax, hrb[b + 1] - hrb[b]);
        if (rmax <= XT_RMAX || nb > 65536) {
            L.xt_rmax = (int)std::max<int64_t>(1, rmax);
            break;
        }
        nb *= 2;
    }
    if (L.xt_rmax > XT_RMAX || 8 * (size_t)(2 * W + L.xt_rmax) > XT_SMEM_MAX) return;
    g_kl++;
    std::vector<int64_t> hsrp(nb + 1);
    for (int b = 0; b <= nb; b++) LAP_CUDA(cudaMemcpyAsync(&hsrp[b], L.srp + hrb[b], 8, cudaMemcpyDeviceToHost, s));
    LAP_CUDA(cudaStreamSynchronize(s));
    L.xt_nb = nb;
    L.xt_T = (int)T;
    L.xt_W = W;
    L.xt_rb = rb.take();
    L.xt_seg = (int64_t *)dalloc(sizeof(int64_t) * ((size_t)nb * T + 1), s);
    L.xt_rc = (uint32_t *)dalloc(sizeof(uint32_t) * (size_t)(nnz + 1), s);
    L.xt_w = (double *)dalloc(sizeof(double) * (size_t)(nnz + 1), s);
    // batches of whole blocks, <= 2^27 entries (one radix sort each)
    const int64_t budget = (int64_t)1 << 27;
    int b0 = 0;
    while (b0 < nb) {
        int b1 = b0 + 1;
        while (b1 < nb && b1 - b0 < 255 && hsrp[b1 + 1] - hsrp[b0] <= budget) b1++;
        const int64_t E0 = hsrp[b0], E1 = hsrp[b1], cnt = E1 - E0;
        if (cnt > 0) {
            DBuf<uint64_t> k1(cnt, s), k2(cnt, s);
            DBuf<int32_t> i1(cnt, s), i2(cnt, s);
            const int64_t nrows = hrb[b1] - hrb[b0];
            LAUNCH_G(group_size(nrows, cnt), k_xt_keys, nrows, s, nrows, hrb[b0], E0, b0, b1, W, L.xt_rb, L.srp,
                     L.scol, k1.p, i1.p);
            size_t bytes = 0;
            LAP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k1.p, k2.p, i1.p, i2.p, cnt, 0, 47, s));
            DBuf<char> tmp((int64_t)bytes, s);
            LAP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, k1.p, k2.p, i1.p, i2.p, cnt, 0, 47, s));
            k_xt_fill<<<grid_for(cnt, 256, 148 * 16), 256, 0, s>>>(cnt, E0, k2.p, i2.p, L.sw, L.xt_rc, L.xt_w);
            k_xt_segs<<<grid_for((int64_t)(b1 - b0) * T, 128, 148 * 8), 128, 0, s>>>(cnt, E0, b0, b1, (int)T, k2.p,
                                                                                     L.xt_seg);
            g_kl += 4;
            LAP_CHECK_LAUNCH();
        } else {
            // empty blocks: every segment starts (and ends) at E0
            std::vector<int64_t> z((size_t)(b1 - b0) * T, E0);
            LAP_CUDA(cudaMemcpyAsync(L.xt_seg + (int64_t)b0 * T, z.data(), 8 * z.size(), cudaMemcpyHostToDevice, s));
            LAP_CUDA(cudaStreamSynchronize(s));
        }
        b0 = b1;
    }
    LAP_CUDA(cudaMemcpyAsync(L.xt_seg + (int64_t)nb * T, &hsrp[nb], 8, cudaMemcpyHostToDevice, s));
    LAP_CUDA(cudaStreamSynchronize(s));
    L.xt = true;
}

}  // namespace lap
