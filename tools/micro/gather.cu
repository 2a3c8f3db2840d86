// gather.cu -- the M3 "second ceiling": throughput of random
// 8-byte gathers x[idx[k]] on one B200, as a function of the size of x, for
// the access shapes the SpMV kernels use.  Not product code; a measurement.
//
// For each |x| (64 KB .. 256 MB) and each variant, M = 2^26 gathers; indices
// uniform in [0, n) from a counter hash (no locality: the worst case of a
// random-ordered power-law level), streamed with coalesced loads.
//   idx     : gather + 4-byte index stream              (request-rate ceiling)
//   spmv    : gather + 4-byte col + 8-byte w streams     (= SpMV without epilogue)
//   spmv_cg : spmv with the gather through L2 only (ld.global.cg)
//   seq     : spmv with idx[k] = k mod n (no randomness; the HBM stream ceiling)
//   hot     : spmv where 50% of gathers hit a 16K-entry hot set (hub x in L1)
// Reported: ms, gathers/s, "SpMV-equivalent" GB/s = 12 B per gather / t and its
// fraction of the measured HBM copy bandwidth, sectors/s = gathers/s (one 32 B
// sector per random 8 B gather).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather gather.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__host__ __device__ inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void k_make_idx(int64_t M, int64_t n, int mode, int32_t *idx, double *w) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < M; k += (int64_t)gridDim.x * blockDim.x) {
        uint64_t h = mix64(k * 0x9E3779B97F4A7C15ULL + 12345);
        int64_t j;
        if (mode == 1) j = k % n;
        else if (mode == 2 && (h >> 63)) j = (int64_t)((h >> 20) % (uint64_t)(n < 16384 ? n : 16384));
        else j = (int64_t)(h % (uint64_t)n);
        idx[k] = (int32_t)j;
        w[k] = 1.0 + (double)(h & 1023) * 1e-3;
    }
}
__global__ void k_fill(int64_t n, double *x) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        x[k] = 1.0 / (1.0 + (double)k);
}

template <int VAR, int U>
__global__ void __launch_bounds__(256) k_gather(int64_t M, const int32_t *__restrict__ idx, const double *__restrict__ w,
                                                const double *__restrict__ x, double *__restrict__ out) {
    double acc = 0.0;
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; k + (U - 1) * T < M; k += U * T) {
        int32_t j[U];
        double ww[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            j[u] = __ldcs(idx + k + u * T);
            ww[u] = VAR == 0 ? 1.0 : __ldcs(w + k + u * T);
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            double xv = VAR == 2 ? __ldcg(x + j[u]) : __ldg(x + j[u]);
            acc += ww[u] * xv;
        }
    }
    for (; k < M; k += T) acc += (VAR == 0 ? 1.0 : w[k]) * x[idx[k]];
    if (acc == 12345.678) out[0] = acc;  // keep the loads live
}

int main(int argc, char **argv) {
    double hbm = argc > 1 ? atof(argv[1]) : 6534.5;
    int dev = 0;
    cudaDeviceProp pr;
    CK(cudaGetDeviceProperties(&pr, dev));
    const int64_t M = 1LL << 26;
    int32_t *idx;
    double *w, *x, *out;
    CK(cudaMalloc(&idx, 4 * M));
    CK(cudaMalloc(&w, 8 * M));
    CK(cudaMalloc(&x, 8LL << 25));
    CK(cudaMalloc(&out, 8));
    k_fill<<<1184, 256>>>(1LL << 25, x);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    printf("# %s, %d SMs; M = %lld gathers per launch; hbm %.1f GB/s\n", pr.name, pr.multiProcessorCount, (long long)M, hbm);
    printf("%-8s %10s %9s %12s %10s %7s\n", "variant", "x_bytes", "ms", "gathers/s", "spmvGB/s", "frac");
    const int grid = pr.multiProcessorCount * 8;
    for (int mode = 0; mode < 3; mode++) {
        for (int64_t n = 1 << 13; n <= (1LL << 25); n <<= 2) {
            k_make_idx<<<1184, 256>>>(M, n, mode, idx, w);
            CK(cudaDeviceSynchronize());
            const char *names[] = {"idx", "spmv", "spmv_cg"};
            for (int var = 0; var < 3; var++) {
                if (mode != 0 && var != 1) continue;
                float best = 1e30f;
                for (int rep = 0; rep < 6; rep++) {
                    CK(cudaEventRecord(a));
                    if (var == 0) k_gather<0, 8><<<grid, 256>>>(M, idx, w, x, out);
                    if (var == 1) k_gather<1, 8><<<grid, 256>>>(M, idx, w, x, out);
                    if (var == 2) k_gather<2, 8><<<grid, 256>>>(M, idx, w, x, out);
                    CK(cudaEventRecord(b));
                    CK(cudaEventSynchronize(b));
                    float ms;
                    CK(cudaEventElapsedTime(&ms, a, b));
                    if (rep >= 2 && ms < best) best = ms;
                }
                double gps = M / (best * 1e-3);
                double gbs = 12.0 * M / (best * 1e-3) / 1e9;
                const char *nm = mode == 1 ? "seq" : mode == 2 ? "hot50" : names[var];
                printf("%-8s %10lld %9.3f %12.4e %10.1f %7.3f\n", nm, (long long)(8 * n), best, gps, gbs, gbs / hbm);
            }
        }
    }
    CK(cudaGetLastError());
    return 0;
}
