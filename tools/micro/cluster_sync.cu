// Microbenchmark: cost of one cluster barrier (barrier.cluster arrive/wait)
// among 8 CTAs, by block size and memory semantics; __syncthreads for scale.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(int iters, double *out) {
    double acc = threadIdx.x;
    for (int i = 0; i < iters; i++) {
        if (MODE == 0) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (MODE == 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
        if (MODE == 2) __syncthreads();
        acc = acc * 1.0000001 + 1.0;
    }
    if (acc == -1.0) out[0] = acc;
}
template <int MODE>
float run(int threads, int cl, int iters) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl);
    cfg.blockDim = dim3(threads);
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = cl; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    double *o; cudaMalloc(&o, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaLaunchKernelEx(&cfg, k<MODE>, iters, o);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k<MODE>, iters, o);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    if (err) printf("err %s\n", cudaGetErrorString(err));
    return ms * 1e3f / iters;
}
int main() {
    int iters = 20000;
    for (int th : {128, 256, 1024}) {
        printf("threads %4d cluster 8: release/acquire %.3f us, relaxed %.3f us, syncthreads %.3f us\n", th,
               run<0>(th, 8, iters), run<1>(th, 8, iters), run<2>(th, 8, iters));
        printf("threads %4d cluster 2: release/acquire %.3f us\n", th, run<0>(th, 2, iters));
    }
    return 0;
}
