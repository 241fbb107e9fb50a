// Single-warp FP64 issue-rate microbenchmarks (not part of the library).
#include <cstdio>
#include <cuda_runtime.h>

// K independent DFMA chains per thread; one warp per SM-subpartition or one
// warp total; reports cycles per DFMA instruction per warp.
template <int K>
__global__ void dfma_ilp(int iters, double x, double* out, long long* cyc) {
    double a[K];
#pragma unroll
    for (int k = 0; k < K; ++k) a[k] = threadIdx.x + k;
    __syncwarp();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < K; ++k) a[k] = fma(a[k], x, 1e-9);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) s += a[k];
    if (s == 12345.0) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int K>
__global__ void dmul_ilp(int iters, double x, double* out, long long* cyc) {
    double a[K];
#pragma unroll
    for (int k = 0; k < K; ++k) a[k] = threadIdx.x + k + 1;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < K; ++k) a[k] = a[k] * x;
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) s += a[k];
    if (s == 12345.0) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 64);
    cudaMalloc(&cyc, 64);
    long long h;
    const int it = 4096;
#define RUN(kern, K, blocks, threads, name)                                              \
    kern<K><<<blocks, threads>>>(it, 0.999999, out, cyc);                                 \
    cudaDeviceSynchronize();                                                             \
    kern<K><<<blocks, threads>>>(it, 0.999999, out, cyc);                                 \
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);                                      \
    printf("%-44s K=%2d  %7.2f cycles per instr per warp\n", name, K, (double)h / (it * (double)K));
    RUN(dfma_ilp, 1, 1, 32, "DFMA 1 warp");
    RUN(dfma_ilp, 2, 1, 32, "DFMA 1 warp");
    RUN(dfma_ilp, 4, 1, 32, "DFMA 1 warp");
    RUN(dfma_ilp, 8, 1, 32, "DFMA 1 warp");
    RUN(dfma_ilp, 16, 1, 32, "DFMA 1 warp");
    RUN(dfma_ilp, 8, 1, 64, "DFMA 2 warps/CTA");
    RUN(dfma_ilp, 8, 1, 128, "DFMA 4 warps/CTA");
    RUN(dfma_ilp, 8, 1, 256, "DFMA 8 warps/CTA");
    RUN(dfma_ilp, 8, 1, 512, "DFMA 16 warps/CTA");
    RUN(dmul_ilp, 8, 1, 32, "DMUL 1 warp");
    RUN(dmul_ilp, 8, 1, 128, "DMUL 4 warps/CTA");
    return 0;
}
