// Latency microbenchmarks for the block-RQ design (not part of the library).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1708_06290_b200/csrc/ss_device.cuh"

using namespace ssd;

__global__ void lat_dfma(int iters, double x, double* out, long long* cyc) {
    double a = threadIdx.x * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) a = fma(a, x, 1e-9);
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = a; cyc[0] = t1 - t0; }
}

__global__ void lat_rsqrt(int iters, double x, double* out, long long* cyc) {
    double a = 1.0 + threadIdx.x * 1e-3 + x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) a = rsqrt(a) + 0.5;
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = a; cyc[0] = t1 - t0; }
}

__global__ void lat_div(int iters, double x, double* out, long long* cyc) {
    double a = 1.0 + threadIdx.x * 1e-3 + x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) a = 1.5 / a + 0.25;
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = a; cyc[0] = t1 - t0; }
}

__global__ void lat_givens(int iters, int fast, double* out, long long* cyc) {
    double2 a = make_double2(0.3 + threadIdx.x * 1e-3, 0.2), b = make_double2(0.1, -0.4);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        double c;
        double2 s, r;
        if (fast) givens_fast(a, b, c, s, r); else givens(a, b, c, s, r);
        a = make_double2(r.x * 0.7 + c, r.y * 0.7);  // dependent chain
        b = make_double2(s.x + 0.1, s.y - 0.2);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = a.x + b.y; cyc[0] = t1 - t0; }
}

__global__ void lat_lds(int iters, double* out, long long* cyc) {
    __shared__ double2 buf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_double2(i & 1023, 0);
    __syncthreads();
    int idx = threadIdx.x & 1023;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) idx = ((int)buf[idx].x + 7) & 1023;
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = idx; cyc[0] = t1 - t0; }
}

__global__ void lat_bar(int iters, double* out, long long* cyc) {
    __shared__ double v[32];
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) v[i & 31] = i;
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = v[3]; cyc[0] = t1 - t0; }
}

// rotation apply over rows of a packed column pair in smem: one step of
// phase B with `rows` rows and TPR threads
__global__ void lat_apply(int iters, int rows, double* out, long long* cyc) {
    __shared__ double2 c1[128], c2[128];
    for (int i = threadIdx.x; i < 128; i += blockDim.x) { c1[i] = make_double2(i, 1); c2[i] = make_double2(1, i); }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        for (int i = threadIdx.x; i < rows; i += blockDim.x) {
            double2 h = c2[i], t = c1[i];
            rot_apply(0.6, make_double2(0.48, 0.64), h, t);
            c2[i] = h; c1[i] = t;
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = c1[5].x; cyc[0] = t1 - t0; }
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 64); cudaMalloc(&cyc, 64);
    long long h;
    const int it = 4096;
#define RUN(name, launch, div)                                          \
    launch; cudaDeviceSynchronize(); launch;                             \
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);                      \
    printf("%-40s %8.1f cycles\n", name, (double)h / (div));
    RUN("DFMA dependent", (lat_dfma<<<1, 32>>>(it, 0.999, out, cyc)), it);
    RUN("rsqrt(double) dependent", (lat_rsqrt<<<1, 32>>>(it, 0.1, out, cyc)), it);
    RUN("div(double) dependent", (lat_div<<<1, 32>>>(it, 0.1, out, cyc)), it);
    RUN("givens (hypot) dependent", (lat_givens<<<1, 32>>>(it, 0, out, cyc)), it);
    RUN("givens_fast dependent", (lat_givens<<<1, 32>>>(it, 1, out, cyc)), it);
    RUN("LDS.128 pointer chase", (lat_lds<<<1, 32>>>(it, out, cyc)), it);
    RUN("__syncthreads 96 thr", (lat_bar<<<1, 96>>>(it, out, cyc)), it);
    RUN("__syncthreads 256 thr", (lat_bar<<<1, 256>>>(it, out, cyc)), it);
    RUN("apply 63 rows / 8 thr + bar", (lat_apply<<<1, 8>>>(it / 8, 63, out, cyc)), it / 8);
    RUN("apply 63 rows / 32 thr + bar", (lat_apply<<<1, 32>>>(it / 8, 63, out, cyc)), it / 8);
    RUN("apply 63 rows / 64 thr + bar", (lat_apply<<<1, 64>>>(it / 8, 63, out, cyc)), it / 8);
    RUN("apply 16 rows / 16 thr + bar", (lat_apply<<<1, 16>>>(it / 8, 16, out, cyc)), it / 8);
    return 0;
}
