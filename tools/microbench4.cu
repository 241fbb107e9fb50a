// Update-loop microbenchmark (not part of the library): the k_update_ws
// inner loop (4 real panel rows x 5 complex P columns = 40 DFMA per panel
// column) with operands from registers or from shared memory, at 1..4 warps
// per SMSP.  Reports DFMA per clock per SM (peak 64).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double2 rfma(double a, double2 b, double2 c) {
    return make_double2(fma(a, b.x, c.x), fma(a, b.y, c.y));
}

template <int MODE, int ORD>  // MODE 0: registers only, 1: LDS like the kernel; ORD 0: c outer, 1: r outer
__global__ void loop(int iters, double* out, long long* cyc) {
    __shared__ __align__(16) double pan[64 * 64];
    __shared__ __align__(16) double2 P[64 * 10];
    for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) pan[i] = 1e-3 * (i & 7);
    for (int i = threadIdx.x; i < 64 * 10; i += blockDim.x) P[i] = make_double2(1e-4 * (i & 3), 1e-4);
    __syncthreads();
    const int lane = threadIdx.x & 31, rg = lane >> 1, q = lane & 1;
    double2 acc[4][5];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 5; ++c) acc[r][c] = make_double2(0, 0);
    const double* pl = pan + rg * 2;
    const double2* Pl = P + q * 5;
    double a[4];
    double2 pv[5];
#pragma unroll
    for (int r = 0; r < 4; ++r) a[r] = pl[r];
#pragma unroll
    for (int c = 0; c < 5; ++c) pv[c] = Pl[c];
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll 2
        for (int j = 0; j < 64; ++j) {
            if (MODE >= 1) {
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    const double2 v = *reinterpret_cast<const double2*>(pl + j * 64 + p * 32);
                    a[2 * p] = v.x;
                    a[2 * p + 1] = v.y;
                }
            }
            if (MODE >= 1) {
#pragma unroll
                for (int c = 0; c < 5; ++c) pv[c] = Pl[(j % 64) * 10 + c];
            }
            if (ORD == 0) {
#pragma unroll
                for (int c = 0; c < 5; ++c)
#pragma unroll
                    for (int r = 0; r < 4; ++r) acc[r][c] = rfma(a[r], pv[c], acc[r][c]);
            } else {
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int c = 0; c < 5; ++c) acc[r][c] = rfma(a[r], pv[c], acc[r][c]);
            }
            if (MODE == 0) {
                a[j & 3] += 1e-12;  // keep the operands live, one DADD per 40 DFMA
            }
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    double s = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 5; ++c) s += acc[r][c].x + acc[r][c].y;
    if (s == 12345.0) out[0] = s;
}

template <int MODE, int ORD>
void run(int warps, int sms) {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 8 * sms);
    const int iters = 400;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    loop<MODE, ORD><<<sms, 32 * warps>>>(10, out, cyc);
    cudaEventRecord(e0);
    loop<MODE, ORD><<<sms, 32 * warps>>>(iters, out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double dfma = 40.0 * 64 * iters * 32.0 * warps;  // per SM (lane ops)
    long long c0 = 0;
    cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
    const double cycles = (double)c0;
    printf("mode %d ord %d warps/SM %2d: %.1f DFMA/clk/SM (%.0f%% of 64) by SM clock; %.0f MHz\n", MODE, ORD,
           warps, dfma / cycles, 100.0 * dfma / cycles / 64, cycles / (ms * 1e3));
    cudaFree(out);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {4, 8, 12, 16}) run<0, 0>(w, sms);
    for (int w : {4, 8, 12, 16}) run<0, 1>(w, sms);
    for (int w : {4, 8, 12, 16}) run<1, 0>(w, sms);
    for (int w : {4, 8, 12, 16}) run<1, 1>(w, sms);
    return 0;
}
