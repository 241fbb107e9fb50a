// Update-loop microbenchmark II (not part of the library): R real panel rows
// x C complex P columns per lane (G = 10 / C column groups... lanes = rg x q),
// operands from shared memory as in k_update_ws, 1..4 warps per SMSP.
// Reports DFMA per clock per SM (peak 64) from the SM clock.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double2 rfma(double a, double2 b, double2 c) {
    return make_double2(fma(a, b.x, c.x), fma(a, b.y, c.y));
}

template <int R, int C, int G>
__global__ void loop(int iters, double* out, long long* cyc) {
    constexpr int RG = 32 / G, ROWS = RG * R;
    __shared__ __align__(16) double pan[32 * ROWS];
    __shared__ __align__(16) double2 P[64 * 10];
    for (int i = threadIdx.x; i < 32 * ROWS; i += blockDim.x) pan[i] = 1e-3 * (i & 7);
    for (int i = threadIdx.x; i < 64 * 10; i += blockDim.x) P[i] = make_double2(1e-4 * (i & 3), 1e-4);
    __syncthreads();
    const int lane = threadIdx.x & 31, rg = lane / G, q = lane % G;
    double2 acc[R][C];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) acc[r][c] = make_double2(0, 0);
    const double* pl = pan + rg * 2;
    const double2* Pl = P + q * C;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll 2
        for (int j = 0; j < 32; ++j) {
            double a[R];
#pragma unroll
            for (int p = 0; p < R / 2; ++p) {
                const double2 v = *reinterpret_cast<const double2*>(pl + j * ROWS + p * (2 * RG));
                a[2 * p] = v.x;
                a[2 * p + 1] = v.y;
            }
            double2 pv[C];
#pragma unroll
            for (int c = 0; c < C; ++c) pv[c] = Pl[j * 10 + c];
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < C; ++c) acc[r][c] = rfma(a[r], pv[c], acc[r][c]);
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    double s = 0;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) s += acc[r][c].x + acc[r][c].y;
    if (s == 12345.0) out[0] = s;
}

template <int R, int C, int G>
void run(int warps, int sms) {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 8 * sms);
    const int iters = 400;
    loop<R, C, G><<<sms, 32 * warps>>>(5, out, cyc);
    loop<R, C, G><<<sms, 32 * warps>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    long long c0 = 0;
    cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
    const double dfma = 2.0 * R * C * 32 * iters * 32.0 * warps;  // lane DFMA per SM
    printf("R %d C %d G %d warps/SM %2d: %.1f DFMA/clk/SM (%.0f%%)\n", R, C, G, warps, dfma / c0,
           100.0 * dfma / c0 / 64);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {4, 8, 12}) run<4, 5, 2>(w, sms);
    for (int w : {4, 8, 12}) run<6, 5, 2>(w, sms);
    for (int w : {4, 8}) run<8, 5, 2>(w, sms);
    for (int w : {4, 8, 12}) run<4, 2, 5>(w, sms);
    for (int w : {4, 8}) run<8, 2, 5>(w, sms);
    for (int w : {4, 8}) run<10, 2, 5>(w, sms);
    return 0;
}
