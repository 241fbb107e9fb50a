// Shared-memory throughput microbenchmarks (not part of the library).
#include <cstdio>
#include <cuda_runtime.h>

// mode 0: LDS.128 broadcast (all lanes same address)
// mode 1: LDS.128 per-lane consecutive
// mode 2: LDS.64 per-lane consecutive
// mode 3: LDS.64 broadcast
// mode 4: LDS.128 two addresses per warp (half-warp broadcast)
template <int MODE>
__global__ void tp_lds(int iters, double* out) {
    __shared__ double2 buf[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, i + 1);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    const double* b64 = reinterpret_cast<const double*>(buf);
    for (int it = 0; it < iters; ++it) {
        const int base = (it * 64) & 1023;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (MODE == 0) { double2 v = buf[base + u]; acc0 += v.x; acc1 += v.y; }
            if (MODE == 1) { double2 v = buf[base + u * 32 + lane]; acc0 += v.x; acc1 += v.y; }
            if (MODE == 2) { double v = b64[base + u * 32 + lane]; acc0 += v; }
            if (MODE == 3) { double v = b64[base + u]; acc0 += v; }
            if (MODE == 4) { double2 v = buf[base + u * 2 + (lane >> 4)]; acc0 += v.x; acc1 += v.y; }
            if (MODE == 5) { double2 v = buf[base + u * 2 + (lane & 1)]; acc0 += v.x; acc1 += v.y; }
            if (MODE == 6) { double2 v = buf[base + u * 32 + (lane & 15)]; acc0 += v.x; acc1 += v.y; }
            if (MODE == 7) { double2 v = buf[base + u * 32 + (lane >> 1)]; acc0 += v.x; acc1 += v.y; }
        }
    }
    if (acc0 + acc1 + acc2 + acc3 == 1234.5) out[0] = acc0;
}

// DFMA throughput with interleaved broadcast LDS.128 (ratio r loads per 4 DFMA)
__global__ void tp_mix(int iters, int nld, double* out) {
    __shared__ double2 buf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_double2(i, i + 1);
    __syncthreads();
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
    double x = 0.999;
    for (int it = 0; it < iters; ++it) {
        double2 p = buf[(it * 3) & 1023];
        x = p.x * 1e-300 + 0.999;
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = fma(a[u], x, 1e-9);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 1234.5) out[0] = s;
}

int main() {
    double* out;
    cudaMalloc(&out, 64);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 20000, threads = 512, blocks = sms * 2;
#define TP(MODE, name)                                                                  \
    {                                                                                   \
        tp_lds<MODE><<<blocks, threads>>>(100, out);                                    \
        cudaEventRecord(a);                                                             \
        tp_lds<MODE><<<blocks, threads>>>(iters, out);                                  \
        cudaEventRecord(b);                                                             \
        cudaEventSynchronize(b);                                                        \
        float ms;                                                                       \
        cudaEventElapsedTime(&ms, a, b);                                                \
        double warp_loads = (double)iters * 8 * blocks * threads / 32;                  \
        double per_sm_per_cyc = warp_loads / sms / (ms * 1e-3 * clk * 1e3);             \
        printf("%-36s %.3f warp-loads / SM / cycle (clock %d MHz nominal)\n", name,     \
               per_sm_per_cyc, clk / 1000);                                             \
    }
    TP(0, "LDS.128 broadcast");
    TP(1, "LDS.128 per-lane");
    TP(2, "LDS.64 per-lane");
    TP(3, "LDS.64 broadcast");
    TP(4, "LDS.128 two addresses (half-warps)");
    TP(5, "LDS.128 two addresses (odd/even)");
    TP(6, "LDS.128 16 distinct (lane&15)");
    TP(7, "LDS.128 16 distinct (lane>>1)");
    return 0;
}
