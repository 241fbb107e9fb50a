// Block RQ of the window step by row Householder reflectors, one warp per
// shift (the B200 replacement of the reference's scheduled Givens batch,
// batched.py:64-122 / PAPER.md Alg. 8).
//
// The block Zb = [Z1 | Z2_l] (nb x (nb+m), upper trapezoid) is reduced
// bottom-up: for row t = nb-1..0 a reflector H_t acting on the m+1 columns
// t..t+m maps row t to (0,..,0,beta) (zlarfg convention on y = conj(row),
// pivot last; same sign rule as kernels.py:74-99).  Only m+1 columns are
// ever active: column t+m is final after step t (R is not needed) and
// column t-1 enters, so the warp keeps a sliding (m+1)-column window in
// shared memory instead of the whole block.  Then
//     P* = H_{nb-1} ... H_0,   P*[:, 0:m] = H_{nb-1}(...(H_0 E))
// is accumulated with lanes = columns of W; H_t touches rows t..t+m of W,
// a window that slides by one row per step, so each lane keeps its window in
// registers and retires one final row of P per step.  Results equal the
// Givens RQ's up to an m x m unitary on the active columns, which leaves
// G(sigma) unchanged (the head RQ is unique up to phases).
//
// Latency per step: one warp reduction (5 shuffle levels), two rsqrt, an
// (m+1)-term dot product per row, no CTA barriers.
#pragma once

#include "ss_device.cuh"

namespace ssd {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double2 shfl2(double2 v, int src) {
    return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

struct RqDims {
    int m, ptop, nb, k, c0, r0, nc, sb;
    const double* A;
    int64_t lda;
    const double2* shifts;
    int64_t LDZ;
};

// shared memory of one k_rq_house block (one shift): pivot buffers, U, tau
__host__ __device__ inline size_t rqh_warp_smem(int nb, int m) {
    const int L = m + 1;
    return (size_t)2 * 32 * 16 + (size_t)nb * L * 16 + (size_t)nb * 16;
}

// Two warps per shift block, thread i owns block row i (nb <= 64) and keeps
// that row's active window r[j] = Z(i, t + j), j = 0..m, in REGISTERS: the
// window slides by one column per step (column t+m retires, panel column
// t-1 -- prefetched from global one step ahead -- enters), so the only
// shared-memory traffic per step is the pivot row t, published by its
// owner (double-buffered: one barrier per step).  Every thread rebuilds the
// reflector of row t from the broadcast (no shuffles), updates its own row
// (z <- z - tau (z u) u^H) and shifts its window.  The reverse accumulation
// (lanes = columns of W, registers) runs on warp 0.
// LMAX >= m+1, <= 32; LFIX > 0 fixes L = m+1 at compile time.
template <int LMAX, int LFIX = 0>
__global__ void __launch_bounds__(64)
    k_rq_house(RqDims d, const double2* __restrict__ Z2, double2* __restrict__ Pbuf) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int l = blockIdx.x;
    const int nb = d.nb;
    const int L = LFIX > 0 ? LFIX : d.m + 1;
    const int m = L - 1;
    double2* Piv = (double2*)smem;           // [2][LMAX] pivot row broadcast
    double2* U = Piv + 2 * LMAX;             // [nb][L]
    double2* Tau = U + (size_t)nb * L;       // [nb]
    const double2 sig = d.shifts[l];
    const int arow0 = d.k - nb;  // A row of block row 0
    const int i = 32 * warp + lane;  // this thread's block row
    const bool live = i < nb;

    // initial window of row i: columns nb-1 .. nb-1+m
    double2 r[LMAX];
#pragma unroll
    for (int j = 0; j < LMAX; ++j) r[j] = cz();
    if (live) {
        double2 v = make_double2(d.A[arow0 + i + (int64_t)(d.c0 + nb - 1) * d.lda], 0.0);
        if (i + m == nb - 1) v = csub(v, sig);  // lazy -sigma on Ahat's diagonal
        r[0] = v;
        const double2* z2 = Z2 + (int64_t)l * m * d.LDZ + d.r0 + i;
#pragma unroll
        for (int j = 1; j < LMAX; ++j)
            if (j < L) r[j] = z2[(int64_t)(j - 1) * d.LDZ];
    }
    double pf = 0.0;  // row i of the panel column entering next
    if (nb >= 2 && i <= nb - 2) pf = d.A[arow0 + i + (int64_t)(d.c0 + nb - 2) * d.lda];

    for (int t = nb - 1; t >= 0; --t) {
        double2* piv = Piv + (t & 1) * LMAX;
        if (i == t) {
#pragma unroll
            for (int j = 0; j < LMAX; ++j)
                if (j < L) piv[j] = r[j];
        }
        __syncthreads();
        // ---- reflector of row t (every thread, from the broadcast) ----
        double2 y[LMAX];
#pragma unroll
        for (int j = 0; j < LMAX; ++j) {
            if (j < L) {
                const double2 x = piv[j];
                y[j] = make_double2(x.x, -x.y);  // conj(row t)
            } else {
                y[j] = cz();
            }
        }
        double sq[LMAX];
#pragma unroll
        for (int j = 0; j < LMAX; ++j) sq[j] = (j < L - 1) ? fma(y[j].x, y[j].x, y[j].y * y[j].y) : 0.0;
#pragma unroll
        for (int w = 1; w < LMAX; w <<= 1)  // tree sum
#pragma unroll
            for (int j = 0; j + w < LMAX; j += 2 * w) sq[j] += sq[j + w];
        const double s2 = sq[0];
        double2 alpha = cz();
#pragma unroll
        for (int j = 0; j < LMAX; ++j)
            if (j == L - 1) alpha = y[j];
        double2 tau = cz(), scale = cz();
        if (!(s2 == 0.0 && alpha.y == 0.0)) {
            const double nrm2 = fma(alpha.x, alpha.x, fma(alpha.y, alpha.y, s2));
            const double rn = rsqrt(nrm2);
            const double sg = alpha.x >= 0.0 ? -1.0 : 1.0;
            const double beta = sg * nrm2 * rn;  // -sign(Re alpha) ||y||
            const double ib = sg * rn;           // 1 / beta
            tau = make_double2(1.0 - alpha.x * ib, -alpha.y * ib);  // (beta - alpha) / beta
            const double zx = alpha.x - beta, zy = alpha.y;
            const double rz = rsqrt(fma(zx, zx, zy * zy));
            const double iz = rz * rz;
            scale = make_double2(zx * iz, -zy * iz);  // 1 / (alpha - beta)
        }
        double2 uu[LMAX];
#pragma unroll
        for (int j = 0; j < LMAX; ++j)
            uu[j] = (j < L - 1) ? cmul(y[j], scale) : (j == L - 1 ? make_double2(1.0, 0.0) : cz());
        if (warp == 0) {
            // select (not branch) this lane's entry: a per-lane branch here
            // compiles to an 11-way divergent switch
            double2 mine = cz();
#pragma unroll
            for (int j = 0; j < LMAX; ++j) mine = (j == lane) ? uu[j] : mine;
            if (lane < L) U[(size_t)t * L + lane] = mine;
            if (lane == 0) Tau[t] = tau;
        }
        // ---- own row (i < t): r <- r - tau (r u) u^H ----
        if (i < t) {
            double2 wp[LMAX];
#pragma unroll
            for (int j = 0; j < LMAX; ++j) wp[j] = (j < L) ? cmul(r[j], uu[j]) : cz();
#pragma unroll
            for (int w = 1; w < LMAX; w <<= 1)  // tree sum
#pragma unroll
                for (int j = 0; j + w < LMAX; j += 2 * w) wp[j] = cadd(wp[j], wp[j + w]);
            const double2 tw = cmul(tau, wp[0]);
#pragma unroll
            for (int j = 0; j < LMAX; ++j)
                if (j < L) r[j] = csub(r[j], cmul(tw, make_double2(uu[j].x, -uu[j].y)));
        }
        // ---- slide: column t+m retires, panel column t-1 enters r[0] ----
#pragma unroll
        for (int j = LMAX - 1; j > 0; --j) r[j] = r[j - 1];
        if (t > 0) {
            double2 v = make_double2(pf, 0.0);
            if (i + m == t - 1) v = csub(v, sig);
            r[0] = v;
            if (t >= 2 && i <= t - 2) pf = d.A[arow0 + i + (int64_t)(d.c0 + t - 2) * d.lda];
        }
    }
    __syncthreads();  // U / Tau complete

    // ---- reverse accumulation in registers (warp 0): lane cc owns column cc ----
    if (warp != 0) return;
    double2* dstP = Pbuf + (int64_t)l * d.nc * m;  // j-major: P[j*m + cc]
    for (int cc0 = 0; cc0 < m; cc0 += 32) {
        const int cc = cc0 + lane;
        double2 w[LMAX];
#pragma unroll
        for (int j = 0; j < LMAX; ++j) w[j] = make_double2((j == cc) ? 1.0 : 0.0, 0.0);
        for (int t = 0; t < nb; ++t) {
            const double2 tau = Tau[t];
            double2 dp[LMAX];
#pragma unroll
            for (int j = 0; j < LMAX; ++j) {
                if (j < L) {
                    const double2 uj = U[(size_t)t * L + j];
                    dp[j] = cmul(make_double2(uj.x, -uj.y), w[j]);
                } else {
                    dp[j] = cz();
                }
            }
#pragma unroll
            for (int s = 1; s < LMAX; s <<= 1)
#pragma unroll
                for (int j = 0; j + s < LMAX; j += 2 * s) dp[j] = cadd(dp[j], dp[j + s]);
            const double2 td = cmul(tau, dp[0]);
#pragma unroll
            for (int j = 0; j < LMAX; ++j)
                if (j < L) w[j] = csub(w[j], cmul(U[(size_t)t * L + j], td));
            if (cc < m) dstP[(size_t)t * m + cc] = w[0];
#pragma unroll
            for (int j = 0; j < LMAX - 1; ++j) w[j] = w[j + 1];
            w[LMAX - 1] = cz();
        }
        if (cc < m) {
#pragma unroll
            for (int j = 0; j < LMAX; ++j)
                if (j < m) dstP[(size_t)(nb + j) * m + cc] = w[j];
        }
    }
}

}  // namespace ssd
