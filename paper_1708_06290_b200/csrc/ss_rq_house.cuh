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

// One warp per shift block: lane owns block rows lane and lane+32 (nb <= 64)
// and keeps each row's active window r[j] = Z(i, t + j), j = 0..m, in
// REGISTERS; the window slides by one column per step (column t+m retires,
// panel column t-1 -- prefetched from global one step ahead -- enters).
// Per step the owner lane publishes the pivot row t in shared memory
// (double-buffered, __syncwarp only), every lane rebuilds the reflector of
// row t from the broadcast (computed once per block, no shuffles), updates
// its rows (z <- z - tau (z u) u^H) and shifts its windows.  The reverse
// accumulation (lanes = columns of W, registers) follows on the same warp.
// LMAX >= m+1, <= 32; LFIX > 0 fixes L = m+1 at compile time.
template <int LMAX>
__device__ __forceinline__ void rq_row_update(double2 (&r)[LMAX], const double2 (&uu)[LMAX],
                                              double2 tau, int L) {
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
        if (j < L) {
            // r_j -= tw conj(u_j)
            r[j].x = fma(-tw.x, uu[j].x, fma(-tw.y, uu[j].y, r[j].x));
            r[j].y = fma(-tw.y, uu[j].x, fma(tw.x, uu[j].y, r[j].y));
        }
}

template <int LMAX, int LFIX = 0>
__global__ void __launch_bounds__(32)
    k_rq_house(RqDims d, const double2* __restrict__ Z2, double2* __restrict__ Pbuf) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int l = blockIdx.x;
    const int nb = d.nb;
    const int L = LFIX > 0 ? LFIX : d.m + 1;
    const int m = L - 1;
    double2* Piv = (double2*)smem;           // [2][LMAX] pivot row broadcast
    double2* U = Piv + 2 * LMAX;             // [nb][L]
    double2* Tau = U + (size_t)nb * L;       // [nb]
    const double2 sig = d.shifts[l];
    const int arow0 = d.k - nb;  // A row of block row 0
    const int i0 = lane, i1 = lane + 32;

    // initial windows: columns nb-1 .. nb-1+m
    double2 ra[LMAX], rb[LMAX];
#pragma unroll
    for (int j = 0; j < LMAX; ++j) ra[j] = rb[j] = cz();
    {
        const double* a0 = d.A + arow0 + (int64_t)(d.c0 + nb - 1) * d.lda;
        const double2* z2 = Z2 + (int64_t)l * m * d.LDZ + d.r0;
        if (i0 < nb) {
            double2 v = make_double2(a0[i0], 0.0);
            if (i0 + m == nb - 1) v = csub(v, sig);  // lazy -sigma on Ahat's diagonal
            ra[0] = v;
#pragma unroll
            for (int j = 1; j < LMAX; ++j)
                if (j < L) ra[j] = z2[(int64_t)(j - 1) * d.LDZ + i0];
        }
        if (i1 < nb) {
            double2 v = make_double2(a0[i1], 0.0);
            if (i1 + m == nb - 1) v = csub(v, sig);
            rb[0] = v;
#pragma unroll
            for (int j = 1; j < LMAX; ++j)
                if (j < L) rb[j] = z2[(int64_t)(j - 1) * d.LDZ + i1];
        }
    }
    double pfa = 0.0, pfb = 0.0;  // rows i0, i1 of the panel column entering next
    if (nb >= 2) {
        const double* an = d.A + arow0 + (int64_t)(d.c0 + nb - 2) * d.lda;
        if (i0 <= nb - 2) pfa = an[i0];
        if (i1 <= nb - 2) pfb = an[i1];
    }

    for (int t = nb - 1; t >= 0; --t) {
        double2* piv = Piv + (t & 1) * LMAX;
        if (i0 == t) {
#pragma unroll
            for (int j = 0; j < LMAX; ++j)
                if (j < L) piv[j] = ra[j];
        }
        if (i1 == t) {
#pragma unroll
            for (int j = 0; j < LMAX; ++j)
                if (j < L) piv[j] = rb[j];
        }
        __syncwarp();
        // ---- reflector of row t (every lane, from the broadcast) ----
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
        {
            // select (not branch) this lane's entry: a per-lane branch here
            // compiles to an L-way divergent switch
            double2 mine = cz();
#pragma unroll
            for (int j = 0; j < LMAX; ++j) mine = (j == lane) ? uu[j] : mine;
            if (lane < L) U[(size_t)t * L + lane] = mine;
            if (lane == 0) Tau[t] = tau;
        }
        // ---- own rows below the pivot's column range: i < t ----
        if (i0 < t) rq_row_update<LMAX>(ra, uu, tau, L);
        if (t > 32 && i1 < t) rq_row_update<LMAX>(rb, uu, tau, L);
        // ---- slide: column t+m retires, panel column t-1 enters r[0] ----
#pragma unroll
        for (int j = LMAX - 1; j > 0; --j) {
            ra[j] = ra[j - 1];
            rb[j] = rb[j - 1];
        }
        if (t > 0) {
            double2 va = make_double2(pfa, 0.0), vb = make_double2(pfb, 0.0);
            if (i0 + m == t - 1) va = csub(va, sig);
            if (i1 + m == t - 1) vb = csub(vb, sig);
            ra[0] = va;
            rb[0] = vb;
            if (t >= 2) {
                const double* an = d.A + arow0 + (int64_t)(d.c0 + t - 2) * d.lda;
                if (i0 <= t - 2) pfa = an[i0];
                if (i1 <= t - 2) pfb = an[i1];
            }
        }
    }
    __syncwarp();  // U / Tau complete

    // ---- reverse accumulation in registers: lane cc owns column cc ----
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
