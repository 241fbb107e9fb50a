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

__host__ __device__ inline size_t rqh_warp_smem(int nb, int m) {
    const int L = m + 1;
    return (size_t)L * nb * 16 + (size_t)nb * L * 16 + (size_t)nb * 16;
}

// LMAX >= m+1, <= 32.  LFIX > 0 fixes L = m+1 at compile time (exact,
// predicate-free unrolling for the common m); LFIX = 0 reads it at run time.
template <int LMAX, int LFIX = 0>
__global__ void __launch_bounds__(128)
    k_rq_house(RqDims d, const double2* __restrict__ Z2, double2* __restrict__ Pbuf) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int l = blockIdx.x * (blockDim.x >> 5) + warp;
    if (l >= d.sb) return;
    const int nb = d.nb;
    const int L = LFIX > 0 ? LFIX : d.m + 1;
    const int m = L - 1;
    double2* Win = (double2*)(smem + (size_t)warp * rqh_warp_smem(nb, m));  // [L slots][nb rows]
    double2* U = Win + (size_t)L * nb;                                       // [nb][L]
    double2* Tau = U + (size_t)nb * L;                                       // [nb]
    const double2 sig = d.shifts[l];
    const int arow0 = d.k - nb;  // A row of block row 0

    // initial window: columns nb-1 .. nb-1+m  (Z1 column nb-1 and the m Z2 columns)
    {
        double2* dst = Win + (size_t)((nb - 1) % L) * nb;
        const double* src = d.A + arow0 + (int64_t)(d.c0 + nb - 1) * d.lda;
        for (int i = lane; i < nb; i += 32) {
            double2 v = make_double2(src[i], 0.0);
            if (i + m == nb - 1) v = csub(v, sig);  // lazy -sigma on Ahat's diagonal
            dst[i] = v;
        }
    }
    for (int c = 0; c < m; ++c) {
        const int j = nb + c;
        double2* dst = Win + (size_t)(j % L) * nb;
        const double2* src = Z2 + ((int64_t)l * m + c) * d.LDZ + d.r0;
        for (int i = lane; i < nb; i += 32) dst[i] = src[i];
    }
    // prefetch of the panel column entering next (rows lane, lane+32)
    double pf0 = 0.0, pf1 = 0.0;
    auto prefetch = [&](int j) {  // column j, rows 0..j
        const double* src = d.A + arow0 + (int64_t)(d.c0 + j) * d.lda;
        pf0 = (lane <= j) ? src[lane] : 0.0;
        pf1 = (lane + 32 <= j) ? src[lane + 32] : 0.0;
    };
    if (nb >= 2) prefetch(nb - 2);
    __syncwarp();

    for (int t = nb - 1; t >= 0; --t) {
        const int base = t % L;  // slot of column t; column t+j sits in slot (base+j) mod L
        // ---- every lane builds the reflector of row t from broadcast loads ----
        double2 y[LMAX];
        double s2a = 0.0, s2b = 0.0;
#pragma unroll
        for (int j = 0; j < LMAX; ++j) {
            if (j < L) {
                int sj = base + j;
                if (sj >= L) sj -= L;
                const double2 x = Win[(size_t)sj * nb + t];
                y[j] = make_double2(x.x, -x.y);  // conj(row t)
                if (j < L - 1) {
                    if (j & 1) s2b = fma(y[j].x, y[j].x, fma(y[j].y, y[j].y, s2b));
                    else s2a = fma(y[j].x, y[j].x, fma(y[j].y, y[j].y, s2a));
                }
            }
        }
        double2 alpha = cz();
#pragma unroll
        for (int j = 0; j < LMAX; ++j)
            if (j == L - 1) alpha = y[j];
        const double s2 = s2a + s2b;
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
        for (int j = 0; j < LMAX; ++j) uu[j] = (j < L - 1) ? cmul(y[j], scale) : (j == L - 1 ? make_double2(1.0, 0.0) : cz());
        if (lane < L) {
#pragma unroll
            for (int j = 0; j < LMAX; ++j)
                if (j == lane) U[(size_t)t * L + j] = uu[j];
        }
        if (lane == 0) Tau[t] = tau;
        // ---- rows 0..t-1 (lanes own rows lane, lane+32): z <- z - tau (z u) u^H ----
        const bool act = t > 0 && (tau.x != 0.0 || tau.y != 0.0);
        if (act) {
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const int i = lane + 32 * rr;
                if (rr == 1 && nb <= 32) break;
                if (i < t) {
                    double2 z[LMAX];
                    double2 w0 = cz(), w1 = cz();
#pragma unroll
                    for (int j = 0; j < LMAX; ++j) {
                        if (j < L) {
                            int sj = base + j;
                            if (sj >= L) sj -= L;
                            z[j] = Win[(size_t)sj * nb + i];
                            if (j & 1) w1 = cfma(z[j], uu[j], w1);
                            else w0 = cfma(z[j], uu[j], w0);
                        }
                    }
                    const double2 tw = cmul(tau, cadd(w0, w1));
#pragma unroll
                    for (int j = 0; j < LMAX; ++j) {
                        if (j < L) {
                            // z_j -= tau w conj(u_j)
                            const double2 cu = make_double2(uu[j].x, -uu[j].y);
                            int sj = base + j;
                            if (sj >= L) sj -= L;
                            Win[(size_t)sj * nb + i] = csub(z[j], cmul(tw, cu));
                        }
                    }
                }
            }
        }
        // ---- slide: column t+m retires, panel column t-1 enters its slot ----
        if (t > 0) {
            const int sl = base == 0 ? L - 1 : base - 1;  // slot of column t-1
            double2* dst = Win + (size_t)sl * nb;
            const int j = t - 1;
            double2 v0 = make_double2(pf0, 0.0), v1 = make_double2(pf1, 0.0);
            if (lane + m == j) v0 = csub(v0, sig);
            if (lane + 32 + m == j) v1 = csub(v1, sig);
            if (lane <= j) dst[lane] = v0;
            if (lane + 32 <= j) dst[lane + 32] = v1;
            if (t >= 2) prefetch(t - 2);
        }
        __syncwarp();
    }

    // ---- reverse accumulation in registers: lane cc owns column cc of W ----
    double2* dstP = Pbuf + (int64_t)l * d.nc * m;  // j-major: P[j*m + cc]
    for (int cc0 = 0; cc0 < m; cc0 += 32) {
        const int cc = cc0 + lane;
        double2 w[LMAX];
#pragma unroll
        for (int j = 0; j < LMAX; ++j) w[j] = make_double2((j == cc) ? 1.0 : 0.0, 0.0);
        for (int t = 0; t < nb; ++t) {
            const double2 tau = Tau[t];
            double2 dd0 = cz(), dd1 = cz();
#pragma unroll
            for (int j = 0; j < LMAX; ++j) {
                if (j < L) {
                    const double2 uj = U[(size_t)t * L + j];
                    const double2 cu = make_double2(uj.x, -uj.y);
                    if (j & 1) dd1 = cfma(cu, w[j], dd1);
                    else dd0 = cfma(cu, w[j], dd0);
                }
            }
            const double2 td = cmul(tau, cadd(dd0, dd1));
#pragma unroll
            for (int j = 0; j < LMAX; ++j)
                if (j < L) w[j] = csub(w[j], cmul(U[(size_t)t * L + j], td));
            if (cc < m) dstP[(size_t)t * m + cc] = w[0];
#pragma unroll
            for (int j = 0; j < LMAX - 1; ++j) w[j] = w[j + 1];
            w[LMAX - 1] = cz();
        }
        // rows nb .. nb+m-1 remain in the window
        if (cc < m) {
#pragma unroll
            for (int j = 0; j < LMAX; ++j)
                if (j < m) dstP[(size_t)(nb + j) * m + cc] = w[j];
        }
    }
}

}  // namespace ssd
