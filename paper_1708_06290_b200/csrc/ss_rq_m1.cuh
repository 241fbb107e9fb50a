// Window block RQ for m = 1 (the pseudospectrum case, config 3: 10 000
// shifts), laid out for throughput instead of latency.
//
// Same math as k_rq_house (ss_rq_house.cuh) for L = 2 -- row Householder
// reflectors bottom-up, kernels.py:74-99's sign rule, here in the
// unnormalised form H = I - kappa v v^H of k_block -- but with m = 1 a row's
// active window is (panel entry of column t, one carried value), so the
// whole state of a 64-row window is 64 complex numbers per shift.  Eight
// lanes per shift hold 8 rows each IN REGISTERS (a warp = 4 shifts); per
// step the pivot's carried value is shuffled within the 8-lane group and
// every lane updates its 8 rows -- independent work beside the serial
// reflector chain, instead of one latency-bound warp per shift.
//
// P (the first column of the window's unitary, nb + 1 entries) is built
// row-wise beside the chain, as k_block's m <= 6 path: row r of P is
// e_r^T H_{nb-1} ... H_0 restricted to column 0, i.e. the same row update
// applied to e_r from step r on; a data row retires exactly when it is the
// pivot, so every register row is live for all steps (data row while t > i,
// row i of P from t = i on) and no reflector is stored.  One extra register
// row (on the last lane of the group) is P's row nb (the old carried column).
//
// The staged panel column t already holds each row's window entry of that
// step: A(i, t) for data rows (i < t), 1 for the pivot row (row t of P
// starts as e_t), 0 below (rows of P have no entry left of their column);
// the pivot's own entry A(t, t) is kept aside, and the per-shift lazy -sigma
// (row t - 1 only) is a correction on one static register slot per step.
#pragma once

#include "ss_rq_house.cuh"

namespace ssd {

constexpr int kM1Warps = 4;  // warps per CTA; 4 shifts per warp (8 lanes x 8 rows each)
constexpr int kM1Ld = 72;    // padded panel column: lane q's rows start at 9 q (conflict-free)

__global__ void __launch_bounds__(32 * kM1Warps)
    k_rq_m1(RqDims d, const double2* __restrict__ Z2, double2* __restrict__ Pbuf) {
    __shared__ double Ap[64 * kM1Ld];  // Ap[t * kM1Ld + 9 q + j]: window entry of row 8 q + j at step t
    __shared__ double Dg[64];          // A(t, t)
    const int nb = d.nb;               // <= 64
    const int64_t arow0 = (int64_t)d.k - nb;
    {
        // nb x 64 panel entries, column-major reads (coalesced), 8 loads in flight per thread
        const int n = nb * 64;
        for (int v0 = threadIdx.x; v0 < n; v0 += 8 * blockDim.x) {
            double val[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int v = v0 + u * blockDim.x;
                const int t = v >> 6, i = v & 63;
                val[u] = (v < n && i <= t) ? d.A[arow0 + i + (int64_t)(d.c0 + t) * d.lda] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int v = v0 + u * blockDim.x;
                if (v < n) {
                    const int t = v >> 6, i = v & 63;
                    if (i == t) Dg[t] = val[u];
                    Ap[t * kM1Ld + (i >> 3) * 9 + (i & 7)] = i == t ? 1.0 : val[u];
                }
            }
        }
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = lane & 7;  // rows 8 q .. 8 q + 7
    const int lq = (blockIdx.x * kM1Warps + warp) * 4 + (lane >> 3);
    const bool valid = lq < d.sb;
    const int l = valid ? lq : d.sb - 1;
    const double2 sig = d.shifts[l];
    const double2* z2 = Z2 + (int64_t)l * d.LDZ + d.r0;
    double2 c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int i = q * 8 + j;
        c[j] = i < nb ? z2[i] : cz();
    }
    double2 cx = make_double2(q == 7 ? 1.0 : 0.0, 0.0);  // P row nb (x-row e_nb)
    const int src0 = lane & ~7;

    for (int tq = (nb - 1) >> 3; tq >= 0; --tq) {
#pragma unroll
        for (int jj = 7; jj >= 0; --jj) {
            const int t = tq * 8 + jj;
            if (t >= nb) continue;  // warp-uniform
            // pivot row t: panel entry p0 (never shifted: the lazy -sigma of
            // column t sits in row t - 1) and its carried value p1
            const double p0 = Dg[t];
            double2 p1;
            p1.x = __shfl_sync(0xffffffffu, c[jj].x, src0 | tq);
            p1.y = __shfl_sync(0xffffffffu, c[jj].y, src0 | tq);
            if (q == tq) c[jj] = cz();  // row t of P starts as (1, 0)
            // reflector of y = conj(p0, p1): v = (p0, alpha - beta), kappa
            const double2 alpha = make_double2(p1.x, -p1.y);
            const double s2 = p0 * p0;
            const bool ident = s2 == 0.0 && alpha.y == 0.0;
            const double nrm2 = ident ? 1.0 : fma(alpha.x, alpha.x, fma(alpha.y, alpha.y, s2));
            const double rn = rsqrt_pos(nrm2);
            const double sg = alpha.x >= 0.0 ? -1.0 : 1.0;
            const double beta = sg * nrm2 * rn, ib = sg * rn;
            const double zx = beta - alpha.x;
            const double f = ib * rcp_pos(fma(zx, zx, alpha.y * alpha.y));
            const double2 kap = ident ? cz() : make_double2(zx * f, -alpha.y * f);
            const double2 vl = make_double2(alpha.x - beta, alpha.y);
            const double* acol = Ap + t * kM1Ld + q * 9;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const double a = acol[j];
                const double2 cc = c[j];
                double2 dot;
                dot.x = fma(a, p0, fma(cc.x, vl.x, -cc.y * vl.y));
                dot.y = fma(cc.x, vl.y, cc.y * vl.x);
                const double2 tw = cmul(kap, dot);
                // new carried value: the row's column-t entry after H_t
                c[j] = make_double2(fma(-tw.x, p0, a), -tw.y * p0);
            }
            {
                const double2 dot = cmul(cx, vl);
                const double2 tw = cmul(kap, dot);
                cx = make_double2(-tw.x * p0, -tw.y * p0);
            }
            // lazy -sigma on row t - 1's entry of column t: its new value is
            // affine in that entry, so the shift enters as -sigma (1 - kappa p0^2)
            if (t >= 1) {
                const int jl = (jj + 7) & 7;           // slot of row t - 1 (static)
                const int ql = jj == 0 ? tq - 1 : tq;  // its lane (warp-uniform)
                if (q == ql) {
                    const double2 g = make_double2(1.0 - kap.x * p0 * p0, -kap.y * p0 * p0);
                    c[jl] = csub(c[jl], cmul(sig, g));
                }
            }
        }
    }
    if (valid) {
        double2* P = Pbuf + (int64_t)l * d.nc;  // nc = nb + 1, P[r] (m = 1)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int i = q * 8 + j;
            if (i < nb) P[i] = c[j];
        }
        if (q == 7) P[nb] = cx;
    }
}

}  // namespace ssd
