// Two-level window sweep: the fused outer-block kernel.
//
// The reference sweep (solvers.py:165-200, Alg. 6) walks windows of
// nb panel columns; after every window every shift's state rows [0, r0) are
// updated with that window's P_l ((nb+m) x m).  Per updated row that costs
// 4 m nb (real panel x P12) + 8 m^2 (state x P22) flops, so the state part is
// a 2m/nb overhead on the algorithmic work -- 31% at nb = 64, m = 10.
//
// Here the windows are grouped into outer blocks of NB = 128 columns; per
// outer block one kernel per shift (k_block below, one warp per shift so all
// shifts' serial reflector chains are resident at once) runs the NB/32 inner
// windows (nb = 32):
//   * inner window i (rows [b, b + 32) of the block, lane = row): row
//     Householder chain (same scheme and sign rule as ss_rq_house.cuh /
//     kernels.py:74-99), then P_i by reverse accumulation (a lane pair per
//     column, in rounds of 16 columns);
//   * P_i is applied row pass by row pass: rows above the inner window get
//     state <- state P22 + A(row, inner cols) P12 - sigma P12[lazy row]
//     (solvers.py:186-199 restricted to the block); the window's own rows
//     are finished and become rows of the composite
//         W <- E_b P12 + W P22,    W = [W_panel (NBo x m); W22 (m x m)]
//     so that after the outer block the far rows [0, r0_out) need ONE update
//         state <- state W22 + Pan(:, outer cols) W_panel - sigma W[lazy row]
//     (k_far, ss_far.cuh, in 64-column passes: the first with W22, the rest
//     with the identity).  The state overhead on the far rows drops to 2m/NB.
// The block's state rows stay in the (L2-resident) window buffer between
// phases; only W ((NBo + m) x m per shift, j-major) is the kernel's product.
#pragma once

#include "ss_rq_house.cuh"
#include "ss_update_ws.cuh"

namespace ssd {

constexpr int kBlkNB = 128;   // outer block (rows per CTA = threads)
constexpr int kBlkInner = 32; // inner window (one warp)
#ifndef SS_BLK_MINB
#define SS_BLK_MINB 4  // resident CTAs per SM the register budget targets
#endif

struct BlkDims {
    int m, ptop, k, NBo;  // outer block: A rows [k-NBo, k), panel cols [c0, c0+NBo)
    int c0, r0;           // r0 = ptop + k - NBo: first stacked row of the block
    const double* A;
    int64_t lda;
    const double2* shifts;
    int64_t LDZ;
    int64_t wstride;  // elements (complex) per shift in W
};

__host__ __device__ inline size_t blk_smem_bytes_1(int m) {
    const int L = m + 1;
    size_t b = 0;
    b += (size_t)(kBlkInner + m) * m * 16;  // P
    b += (size_t)kBlkInner * L * 16;        // U
    b += (size_t)kBlkInner * 16;            // Tau
    b += (size_t)2 * 32 * 16;               // pivot broadcast
    b += (size_t)m * m * 16;                // W22
    return b;
}

constexpr int kBlkShiftsPerWarp = 1;  // 2 measured slower on B200 (per-warp issue bound)

__host__ __device__ inline size_t blk_smem_bytes(int m) {
    return kBlkShiftsPerWarp * blk_smem_bytes_1(m);
}

// Row update of the chain with FMA-chain dot products (two partial sums, no
// add tree): z <- z - tau (z u) u^H over the L-column window.
template <int L>
__device__ __forceinline__ void blk_row_update(double2 (&z)[L], const double2* __restrict__ u,
                                               double2 tau) {
    double2 d0 = cz(), d1 = cz();
#pragma unroll
    for (int j = 0; j < L; ++j) {
        const double2 uj = u[j];
        double2& d = (j & 1) ? d1 : d0;
        d.x = fma(z[j].x, uj.x, d.x);
        d.x = fma(-z[j].y, uj.y, d.x);
        d.y = fma(z[j].x, uj.y, d.y);
        d.y = fma(z[j].y, uj.x, d.y);
    }
    const double2 tw = cmul(tau, cadd(d0, d1));
#pragma unroll
    for (int j = 0; j < L; ++j) {
        const double2 uj = u[j];
        z[j].x = fma(-tw.x, uj.x, fma(-tw.y, uj.y, z[j].x));
        z[j].y = fma(-tw.y, uj.x, fma(tw.x, uj.y, z[j].y));
    }
}

// One warp per NSW shifts.  Block row t of the outer block is handled by
// lane (t + 128 - NBo) & 31 in pass (t + 128 - NBo) >> 5 in every phase, so
// the inner window i is pass 3 - i, the state rows above it are passes
// < 3 - i and the W rows below it passes > 3 - i; a row never changes lanes,
// so its values can stay in the (L2-resident) window buffer Z / the W output
// between phases without cross-lane hazards.
//
// The reflector chain is a serial dependency: a warp running one shift's
// chain is latency-bound (measured ~3.7 cycles per instruction).  Each warp
// therefore carries NSW = 2 shifts through identical control flow (the row
// mapping does not depend on the shift), so every phase issues two
// independent instruction streams back to back and the second hides the
// first's latencies; all shifts' chains stay resident (15 KB of shared
// memory per shift).
//
// NSW independent row updates with the shift index innermost, so the two
// dependency chains interleave instruction by instruction.
template <int L, int NSW>
__device__ __forceinline__ void blk_row_update_n(double2 (&z)[NSW][L], double2* const (&U)[NSW],
                                                 int off, const double2 (&tau)[NSW]) {
    double2 d0[NSW], d1[NSW];
#pragma unroll
    for (int q = 0; q < NSW; ++q) d0[q] = d1[q] = cz();
#pragma unroll
    for (int j = 0; j < L; ++j) {
#pragma unroll
        for (int q = 0; q < NSW; ++q) {
            const double2 uj = U[q][off + j];
            double2& dd = (j & 1) ? d1[q] : d0[q];
            dd.x = fma(z[q][j].x, uj.x, dd.x);
            dd.y = fma(z[q][j].x, uj.y, dd.y);
        }
#pragma unroll
        for (int q = 0; q < NSW; ++q) {
            const double2 uj = U[q][off + j];
            double2& dd = (j & 1) ? d1[q] : d0[q];
            dd.x = fma(-z[q][j].y, uj.y, dd.x);
            dd.y = fma(z[q][j].y, uj.x, dd.y);
        }
    }
    double2 tw[NSW];
#pragma unroll
    for (int q = 0; q < NSW; ++q) tw[q] = cmul(tau[q], cadd(d0[q], d1[q]));
#pragma unroll
    for (int j = 0; j < L; ++j) {
#pragma unroll
        for (int q = 0; q < NSW; ++q) {
            const double2 uj = U[q][off + j];
            z[q][j].x = fma(-tw[q].x, uj.x, fma(-tw[q].y, uj.y, z[q][j].x));
            z[q][j].y = fma(-tw[q].y, uj.x, fma(tw[q].x, uj.y, z[q][j].y));
        }
    }
}

// After the chain, P_i = H_{nbi-1}(...(H_0 E)) by reverse accumulation:
// lane pair (2c, 2c+1) owns column c of P, each lane half of the sliding
// L-window (6 entries), so a step is 6 complex dot terms + one shuffle
// exchange.
template <int M, int NSW>
__global__ void __launch_bounds__(32, NSW == 1 ? 8 : 6)
    k_block(BlkDims d, double2* __restrict__ Z, double2* __restrict__ W, int sb) {
    constexpr int L = M + 1;
    constexpr int HW = (L + 1) / 2;  // window entries per lane of a column pair
    constexpr int CR = 16;           // columns per reverse-accumulation round (2 lanes each)
    static_assert(L <= 32, "k_block: m <= 31");
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int PSZ = (kBlkInner + M) * M, USZ = kBlkInner * L;
    constexpr int QSZ = PSZ + USZ + kBlkInner + 64 + M * M;  // complex per shift
    double2* P[NSW];
    double2* U[NSW];
    double2* Tau[NSW];
    double2* Piv[NSW];
    double2* W22[NSW];
    const int lane = threadIdx.x;
    const int NBo = d.NBo;
    const int off = kBlkNB - NBo;  // rows are numbered from the top of a 128-row frame
    const double* Ab = d.A + (int64_t)d.c0 * d.lda;  // panel column 0
    double2 sig[NSW];
    double2* Zl[NSW];
    double2* Wl[NSW];
    bool vq[NSW];
#pragma unroll
    for (int q = 0; q < NSW; ++q) {
        double2* base = reinterpret_cast<double2*>(smem) + q * QSZ;
        P[q] = base;
        U[q] = P[q] + PSZ;
        Tau[q] = U[q] + USZ;
        Piv[q] = Tau[q] + kBlkInner;
        W22[q] = Piv[q] + 64;
        const int lq = blockIdx.x * NSW + q;
        vq[q] = lq < sb;
        const int l = vq[q] ? lq : sb - 1;  // a missing partner shadows the last shift
        sig[q] = d.shifts[l];
        Zl[q] = Z + (int64_t)l * M * d.LDZ + d.r0;  // block row t, column c: Zl[c*LDZ + t]
        Wl[q] = W + (int64_t)l * d.wstride;         // W row t, column c: Wl[t*M + c]
        for (int u = lane; u < M * M; u += 32)
            W22[q][u] = make_double2((u / M) == (u % M) ? 1.0 : 0.0, 0.0);
    }

    const int ni = (NBo + kBlkInner - 1) / kBlkInner;
    for (int i = 0; i < ni; ++i) {
        const int top = NBo - kBlkInner * i;  // rows [b, top) = inner block
        const int b = max(0, top - kBlkInner);
        const int nbi = top - b;
        const int pass_rq = 3 - i;
        {
            // ---------------- reflector chains over the inner block ----------------
            const int t = pass_rq * 32 + lane - off;  // this lane's block row
            const int rho = t - b;
            const bool mine = t >= 0 && rho >= 0;
            const int64_t arow = (int64_t)(d.k - NBo) + t;
            double2 z[NSW][L];  // window: z[0] = panel column, z[1..L) = state
            double pf = 0.0;
            {
                const double a0 = mine ? Ab[arow + (int64_t)(b + nbi - 1) * d.lda] : 0.0;
                if (mine && nbi >= 2 && rho <= nbi - 2) pf = Ab[arow + (int64_t)(b + nbi - 2) * d.lda];
#pragma unroll
                for (int q = 0; q < NSW; ++q) {
#pragma unroll
                    for (int c = 0; c < M; ++c) z[q][c + 1] = mine ? Zl[q][(int64_t)c * d.LDZ + t] : cz();
                    z[q][0] = make_double2(a0, 0.0);
                    if (mine && nbi - 1 == rho + M) z[q][0] = csub(z[q][0], sig[q]);
                }
            }
            for (int ti = nbi - 1; ti >= 0; --ti) {
                const int pb = (ti & 1) * 32;
                if (mine && rho == ti) {
#pragma unroll
                    for (int q = 0; q < NSW; ++q)
#pragma unroll
                        for (int j = 0; j < L; ++j) Piv[q][pb + j] = z[q][j];
                }
                __syncwarp();
                double2 tau[NSW], scale[NSW];
                double sq[NSW][L - 1];
#pragma unroll
                for (int j = 0; j < L - 1; ++j)
#pragma unroll
                    for (int q = 0; q < NSW; ++q) {
                        const double2 x = Piv[q][pb + j];
                        sq[q][j] = fma(x.x, x.x, x.y * x.y);
                    }
#pragma unroll
                for (int w = 1; w < L - 1; w <<= 1)
#pragma unroll
                    for (int j = 0; j + w < L - 1; j += 2 * w)
#pragma unroll
                        for (int q = 0; q < NSW; ++q) sq[q][j] += sq[q][j + w];
#pragma unroll
                for (int q = 0; q < NSW; ++q) {
                    // branch-free reflector (tau = 0 for an already-collapsed row)
                    const double s2 = L > 1 ? sq[q][0] : 0.0;
                    const double2 pv = Piv[q][pb + L - 1];
                    const double2 alpha = make_double2(pv.x, -pv.y);  // conj: row -> reflector space
                    const bool ident = s2 == 0.0 && alpha.y == 0.0;
                    const double nrm2 = ident ? 1.0 : fma(alpha.x, alpha.x, fma(alpha.y, alpha.y, s2));
                    const double rn = rsqrt(nrm2);
                    const double sg = alpha.x >= 0.0 ? -1.0 : 1.0;
                    const double beta = sg * nrm2 * rn;
                    const double ib = sg * rn;
                    const double zx = alpha.x - beta, zy = alpha.y;
                    const double zz = fma(zx, zx, zy * zy);
                    const double rz = rsqrt(zz > 0.0 ? zz : 1.0);
                    const double iz = rz * rz;
                    tau[q] = ident ? cz() : make_double2(1.0 - alpha.x * ib, -alpha.y * ib);
                    scale[q] = ident ? cz() : make_double2(zx * iz, -zy * iz);
                }
#pragma unroll
                for (int q = 0; q < NSW; ++q) {
                    if (lane < L) {
                        const double2 x = Piv[q][pb + lane];
                        U[q][ti * L + lane] =
                            lane < L - 1 ? cmul(make_double2(x.x, -x.y), scale[q]) : make_double2(1.0, 0.0);
                    }
                    if (lane == 0) Tau[q][ti] = tau[q];
                }
                __syncwarp();
                if (mine && rho < ti) blk_row_update_n<L, NSW>(z, U, ti * L, tau);
                if (ti > 0) {
#pragma unroll
                    for (int q = 0; q < NSW; ++q) {
#pragma unroll
                        for (int j = L - 1; j > 0; --j) z[q][j] = z[q][j - 1];
                        double2 v = make_double2(pf, 0.0);
                        if (mine && rho + M == ti - 1) v = csub(v, sig[q]);
                        z[q][0] = v;
                    }
                    if (mine && ti >= 2 && rho <= ti - 2) pf = Ab[arow + (int64_t)(b + ti - 2) * d.lda];
                }
            }
            __syncwarp();
        }
        // ---------------- reverse accumulation -> P (j-major) ----------------
        for (int cr = 0; cr < M; cr += CR)
        if (lane < 2 * min(CR, M - cr)) {
            const int ncr = min(CR, M - cr);
            const unsigned pm = ncr == 16 ? 0xffffffffu : ((1u << (2 * ncr)) - 1u);
            const int c = cr + (lane >> 1), hh = lane & 1, base = hh * HW;
            double2 w[NSW][HW];
#pragma unroll
            for (int q = 0; q < NSW; ++q)
#pragma unroll
                for (int k = 0; k < HW; ++k) w[q][k] = make_double2(base + k == c ? 1.0 : 0.0, 0.0);
            for (int s = 0; s < nbi; ++s) {
                double2 dp[NSW];
#pragma unroll
                for (int q = 0; q < NSW; ++q) {
                    const double2* us = U[q] + s * L + base;
                    dp[q] = cz();
#pragma unroll
                    for (int k = 0; k < HW; ++k) {
                        if (base + k < L) {
                            const double2 uk = us[k];  // conj(u) w
                            dp[q].x = fma(uk.x, w[q][k].x, dp[q].x);
                            dp[q].x = fma(uk.y, w[q][k].y, dp[q].x);
                            dp[q].y = fma(uk.x, w[q][k].y, dp[q].y);
                            dp[q].y = fma(-uk.y, w[q][k].x, dp[q].y);
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < NSW; ++q) {
                    dp[q].x += __shfl_xor_sync(pm, dp[q].x, 1);
                    dp[q].y += __shfl_xor_sync(pm, dp[q].y, 1);
                }
#pragma unroll
                for (int q = 0; q < NSW; ++q) {
                    const double2* us = U[q] + s * L + base;
                    const double2 td = cmul(Tau[q][s], dp[q]);
#pragma unroll
                    for (int k = 0; k < HW; ++k) {
                        if (base + k < L) {
                            const double2 uk = us[k];
                            w[q][k].x = fma(-uk.x, td.x, fma(uk.y, td.y, w[q][k].x));
                            w[q][k].y = fma(-uk.x, td.y, fma(-uk.y, td.x, w[q][k].y));
                        }
                    }
                    if (hh == 0) P[q][s * M + c] = w[q][0];
                }
#pragma unroll
                for (int q = 0; q < NSW; ++q) {
                    const double nx = __shfl_xor_sync(pm, w[q][0].x, 1);
                    const double ny = __shfl_xor_sync(pm, w[q][0].y, 1);
#pragma unroll
                    for (int k = 0; k < HW - 1; ++k) w[q][k] = w[q][k + 1];
                    w[q][HW - 1] = hh == 0 ? make_double2(nx, ny) : cz();
                }
            }
#pragma unroll
            for (int q = 0; q < NSW; ++q)
#pragma unroll
                for (int k = 0; k < HW; ++k)
                    if (base + k < M) P[q][(nbi + base + k) * M + c] = w[q][k];
        }
        __syncwarp();
        // ---------------- apply P_i: W22, then every row pass ----------------
#pragma unroll
        for (int q = 0; q < NSW; ++q) {
            double2 w22n[(M * M + 31) / 32];
#pragma unroll
            for (int e = 0; e < (M * M + 31) / 32; ++e) {
                const int u = lane + 32 * e;
                w22n[e] = cz();
                if (u < M * M) {
                    const int r = u / M, c = u - (u / M) * M;
#pragma unroll
                    for (int j = 0; j < M; ++j)
                        w22n[e] = cfma(W22[q][r * M + j], P[q][(nbi + j) * M + c], w22n[e]);
                }
            }
            __syncwarp();
#pragma unroll
            for (int e = 0; e < (M * M + 31) / 32; ++e) {
                const int u = lane + 32 * e;
                if (u < M * M) W22[q][u] = w22n[e];
            }
        }
        for (int pass = 0; pass < 4; ++pass) {
            const int t = pass * 32 + lane - off;
            if (t < 0) continue;
            if (pass == pass_rq) {
                // finished inner-block row: W row t = P12[t - b]
#pragma unroll
                for (int q = 0; q < NSW; ++q)
                    if (vq[q]) {
#pragma unroll
                        for (int c = 0; c < M; ++c) Wl[q][(int64_t)t * M + c] = P[q][(t - b) * M + c];
                    }
                continue;
            }
            const bool state = pass < pass_rq;  // t < b: state row; else W row
            double2 acc[NSW][M];
#pragma unroll
            for (int q = 0; q < NSW; ++q) {
#pragma unroll
                for (int c = 0; c < M; ++c) acc[q][c] = cz();
#pragma unroll
                for (int j = 0; j < M; ++j) {
                    const double2 zj = state ? Zl[q][(int64_t)j * d.LDZ + t] : Wl[q][(int64_t)t * M + j];
#pragma unroll
                    for (int c = 0; c < M; ++c) acc[q][c] = cfma(zj, P[q][(nbi + j) * M + c], acc[q][c]);
                }
            }
            if (state) {
                const double* ap = Ab + (int64_t)(d.k - NBo) + t + (int64_t)b * d.lda;
                double av[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) av[e] = e < nbi ? ap[(int64_t)e * d.lda] : 0.0;
                for (int jj = 0; jj < nbi; jj += 4) {
                    double an[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        an[e] = jj + 4 + e < nbi ? ap[(int64_t)(jj + 4 + e) * d.lda] : 0.0;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        if (jj + e < nbi) {
#pragma unroll
                            for (int q = 0; q < NSW; ++q)
#pragma unroll
                                for (int c = 0; c < M; ++c)
                                    acc[q][c] = rfma(av[e], P[q][(jj + e) * M + c], acc[q][c]);
                        }
                    }
#pragma unroll
                    for (int e = 0; e < 4; ++e) av[e] = an[e];
                }
                // lazy shift: A's diagonal in column b + dd sits in row b - M + dd
                const int dd = t - (b - M);
#pragma unroll
                for (int q = 0; q < NSW; ++q) {
                    if (dd >= 0 && dd < min(M, nbi)) {
#pragma unroll
                        for (int c = 0; c < M; ++c) acc[q][c] = csub(acc[q][c], cmul(sig[q], P[q][dd * M + c]));
                    }
                    if (vq[q]) {
#pragma unroll
                        for (int c = 0; c < M; ++c) Zl[q][(int64_t)c * d.LDZ + t] = acc[q][c];
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < NSW; ++q)
                    if (vq[q]) {
#pragma unroll
                        for (int c = 0; c < M; ++c) Wl[q][(int64_t)t * M + c] = acc[q][c];
                    }
            }
        }
        __syncwarp();
    }
    // W22 rows [NBo, NBo + m)
#pragma unroll
    for (int q = 0; q < NSW; ++q) {
        if (!vq[q]) continue;
        for (int u = lane; u < M * M; u += 32) {
            const int r = u / M, c = u - (u / M) * M;
            Wl[q][(int64_t)(NBo + r) * M + c] = W22[q][r * M + c];
        }
    }
}

}  // namespace ssd
