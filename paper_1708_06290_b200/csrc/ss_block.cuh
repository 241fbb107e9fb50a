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
#ifndef SS_BLK_OCC
#define SS_BLK_OCC 8  // resident one-warp CTAs per SM the register budget targets
#endif

struct BlkDims {
    int m, ptop, k, NBo;  // outer block: A rows [k-NBo, k), panel cols [c0, c0+NBo)
    int c0, r0;           // r0 = ptop + k - NBo: first stacked row of the block
    const double* A;
    int64_t lda;
    const double2* shifts;
    int64_t LDZ;
    int64_t wstride;  // elements (complex) per shift in W
    int woff;         // first W row of this block in the per-shift buffer
    // grouped outer blocks: > 0 = the wprod rows after this block's 128 W rows
    // hold the composite of the blocks below it in the group; they are
    // multiplied in place by this block's W22 (the composite now covers this
    // block too) and this block's W22 rows are not written (ss_sweep.cu,
    // enqueue_part)
    int wprod;
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
// The chain's staged panel rows (32 x 32 f64 per warp) alias P when P is
// large enough (P of the previous inner window is dead during the chain).
constexpr size_t kBlkPanelBytes = (size_t)kBlkInner * kBlkInner * 8;
__host__ __device__ constexpr bool blk_panel_in_p(int m) {
    return (size_t)(kBlkInner + m) * m * 16 >= kBlkPanelBytes;
}

constexpr int kBlkShiftsPerWarp = 1;  // 2 measured slower on B200 (per-warp issue bound)

__host__ __device__ inline size_t blk_smem_bytes(int m) {
    return kBlkShiftsPerWarp * blk_smem_bytes_1(m) + (blk_panel_in_p(m) ? 0 : kBlkPanelBytes);
}

// One warp per NSW shifts.  Block row t of the outer block is handled by
// lane (t + 128 - NBo) & 31 in pass (t + 128 - NBo) >> 5 in every phase, so
// the inner window i is pass 3 - i, the state rows above it are passes
// < 3 - i and the W rows below it passes > 3 - i; a row never changes lanes,
// so its values can stay in the (L2-resident) window buffer Z / the W output
// between phases without cross-lane hazards.
//
// The reflector chain is a serial dependency, so each warp runs one shift
// (NSW = 1; two interleaved shifts per warp measured slower) and all shifts'
// chains stay resident at once.
//
// P_i = H_{nbi-1}(...(H_0 E)) (first m columns of the window's unitary):
//  * m > 6: after the chain, by reverse accumulation: lane pair (2c, 2c+1)
//    owns column c of P, each lane half of the sliding L-window, so a step
//    is (L+1)/2 complex dot terms + one shuffle exchange;
//  * m <= 6 (kFuse): row-wise, beside the chain.  Row r of P is
//    e_r^T H_{nbi-1} ... H_0 restricted to columns < m: the chain's own row
//    update applied to e_r, starting at step r (columns right of r are zero
//    before), and a data row retires exactly when it is the pivot -- so lane
//    rho carries data row rho while ti > rho and P row rho from ti = rho on,
//    at no extra instruction; lanes < m carry the m rows of P22 (e_{nbi+j})
//    in a second window.
template <int M, int NSW>
__global__ void __launch_bounds__(32, NSW == 1 ? SS_BLK_OCC : 6)
    k_block(BlkDims d, double2* __restrict__ Z, double2* __restrict__ W, int sb) {
    constexpr int L = M + 1;
    constexpr int HW = (L + 1) / 2;  // window entries per lane of a column pair
    constexpr int CR = 16;           // columns per reverse-accumulation round (2 lanes each)
    static_assert(L <= 32, "k_block: m <= 31");
    // P rows beside the chain for narrow windows: measured on B200, config 1
    // (m = 5) block kernel 0.34 -> 0.28 ms, config 2 (m = 10) 5.27 -> 5.53 ms
    // (the extra P-row window's 8L DFMA per step outweigh the column-wise
    // reverse accumulation they replace once the window is wide)
    constexpr bool kFuse = M <= 6;
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
    double* Apn = reinterpret_cast<double*>(reinterpret_cast<double2*>(smem) +
                                            (blk_panel_in_p(M) ? 0 : NSW * QSZ));  // [32][32]
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
        Wl[q] = W + (int64_t)l * d.wstride + (int64_t)d.woff * M;  // W row t, column c: Wl[t*M + c]
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
            // Reflector of pivot row p (y = conj(p), alpha = y[L-1]) in the
            // unnormalised form H = I - kappa v v^H, v = y - beta e_L,
            // kappa = 1 / (beta (beta - conj(alpha))) (|beta - conj(alpha)| >=
            // |beta| > 0, no cancellation): the same H as
            // I - tau u u^H with u = v / (alpha - beta), tau = (beta - alpha) /
            // beta (kernels.py:74-99's sign rule), but the row update needs only
            // the broadcast pivot row and kappa, so each lane's dot product runs
            // beside the rsqrt / reciprocal chain and no second broadcast (of u)
            // sits on the serial path.  Rows not updated this step get tw = 0
            // (z - 0 v = z exactly), so the update is branch-free.
            const int t = pass_rq * 32 + lane - off;  // this lane's block row
            const int rho = t - b;
            const bool mine = t >= 0 && rho >= 0;
            const int64_t arow = (int64_t)(d.k - NBo) + t;
            // this lane's panel row over the inner window, staged once (all
            // loads in flight together) instead of one dependent load per step
            for (int c = 0; c < nbi; ++c) Apn[c * 32 + lane] = mine ? Ab[arow + (int64_t)(b + c) * d.lda] : 0.0;
            double2 z[NSW][L];  // window: z[0] = panel column, z[1..L) = state
            // kFuse: P_i's rows are accumulated beside the chain (see k_block's
            // comment): lane rho carries data row rho while ti > rho and row
            // rho of P from ti = rho on; lanes < M also carry P row nbi + lane
            double2 x2[NSW][kFuse ? L : 1];
            if (kFuse) {
#pragma unroll
                for (int q = 0; q < NSW; ++q)
#pragma unroll
                    for (int j = 0; j < (kFuse ? L : 1); ++j)
                        x2[q][j] = make_double2(j == lane + 1 ? 1.0 : 0.0, 0.0);
            }
            {
                const double a0 = Apn[(nbi - 1) * 32 + lane];
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
                    if (kFuse) {  // the pivot row retires; row rho of P starts as e_rho
#pragma unroll
                        for (int q = 0; q < NSW; ++q)
#pragma unroll
                            for (int j = 0; j < L; ++j) z[q][j] = make_double2(j == 0 ? 1.0 : 0.0, 0.0);
                    }
                }
                const double pf = ti > 0 ? Apn[(ti - 1) * 32 + lane] : 0.0;
                __syncwarp();
                const bool upd = kFuse ? mine : (mine && rho < ti);
#pragma unroll
                for (int q = 0; q < NSW; ++q) {
                    double2 pv[L];
#pragma unroll
                    for (int j = 0; j < L; ++j) pv[j] = Piv[q][pb + j];
                    // z . y over the first L-1 entries (two partial sums) and |y|^2
                    double2 d0 = cz(), d1 = cz();
                    double sq[L > 1 ? L - 1 : 1];
#pragma unroll
                    for (int j = 0; j < L - 1; ++j) {
                        double2& dd = (j & 1) ? d1 : d0;  // z_j conj(p_j)
                        dd.x = fma(z[q][j].x, pv[j].x, dd.x);
                        dd.x = fma(z[q][j].y, pv[j].y, dd.x);
                        dd.y = fma(z[q][j].y, pv[j].x, dd.y);
                        dd.y = fma(-z[q][j].x, pv[j].y, dd.y);
                        sq[j] = fma(pv[j].x, pv[j].x, pv[j].y * pv[j].y);
                    }
#pragma unroll
                    for (int w = 1; w < L - 1; w <<= 1)
#pragma unroll
                        for (int j = 0; j + w < L - 1; j += 2 * w) sq[j] += sq[j + w];
                    const double s2 = L > 1 ? sq[0] : 0.0;
                    const double2 alpha = make_double2(pv[L - 1].x, -pv[L - 1].y);
                    const bool ident = s2 == 0.0 && alpha.y == 0.0;
                    const double nrm2 = ident ? 1.0 : fma(alpha.x, alpha.x, fma(alpha.y, alpha.y, s2));
                    const double rn = rsqrt_pos(nrm2);
                    const double sg = alpha.x >= 0.0 ? -1.0 : 1.0;
                    const double beta = sg * nrm2 * rn, ib = sg * rn;  // beta, 1 / beta
                    // kappa = (1 / beta) conj(beta - conj(alpha)) / |beta - conj(alpha)|^2
                    const double zx = beta - alpha.x;
                    const double f = ib * rcp_pos(fma(zx, zx, alpha.y * alpha.y));
                    const double2 kap = ident ? cz() : make_double2(zx * f, -alpha.y * f);
                    // rows not updated this step: kappa -> 0 (a select, so the
                    // dot product stays unconditional and overlaps the chain)
                    const double2 kup = upd ? kap : cz();
                    const double2 vl = make_double2(alpha.x - beta, alpha.y);  // v[L-1]
                    double2 dot = cadd(d0, d1);
                    dot = cfma(z[q][L - 1], vl, dot);
                    const double2 tw = cmul(kup, dot);
#pragma unroll
                    for (int j = 0; j < L - 1; ++j) {  // z_j -= tw conj(v_j) = tw p_j
                        // wide windows re-read the pivot (register pressure)
                        const double2 pj = L > 16 ? Piv[q][pb + j] : pv[j];
                        z[q][j].x = fma(-tw.x, pj.x, fma(tw.y, pj.y, z[q][j].x));
                        z[q][j].y = fma(-tw.x, pj.y, fma(-tw.y, pj.x, z[q][j].y));
                    }
                    z[q][L - 1].x = fma(-tw.x, vl.x, fma(-tw.y, vl.y, z[q][L - 1].x));
                    z[q][L - 1].y = fma(tw.x, vl.y, fma(-tw.y, vl.x, z[q][L - 1].y));
                    if (kFuse) {
                        // P row nbi + lane (zero windows on lanes >= M stay zero)
                        double2 e0 = cz(), e1 = cz();
#pragma unroll
                        for (int j = 0; j < L - 1; ++j) {
                            double2& dd = (j & 1) ? e1 : e0;
                            dd.x = fma(x2[q][j].x, pv[j].x, dd.x);
                            dd.x = fma(x2[q][j].y, pv[j].y, dd.x);
                            dd.y = fma(x2[q][j].y, pv[j].x, dd.y);
                            dd.y = fma(-x2[q][j].x, pv[j].y, dd.y);
                        }
                        double2 dot2 = cadd(e0, e1);
                        dot2 = cfma(x2[q][L - 1], vl, dot2);
                        const double2 tw2 = cmul(kap, dot2);
#pragma unroll
                        for (int j = 0; j < L - 1; ++j) {
                            x2[q][j].x = fma(-tw2.x, pv[j].x, fma(tw2.y, pv[j].y, x2[q][j].x));
                            x2[q][j].y = fma(-tw2.x, pv[j].y, fma(-tw2.y, pv[j].x, x2[q][j].y));
                        }
                        x2[q][L - 1].x = fma(-tw2.x, vl.x, fma(-tw2.y, vl.y, x2[q][L - 1].x));
                        x2[q][L - 1].y = fma(tw2.x, vl.y, fma(-tw2.y, vl.x, x2[q][L - 1].y));
                    } else {
                        // v and kappa for the reverse accumulation (off the serial path)
                        if (lane < L) {
                            const double2 x = Piv[q][pb + lane];
                            U[q][ti * L + lane] = lane < L - 1 ? make_double2(x.x, -x.y) : vl;
                        }
                        if (lane == 0) Tau[q][ti] = kap;
                    }
                }
                // slide (unconditionally: after the last step z is dead)
#pragma unroll
                for (int q = 0; q < NSW; ++q) {
#pragma unroll
                    for (int j = L - 1; j > 0; --j) z[q][j] = z[q][j - 1];
                    // P rows (kFuse, rho >= ti) take a zero: e_rho has no entry left of rho
                    double2 v = (!kFuse || rho < ti) ? make_double2(pf, 0.0) : cz();
                    if (mine && rho + M == ti - 1) v = csub(v, sig[q]);
                    z[q][0] = v;
                    if (kFuse) {
#pragma unroll
                        for (int j = (kFuse ? L : 1) - 1; j > 0; --j) x2[q][j] = x2[q][j - 1];
                        x2[q][0] = cz();
                    }
                }
            }
            if (kFuse) {
                // after the last step's slide, window entry c + 1 is column c
#pragma unroll
                for (int q = 0; q < NSW; ++q) {
                    if (mine) {
#pragma unroll
                        for (int c = 0; c < M; ++c) P[q][rho * M + c] = z[q][c + 1];
                    }
                    if (lane < M) {
#pragma unroll
                        for (int c = 0; c < M; ++c) P[q][(nbi + lane) * M + c] = x2[q][(kFuse ? c + 1 : 0)];
                    }
                }
            }
            __syncwarp();
        }
        // ---------------- reverse accumulation -> P (j-major) ----------------
        for (int cr = 0; cr < (kFuse ? 0 : M); cr += CR)
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
                    double2 d2[2] = {cz(), cz()};  // two partial sums: half the FMA chain depth
#pragma unroll
                    for (int k = 0; k < HW; ++k) {
                        if (base + k < L) {
                            const double2 uk = us[k];  // conj(u) w
                            double2& dd = d2[k & 1];
                            dd.x = fma(uk.x, w[q][k].x, dd.x);
                            dd.x = fma(uk.y, w[q][k].y, dd.x);
                            dd.y = fma(uk.x, w[q][k].y, dd.y);
                            dd.y = fma(-uk.y, w[q][k].x, dd.y);
                        }
                    }
                    dp[q] = cadd(d2[0], d2[1]);
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
    if (d.wprod > 0) {
        // composite of this block and the previous one: W_prev <- W_prev W22
#pragma unroll
        for (int q = 0; q < NSW; ++q) {
            if (!vq[q]) continue;
            double2* Wp = Wl[q] + (int64_t)kBlkNB * M;  // the composite rows below this block's
            for (int row = lane; row < d.wprod; row += 32) {
                // keep the W22 loads inside the loop (hoisting all m^2 of them
                // out of it spills)
                asm volatile("" ::: "memory");
                double2 w[M], acc[M];
#pragma unroll
                for (int j = 0; j < M; ++j) w[j] = Wp[(int64_t)row * M + j];
#pragma unroll
                for (int c = 0; c < M; ++c) acc[c] = cz();
#pragma unroll
                for (int j = 0; j < M; ++j)
#pragma unroll
                    for (int c = 0; c < M; ++c) acc[c] = cfma(w[j], W22[q][j * M + c], acc[c]);
#pragma unroll
                for (int c = 0; c < M; ++c) Wp[(int64_t)row * M + c] = acc[c];
            }
        }
        return;
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
