// Two-level window sweep: the fused outer-block kernel.
//
// The reference sweep (solvers.py:165-200, Alg. 6) walks windows of
// nb panel columns; after every window every shift's state rows [0, r0) are
// updated with that window's P_l ((nb+m) x m).  Per updated row that costs
// 4 m nb (real panel x P12) + 8 m^2 (state x P22) flops, so the state part is
// a 2m/nb overhead on the algorithmic work -- 31% at nb = 64, m = 10.
//
// Here the windows are grouped into outer blocks of NB = 128 columns.  One
// CTA per shift runs the NB/32 inner windows (nb = 32) of an outer block
// entirely on chip:
//   * the block rows [r0_out, r0_out + NBo) of the state live in registers,
//     one row per thread (128 threads);
//   * inner step i: warp 3-i owns the inner block's 32 rows and factors it
//     with row Householder reflectors (same scheme and sign rule as
//     ss_rq_house.cuh / kernels.py:74-99), then forms P_i by reverse
//     accumulation (lanes = columns);
//   * every thread then applies P_i to its row: rows above the inner block
//     get state <- state P22 + A(row, inner cols) P12 - sigma P12[lazy row]
//     (solvers.py:186-199 restricted to the block); the inner block's own rows
//     are finished and their registers are reused for rows of the composite
//         W <- E_b P12 + W P22,    W = [W_panel (NBo x m); W22 (m x m)]
//     so that after the outer block the far rows [0, r0_out) need ONE update
//         state <- state W22 + Pan(:, outer cols) W_panel - sigma W[lazy row]
//     (done by k_update_ws in 64-column passes, the first with W22, the rest
//     with the identity).  The state overhead on the far rows drops to 2m/NB.
// Only W ((NBo + m) x m per shift, j-major) leaves the kernel; the outer
// block's rows are finished (part of R, never needed again).
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

__host__ __device__ inline size_t blk_smem_bytes(int m) {
    const int L = m + 1;
    size_t b = 32 * 8;                      // one mbarrier per reflector of the inner window
    b += (size_t)(kBlkInner + m) * m * 16;  // P
    b += (size_t)kBlkInner * L * 16;        // U
    b += (size_t)kBlkInner * 16;            // Tau
    b += (size_t)2 * 32 * 16;               // pivot broadcast
    b += (size_t)m * m * 16;                // W22
    b += (size_t)kBlkNB * m * 16;           // block state / W rows, column-major [c][128]
    return b;
}

// P_i rows by forward accumulation: P = Q E with Q = H_{nbi-1} ... H_0, so
// row r of P is e_r^T run through the same right-applied reflector sequence
// as a block row (window of L columns sliding one column per reflector; the
// entering column holds e_r's entry).  Two helper warps do this for the
// nbi + m rows of P in lockstep with the reflector chain (one mbarrier per
// reflector), so P is complete one step after the chain -- no serial
// reverse accumulation.
template <int M>
__global__ void __launch_bounds__(kBlkNB, SS_BLK_MINB)
    k_block(BlkDims d, const double2* __restrict__ Z, double2* __restrict__ W) {
    constexpr int L = M + 1;
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* mb = reinterpret_cast<uint64_t*>(smem);                 // [32]
    double2* P = reinterpret_cast<double2*>(smem + 32 * 8);          // [(32 + M) * M] j-major
    double2* U = P + (kBlkInner + M) * M;                            // [32][L]
    double2* Tau = U + kBlkInner * L;                                // [32]
    double2* Piv = Tau + kBlkInner;                                  // [2][32]
    double2* W22 = Piv + 64;                                         // [M][M]: W22[r * M + c]
    double2* S = W22 + M * M;  // [M][128]: state row t (later W row t), column c at S[c*128 + tid]

    const int l = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int NBo = d.NBo;
    const int t = tid - (kBlkNB - NBo);  // block row of this thread (< 0: idle)
    const bool active = t >= 0;
    const int64_t arow = (int64_t)(d.k - NBo) + t;  // A row of block row t
    const double2 sig = d.shifts[l];
    const double* Ab = d.A + (int64_t)d.c0 * d.lda;  // panel column 0

    if (tid == 0) {
        for (int q = 0; q < kBlkInner; ++q) mbar_init(mb + q, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // the block's state rows live in shared memory (column-major, one row per
    // thread); only the RQ warp holds its rows in registers during its chain
    {
        const double2* zr = Z + (int64_t)l * M * d.LDZ + d.r0 + t;
#pragma unroll
        for (int c = 0; c < M; ++c) S[c * kBlkNB + tid] = active ? zr[(int64_t)c * d.LDZ] : cz();
    }
    for (int u = tid; u < M * M; u += kBlkNB) W22[u] = make_double2((u / M) == (u % M) ? 1.0 : 0.0, 0.0);
    __syncthreads();

    const int ni = (NBo + kBlkInner - 1) / kBlkInner;
    for (int i = 0; i < ni; ++i) {
        const int top = NBo - kBlkInner * i;  // rows [b, top) = inner block
        const int b = max(0, top - kBlkInner);
        const int nbi = top - b;
        const int rqw = 3 - i;
        const int hw = (warp - rqw - 1) & 3;  // helper index 0, 1 (2: idle)
        if (warp == rqw) {
            // ---------------- reflector chain over the inner block ----------------
            const int rho = t - b;
            const bool mine = active && rho >= 0;
            double2 z[L];  // window: z[0] = panel column, z[1..L) = state
#pragma unroll
            for (int c = 0; c < M; ++c) z[c + 1] = S[c * kBlkNB + tid];
            z[0] = cz();
            if (mine) {
                z[0] = make_double2(Ab[arow + (int64_t)(b + nbi - 1) * d.lda], 0.0);
                if (nbi - 1 == rho + M) z[0] = csub(z[0], sig);
            }
            double pf = 0.0;
            if (mine && nbi >= 2 && rho <= nbi - 2) pf = Ab[arow + (int64_t)(b + nbi - 2) * d.lda];
            for (int ti = nbi - 1; ti >= 0; --ti) {
                double2* piv = Piv + (ti & 1) * 32;
                if (mine && rho == ti) {
#pragma unroll
                    for (int j = 0; j < L; ++j) piv[j] = z[j];
                }
                __syncwarp();
                // ||row||^2 without the pivot entry, and the pivot (redundant per lane)
                double sq[L - 1];
#pragma unroll
                for (int j = 0; j < L - 1; ++j) {
                    const double2 x = piv[j];
                    sq[j] = fma(x.x, x.x, x.y * x.y);
                }
#pragma unroll
                for (int w = 1; w < L - 1; w <<= 1)
#pragma unroll
                    for (int j = 0; j + w < L - 1; j += 2 * w) sq[j] += sq[j + w];
                const double s2 = L > 1 ? sq[0] : 0.0;
                const double2 pv = piv[L - 1];
                const double2 alpha = make_double2(pv.x, -pv.y);  // conj: row -> reflector space
                double2 tau = cz(), scale = cz();
                if (!(s2 == 0.0 && alpha.y == 0.0)) {
                    const double nrm2 = fma(alpha.x, alpha.x, fma(alpha.y, alpha.y, s2));
                    const double rn = rsqrt(nrm2);
                    const double sg = alpha.x >= 0.0 ? -1.0 : 1.0;
                    const double beta = sg * nrm2 * rn;
                    const double ib = sg * rn;
                    tau = make_double2(1.0 - alpha.x * ib, -alpha.y * ib);
                    const double zx = alpha.x - beta, zy = alpha.y;
                    const double rz = rsqrt(fma(zx, zx, zy * zy));
                    const double iz = rz * rz;
                    scale = make_double2(zx * iz, -zy * iz);
                }
                // lane j < L publishes u_j (u_{L-1} = 1) and tau
                if (lane < L) {
                    const double2 x = piv[lane];
                    U[ti * L + lane] =
                        lane < L - 1 ? cmul(make_double2(x.x, -x.y), scale) : make_double2(1.0, 0.0);
                }
                if (lane == 0) Tau[ti] = tau;
                __syncwarp();
                if (lane == 0) mbar_arrive(mb + ti);  // release U[ti], Tau[ti] to the helpers
                if (mine && rho < ti) {
                    double2 uu[L];
#pragma unroll
                    for (int j = 0; j < L; ++j) uu[j] = U[ti * L + j];
                    rq_row_update<L>(z, uu, tau, L);
                }
#pragma unroll
                for (int j = L - 1; j > 0; --j) z[j] = z[j - 1];
                if (ti > 0) {
                    double2 v = make_double2(pf, 0.0);
                    if (mine && rho + M == ti - 1) v = csub(v, sig);
                    z[0] = v;
                    if (mine && ti >= 2 && rho <= ti - 2) pf = Ab[arow + (int64_t)(b + ti - 2) * d.lda];
                }
            }
        } else if (hw < 2) {
            // ---------------- P rows, one reflector behind the chain ----------------
            const int pr = hw * 32 + lane;  // row of P_i
            const bool prow = pr < nbi + M;
            double2 w[L];
#pragma unroll
            for (int j = 0; j < L; ++j) w[j] = make_double2(pr == nbi - 1 + j ? 1.0 : 0.0, 0.0);
            for (int ti = nbi - 1; ti >= 0; --ti) {
                mbar_wait(mb + ti, i & 1);
                const double2 ts = Tau[ti];
                const double2* uu = U + ti * L;
                double2 dp = cz(), dq = cz();
#pragma unroll
                for (int j = 0; j < L; j += 2) {
                    dp = cfma(w[j], uu[j], dp);
                    if (j + 1 < L) dq = cfma(w[j + 1], uu[j + 1], dq);
                }
                const double2 tw = cmul(ts, cadd(dp, dq));
#pragma unroll
                for (int j = 0; j < L; ++j) {
                    const double2 uj = uu[j];
                    w[j].x = fma(-tw.x, uj.x, fma(-tw.y, uj.y, w[j].x));
                    w[j].y = fma(-tw.y, uj.x, fma(tw.x, uj.y, w[j].y));
                }
                if (ti > 0) {
#pragma unroll
                    for (int j = L - 1; j > 0; --j) w[j] = w[j - 1];
                    w[0] = make_double2(pr == ti - 1 ? 1.0 : 0.0, 0.0);
                }
            }
            if (prow) {
#pragma unroll
                for (int c = 0; c < M; ++c) P[pr * M + c] = w[c];
            }
        }
        __syncthreads();  // P ready
        // ---------------- apply P_i to every row of the block ----------------
        double2 w22n = cz();
        if (tid < M * M) {  // W22 <- W22 P22 (identity-part rows of W)
            const int r = tid / M, c = tid - (tid / M) * M;
#pragma unroll
            for (int j = 0; j < M; ++j) w22n = cfma(W22[r * M + j], P[(nbi + j) * M + c], w22n);
        }
        if (active) {
            double2 acc[M];
            if (t >= b && t < top) {
                // finished inner-block row: becomes W row t = P12[t - b]
#pragma unroll
                for (int c = 0; c < M; ++c) acc[c] = P[(t - b) * M + c];
            } else {
                // state (t < b) or W row (t >= top): row <- row P22 (+ panel part)
#pragma unroll
                for (int c = 0; c < M; ++c) acc[c] = cz();
#pragma unroll
                for (int j = 0; j < M; ++j) {
                    const double2 zj = S[j * kBlkNB + tid];
#pragma unroll
                    for (int c = 0; c < M; ++c) acc[c] = cfma(zj, P[(nbi + j) * M + c], acc[c]);
                }
                if (t < b) {
                    const double* ap = Ab + arow + (int64_t)b * d.lda;
                    int jj = 0;
                    for (; jj + 4 <= nbi; jj += 4) {
                        double av[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) av[e] = ap[(int64_t)(jj + e) * d.lda];
#pragma unroll
                        for (int e = 0; e < 4; ++e)
#pragma unroll
                            for (int c = 0; c < M; ++c) acc[c] = rfma(av[e], P[(jj + e) * M + c], acc[c]);
                    }
                    for (; jj < nbi; ++jj) {
                        const double av = ap[(int64_t)jj * d.lda];
#pragma unroll
                        for (int c = 0; c < M; ++c) acc[c] = rfma(av, P[jj * M + c], acc[c]);
                    }
                    // lazy shift: A's diagonal in column b + dd sits in row b - M + dd
                    const int dd = t - (b - M);
                    if (dd >= 0 && dd < min(M, nbi)) {
#pragma unroll
                        for (int c = 0; c < M; ++c) acc[c] = csub(acc[c], cmul(sig, P[dd * M + c]));
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < M; ++c) S[c * kBlkNB + tid] = acc[c];
        }
        __syncthreads();  // everyone done with P / W22 (old)
        if (tid < M * M) W22[tid] = w22n;
    }
    __syncthreads();
    // ---------------- W out: rows [0, NBo) from registers, W22 from smem ----------------
    double2* wl = W + (int64_t)l * d.wstride;
    for (int u = tid; u < NBo * M; u += kBlkNB) {  // coalesced: W is j-major
        const int r = u / M, c = u - (u / M) * M;
        wl[u] = S[c * kBlkNB + (kBlkNB - NBo) + r];
    }
    for (int u = tid; u < M * M; u += kBlkNB) {
        const int r = u / M, c = u - (u / M) * M;
        wl[(int64_t)(NBo + r) * M + c] = W22[r * M + c];
    }
}

}  // namespace ssd
