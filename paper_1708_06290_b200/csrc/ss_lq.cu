// Transposed shifted solves (A - sigma_l I)^T x_l = c_l, general right-hand
// sides, sm_100a.
//
// Reference path (solvers.py:320-486 solve_shifted_transposed / _sweep_lq,
// batched.py:125-182 batched_lq): the stacked matrix [A^T - sigma I; -I] is
// brought to lower-triangular form top-down by a sliding window; the stacked
// vector w = [rhs; 0] is forward-substituted in the same sweep, so its lower
// half accumulates the solution.  Per shift the state is S = [z2 | w]:
// (2n) x (m+1) complex (z2 = the m active transformed columns).
//
// B200 mapping (one launch of each per window step of nb <= 32 rows):
//   k_tseed   S = [A^T(:, 0:m) - sigma E; -E | rhs; 0]
//   k_lq      one warp per shift: lane = block row.  The nb x (nb+m) lower
//             trapezoid [z2 rows | panel of A^T] is reduced top-down by row
//             Householder reflectors (row i's window = columns i..i+m, pivot
//             first; same sign rule as kernels.py:74-99), the window's w
//             segment is forward-substituted in the same pass (every pivot
//             checked against tol_l, batched.py:168-178), then the m new
//             active columns P[:, nb:nb+m] and dW = P[:, :nb] y are formed by
//             reverse accumulation (lanes = the m+1 vectors).  Householder
//             and the reference's mirrored Givens schedule give the same
//             |L_ii| (the LQ factor is unique up to phases), so the
//             singularity decisions agree.
//   update    rows below the window: S <- S T + Pan(A^T, -I) U12 (the
//             reference's update_shift + trail_shift, solvers.py:431-468),
//             with w treated as an extra state column; lazy-shift rows get
//             -sigma P12.  The forward sweep's window-update kernel with the
//             [A^T; -I] panel (k_update<..., TR>, register tiles, staged P and
//             rows; the -I rows past the window's last column are skipped:
//             their state is still zero); k_tupd (row per thread) for m > 99.
//   k_ttail   one CTA per shift: the unblocked m-column tail with the
//             reference's Givens rotations fused with the last substitutions
//             (solvers.py:470-486); x = w[n:].
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "ss_device.cuh"
#include "ss_internal.h"
#include "ss_rq_house.cuh"
#include "ss_update.cuh"

using namespace ssd;

namespace ss {
// ss_sweep.cu: the window-update kernel on the [A^T; -I] panel, and the
// composite fold / K-streamed far pass
int launch_update_tr(ss_handle* h, ssd::UpdDims u, int rows, double2* S, const double2* P, cudaStream_t st);

bool tr_far_supported(ss_handle* h, int M);
int wsuffix(ss_handle* h, cudaStream_t st, int sb, int g, const int* x, const int* nb, int M, int mc, int K,
            const double2* P, int64_t slab, double2* W, int64_t wstride);
bool tr_split_supported(ss_handle* h, int m);
int tr_far_split(ss_handle* h, cudaStream_t st, int n, int m, const double* A, int64_t lda,
                 const double2* shifts, int sb, double2* S, int64_t LDS, int rlo, int r0_all, int c0, int K,
                 const double2* W, int64_t wstride, double2* Wz, int64_t wzstride, double2* Ww, int64_t gstride);
int tr_far(ss_handle* h, cudaStream_t st, int n, int m, int M, const double* A, int64_t lda,
           const double2* shifts, int sb, double2* S, int64_t LDS, int rlo, int r0, int c0, int K,
           const double2* W, int64_t wstride);
}

namespace {

constexpr int kLqMaxNb = 32;
constexpr int kFkmShiftsLq = 80;  // k_farkm's shifts per unit (ss_fark.cuh kFkmShifts)
// panel columns per transposed composite (the packed panel's capacity): 16
// windows of 32 rows; 12 / 8 / 6 windows measured 1.71k / 1.61k / 1.50k vs
// 1.72k shifts/s (n = 10000, m = 20)
constexpr int kTrK = 512;

struct TDims {
    int n, m, mp;  // mp = m + 1 state columns per shift
    int ms;        // columns per shift in S and P: mp, or mp padded to a multiple of 10 (composites)
    const double* A;
    int64_t lda;
    const double2* shifts;  // batch-local
    int sb;
    int64_t LDS;     // leading dimension of one state column (>= 2n)
    int32_t* fail;   // batch-local fail rows (-1 = ok)
    const double* tol;  // batch-local pivot tolerances
};

// ---------------------------------------------------------------------------
// seed (solvers.py:375-381)
// ---------------------------------------------------------------------------
__global__ void k_tseed(TDims d, const double2* __restrict__ rhs, int64_t ldr,
                        double2* __restrict__ S) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int l = blockIdx.y;
    if (i >= d.LDS) return;
    const double2 sig = d.shifts[l];
    double2* Sl = S + (int64_t)l * d.ms * d.LDS;
    for (int c = d.mp; c < d.ms; ++c) Sl[(int64_t)c * d.LDS + i] = cz();  // padding columns
    for (int c = 0; c < d.m; ++c) {
        double2 v = cz();
        if (i < d.n) {
            v.x = d.A[c + (int64_t)i * d.lda];  // A^T(i, c)
            if (i == c) v = csub(v, sig);
        } else if (i < 2 * d.n && i - d.n == c) {
            v.x = -1.0;
        }
        Sl[(int64_t)c * d.LDS + i] = v;
    }
    Sl[(int64_t)d.m * d.LDS + i] = i < d.n ? rhs[i + (int64_t)l * ldr] : cz();
    if (i == 0) d.fail[l] = -1;
}

// ---------------------------------------------------------------------------
// per-window block LQ with fused forward substitution (batched.py:125-182)
// ---------------------------------------------------------------------------
struct LqStep {
    int k0;   // 0-based first row of the window (k1 - 1)
    int nb;   // window rows (<= 32)
    int c0;   // 0-based first panel column of A^T (k0 + m)
};

// Output per shift: Pout ((nb + mp) x mp, j-major) for k_tupd:
//   rows j < nb          panel part  [P[m+j, nb:nb+m] | -dW[m+j]]
//   rows nb + r, r < m   state part  [P[r, nb:nb+m]   | -dW[r]]
//   row  nb + m          w row       [0 ... 0         | 1]
template <int LMAX>
__global__ void __launch_bounds__(32) k_lq(TDims d, LqStep st, const double2* __restrict__ S,
                                           double2* __restrict__ Pout) {
    __shared__ double2 Piv[LMAX];
    __shared__ double2 U[kLqMaxNb][LMAX];
    __shared__ double2 Tau[kLqMaxNb];
    __shared__ double2 Y[kLqMaxNb];
    const int l = blockIdx.x;
    const int lane = threadIdx.x;
    const int m = d.m, L = m + 1, nb = st.nb, mp = d.mp;
    const double2 sig = d.shifts[l];
    const int ms = d.ms;
    const double2* Sl = S + (int64_t)l * ms * d.LDS;
    double2* Po = Pout + (int64_t)l * (nb + ms) * ms;
    if (d.fail[l] >= 0) return;  // failed in an earlier window: left as is (NaN at the end)
    // padding of a widened P (composites): zero rows nb + mp .. and columns mp ..
    for (int e = lane; e < (nb + ms) * (ms - mp); e += 32) Po[(int64_t)(e / (ms - mp)) * ms + mp + e % (ms - mp)] = cz();
    for (int e = lane; e < (ms - mp) * mp; e += 32) Po[(int64_t)(nb + mp + e / mp) * ms + e % mp] = cz();
    const bool mine = lane < nb;
    const int row = st.k0 + lane;  // A^T row / stacked row of this lane
    // window of row `lane` at step 0: columns 0..m = [z2 row | panel col 0]
    double2 r[LMAX];
#pragma unroll
    for (int j = 0; j < LMAX; ++j) r[j] = cz();
    double2 y = cz();
    if (mine) {
#pragma unroll
        for (int j = 0; j < LMAX; ++j)
            if (j < m) r[j] = Sl[(int64_t)j * d.LDS + row];
        double2 v = make_double2(d.A[st.c0 + (int64_t)row * d.lda], 0.0);  // A^T(row, c0)
        if (lane == m) v = csub(v, sig);  // block diagonal (lazy shift), solvers.py:398-400
#pragma unroll
        for (int j = 0; j < LMAX; ++j)
            if (j == m) r[j] = v;
        y = Sl[(int64_t)m * d.LDS + row];
    }
    const double tol = d.tol[l];
    int fail = -1;
    for (int t = 0; t < nb; ++t) {
        if (lane == t) {
#pragma unroll
            for (int j = 0; j < LMAX; ++j)
                if (j < L) Piv[j] = r[j];
        }
        __syncwarp();
        // reflector of row t (pivot first): zlarfg on y = conj(row)
        double s2 = 0.0;
        for (int j = 1; j < L; ++j) s2 = fma(Piv[j].x, Piv[j].x, fma(Piv[j].y, Piv[j].y, s2));
        const double2 alpha = make_double2(Piv[0].x, -Piv[0].y);
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
        double2 uu[LMAX];
#pragma unroll
        for (int j = 0; j < LMAX; ++j) {
            if (j == 0) {
                uu[j] = make_double2(1.0, 0.0);
            } else if (j < L) {
                const double2 x = Piv[j];
                uu[j] = cmul(make_double2(x.x, -x.y), scale);
            } else {
                uu[j] = cz();
            }
        }
        if (lane < L) {
            double2 mineu = cz();
#pragma unroll
            for (int j = 0; j < LMAX; ++j) mineu = (j == lane) ? uu[j] : mineu;
            U[t][lane] = mineu;
        }
        if (lane == 0) Tau[t] = tau;
        if (mine && lane >= t) rq_row_update<LMAX>(r, uu, tau, L);
        // forward substitution on the window's w segment (batched.py:170-178):
        // lane t holds L(t,t), lanes below hold L(lane, t) in r[0]
        const double2 piv = make_double2(__shfl_sync(0xffffffffu, r[0].x, t),
                                         __shfl_sync(0xffffffffu, r[0].y, t));
        if (fail < 0 && hypot(piv.x, piv.y) <= tol) fail = st.k0 + t;
        double2 yt = make_double2(__shfl_sync(0xffffffffu, y.x, t), __shfl_sync(0xffffffffu, y.y, t));
        yt = cdiv(yt, piv);
        if (lane == t) y = yt;
        if (mine && lane > t) y = csub(y, cmul(r[0], yt));
        // slide: column t retires, column t + m + 1 (panel column t + 1) enters
#pragma unroll
        for (int j = 0; j < LMAX - 1; ++j) r[j] = r[j + 1];
        r[LMAX - 1] = cz();
        if (t + 1 < nb) {
            double2 v = cz();
            if (mine && lane > t) {
                v.x = d.A[st.c0 + t + 1 + (int64_t)row * d.lda];  // A^T(row, c0 + t + 1)
                if (lane == m + t + 1) v = csub(v, sig);
            }
#pragma unroll
            for (int j = 0; j < LMAX; ++j)
                if (j == m) r[j] = v;
        }
        __syncwarp();
    }
    if (fail >= 0) {
        if (lane == 0) d.fail[l] = fail;
        return;
    }
    if (mine) Y[lane] = y;
    __syncwarp();
    // reverse accumulation: vector q < m is e_{nb+q}, vector m is [y; 0];
    // P = H_0 H_1 ... H_{nb-1}: apply H_{nb-1} first; window = entries t..t+m
    if (lane <= m) {
        const int q = lane;
        double2 w[LMAX];
#pragma unroll
        for (int j = 0; j < LMAX; ++j) {
            w[j] = cz();
            if (q < m && j == q + 1) w[j] = make_double2(1.0, 0.0);
        }
        if (q == m) w[0] = Y[nb - 1];
        for (int t = nb - 1; t >= 0; --t) {
            const double2 ts = Tau[t];
            double2 dp = cz();
            for (int j = 0; j < L; ++j) {
                const double2 uj = U[t][j];
                dp = cfma(make_double2(uj.x, -uj.y), w[j], dp);
            }
            const double2 td = cmul(ts, dp);
#pragma unroll
            for (int j = 0; j < LMAX; ++j)
                if (j < L) w[j] = csub(w[j], cmul(U[t][j], td));
            // entry t + m is final: block column index e = t + m
            {
                const int e = t + m;
                double2 v = cz();
#pragma unroll
                for (int j = 0; j < LMAX; ++j)
                    if (j == m) v = w[j];
                if (q == m) v = make_double2(-v.x, -v.y);
                const int prow = e < m ? nb + e : e - m;  // Pout row of block column e
                Po[(int64_t)prow * ms + q] = v;
            }
#pragma unroll
            for (int j = LMAX - 1; j > 0; --j) w[j] = w[j - 1];
            w[0] = (q == m && t > 0) ? Y[t - 1] : cz();
        }
        // remaining entries 0..m-1 (block columns 0..m-1 = state rows)
#pragma unroll
        for (int j = 0; j < LMAX; ++j) {
            if (j >= 1 && j <= m) {
                const int e = j - 1;
                double2 v = w[j];
                if (q == m) v = make_double2(-v.x, -v.y);
                const int prow = e < m ? nb + e : e - m;
                Po[(int64_t)prow * ms + q] = v;
            }
        }
        // w row: identity on the w column
        Po[(int64_t)(nb + m) * ms + q] = make_double2(q == m ? 1.0 : 0.0, 0.0);
    }
}

// ---------------------------------------------------------------------------
// wide windows (m + 1 > 32): the same per-window LQ, chain and forward
// substitution, with the block rows in shared memory instead of registers.
//   * chain (warp 0, lane = block row): R[i][e] holds block columns
//     e = 0..nb+m-1 of row i (e < m: the state z2, e >= m: panel column
//     e - m of A^T, lazy -sigma on the block diagonal); step t's window is
//     columns t..t+m of every row >= t.  The reflector vector u_t (L
//     entries) is written over row t's window once row t has retired (only
//     its diagonal, the pivot, is still needed, and it has been broadcast).
//   * reverse accumulation (all threads): G threads per vector (G = 4, 8, 16
//     for L <= 64, 128, 256), each holding 16 consecutive window entries in
//     registers; dot products reduce over the group with xor shuffles and
//     the window slides across the group with shfl_up.  Vectors are taken in
//     rounds of blockDim / G.
// Output Pout as k_lq.
// ---------------------------------------------------------------------------
constexpr int kLqBigThreads = 128;
constexpr int kLqBigHW = 16;  // window entries per thread of a group (64 registers)

__host__ __device__ inline int lq_big_rs(int nb, int m) { return (nb + m) | 1; }  // odd: conflict-free
__host__ __device__ inline size_t lq_big_smem(int nb, int m) {
    return ((size_t)32 * lq_big_rs(nb, m) + (m + 1) + 32 + 32 + 1) * 16;
}

template <int G>
__global__ void __launch_bounds__(kLqBigThreads) k_lq_big(TDims d, LqStep st, const double2* __restrict__ S,
                                                          double2* __restrict__ Pout) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int HW = kLqBigHW;
    const int m = d.m, L = m + 1, nb = st.nb, mp = d.mp;
    const int RS = lq_big_rs(nb, m);
    double2* R = reinterpret_cast<double2*>(smem);  // [32][RS]
    double2* Uu = R + 32 * RS;                      // [L] current reflector
    double2* Tau = Uu + L;                          // [32]
    double2* Y = Tau + 32;                          // [32]
    int* sfail = reinterpret_cast<int*>(Y + 32);
    const int l = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (d.fail[l] >= 0) return;  // failed in an earlier window: left as is (NaN at the end)
    const double2 sig = d.shifts[l];
    const int ms = d.ms;
    const double2* Sl = S + (int64_t)l * ms * d.LDS;
    double2* Po = Pout + (int64_t)l * (nb + ms) * ms;
    // stage the block rows: state columns (coalesced along rows), then the
    // panel of A^T (coalesced along columns: A^T(row, c) = A[c + row lda])
    for (int v = tid; v < nb * m; v += blockDim.x) {
        const int e = v / nb, i = v - e * nb;
        R[i * RS + e] = Sl[(int64_t)e * d.LDS + st.k0 + i];
    }
    for (int v = tid; v < nb * nb; v += blockDim.x) {
        const int i = v / nb, j = v - i * nb;
        double2 x = make_double2(d.A[st.c0 + j + (int64_t)(st.k0 + i) * d.lda], 0.0);
        if (i == m + j) x = csub(x, sig);  // block diagonal (lazy shift), solvers.py:398-400
        R[i * RS + m + j] = x;
    }
    // padding of a widened P (composites): zero rows nb + mp .. and columns mp ..
    for (int e = tid; e < (nb + ms) * (ms - mp); e += blockDim.x)
        Po[(int64_t)(e / (ms - mp)) * ms + mp + e % (ms - mp)] = cz();
    for (int e = tid; e < (ms - mp) * mp; e += blockDim.x) Po[(int64_t)(nb + mp + e / mp) * ms + e % mp] = cz();
    __syncthreads();
    if (warp == 0) {
        const bool mine = lane < nb;
        const double tol = d.tol[l];
        double2 y = mine ? Sl[(int64_t)m * d.LDS + st.k0 + lane] : cz();
        int fail = -1;
        for (int t = 0; t < nb; ++t) {
            double2* Rt = R + t * RS + t;
            // reflector of row t (pivot first): zlarfg on y = conj(row)
            double s2 = 0.0;
            for (int j = 1 + lane; j < L; j += 32) s2 = fma(Rt[j].x, Rt[j].x, fma(Rt[j].y, Rt[j].y, s2));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
            const double2 alpha = make_double2(Rt[0].x, -Rt[0].y);
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
            for (int j = lane; j < L; j += 32) {
                const double2 x = Rt[j];
                Uu[j] = j == 0 ? make_double2(1.0, 0.0) : cmul(make_double2(x.x, -x.y), scale);
            }
            __syncwarp();
            // rows t..nb-1 (row t included): r <- r - tau (r . u) conj(u)
            double2 r0 = cz();
            if (mine && lane >= t) {
                double2* rr = R + lane * RS + t;
                double2 d0 = cz(), d1 = cz();
                for (int j = 0; j < L; ++j) {
                    double2& dd = (j & 1) ? d1 : d0;
                    dd = cfma(rr[j], Uu[j], dd);
                }
                const double2 tw = cmul(tau, cadd(d0, d1));
                for (int j = 0; j < L; ++j) {
                    const double2 u = Uu[j];
                    double2 r = rr[j];
                    r.x = fma(-tw.x, u.x, fma(-tw.y, u.y, r.x));
                    r.y = fma(-tw.y, u.x, fma(tw.x, u.y, r.y));
                    rr[j] = r;
                }
                r0 = rr[0];
            }
            // forward substitution on the window's w segment (batched.py:170-178)
            const double2 piv = make_double2(__shfl_sync(0xffffffffu, r0.x, t), __shfl_sync(0xffffffffu, r0.y, t));
            if (fail < 0 && hypot(piv.x, piv.y) <= tol) fail = st.k0 + t;
            double2 yt = make_double2(__shfl_sync(0xffffffffu, y.x, t), __shfl_sync(0xffffffffu, y.y, t));
            yt = cdiv(yt, piv);
            if (lane == t) y = yt;
            if (mine && lane > t) y = csub(y, cmul(r0, yt));
            if (lane == 0) Tau[t] = tau;
            __syncwarp();
            for (int j = lane; j < L; j += 32) Rt[j] = Uu[j];  // row t retired: keep u_t
            __syncwarp();
        }
        if (mine) Y[lane] = y;
        if (lane == 0) *sfail = fail;
    }
    __syncthreads();
    if (*sfail >= 0) {
        if (tid == 0) d.fail[l] = *sfail;
        return;
    }
    // reverse accumulation: vector q < m is e_{nb+q}, vector m is [y; 0];
    // P = H_0 ... H_{nb-1}: H_{nb-1} first; window = block columns t..t+m
    const int gi = tid % G, base = gi * HW;
    const unsigned gmask = 0xffffffffu;
    for (int q0 = 0; q0 <= m; q0 += kLqBigThreads / G) {
        const int q = q0 + tid / G;
        const bool act = q <= m;
        double2 w[HW];
#pragma unroll
        for (int k = 0; k < HW; ++k)
            w[k] = make_double2(q < m && base + k == q + 1 ? 1.0 : 0.0, 0.0);
        if (q == m && gi == 0) w[0] = Y[nb - 1];
        for (int t = nb - 1; t >= 0; --t) {
            const double2* U = R + t * RS + t;
            double2 d0 = cz(), d1 = cz();
#pragma unroll
            for (int k = 0; k < HW; ++k) {
                if (base + k < L) {
                    const double2 u = U[base + k];
                    double2& dd = (k & 1) ? d1 : d0;
                    dd = cfma(make_double2(u.x, -u.y), w[k], dd);
                }
            }
            double2 dp = cadd(d0, d1);
#pragma unroll
            for (int o = 1; o < G; o <<= 1) {
                dp.x += __shfl_xor_sync(gmask, dp.x, o);
                dp.y += __shfl_xor_sync(gmask, dp.y, o);
            }
            const double2 td = cmul(Tau[t], dp);
            double2 fin = cz();
#pragma unroll
            for (int k = 0; k < HW; ++k) {
                if (base + k < L) w[k] = csub(w[k], cmul(U[base + k], td));
                if (base + k == m) fin = w[k];
            }
            // entry t + m (block column e = t + m >= m: Pout row t) is final
            if (act && base <= m && m < base + HW) {
                if (q == m) fin = make_double2(-fin.x, -fin.y);
                Po[(int64_t)t * ms + q] = fin;
            }
            // slide right by one across the group
            const double nx = __shfl_up_sync(gmask, w[HW - 1].x, 1);
            const double ny = __shfl_up_sync(gmask, w[HW - 1].y, 1);
#pragma unroll
            for (int k = HW - 1; k > 0; --k) w[k] = w[k - 1];
            w[0] = gi > 0 ? make_double2(nx, ny) : ((q == m && t > 0) ? Y[t - 1] : cz());
        }
        // remaining entries 1..m (block columns 0..m-1 = state rows)
        if (act) {
#pragma unroll
            for (int k = 0; k < HW; ++k) {
                const int j = base + k;
                if (j >= 1 && j <= m) {
                    double2 v = w[k];
                    if (q == m) v = make_double2(-v.x, -v.y);
                    Po[(int64_t)(nb + j - 1) * ms + q] = v;
                }
            }
            if (gi == 0) Po[(int64_t)(nb + m) * ms + q] = make_double2(q == m ? 1.0 : 0.0, 0.0);
        }
    }
}

// ---------------------------------------------------------------------------
// rows below the window (solvers.py:431-468): S <- S T + Pan U12, with
//   Pan(i, j) = A^T(i, c0 + j) for i < n, -[i - n == c0 + j] for i >= n,
// lazy-shift rows k0 + nb + (m - mnb) + dd: S -= sigma P12[nb - mnb + dd].
// One thread per row, all mp columns; panel tile staged in shared memory,
// the shift's P in shared memory too when it fits (PSM), else read through
// L1 (the same element for every thread: a broadcast).
// ---------------------------------------------------------------------------
__host__ inline size_t tupd_smem(int rows, bool psm, int nb, int mp) {
    return (size_t)nb * rows * 8 + (psm ? (size_t)(nb + mp) * mp * 16 : 0) + (size_t)mp * rows * 16;
}

template <int ROWS, bool PSM>
__global__ void __launch_bounds__(ROWS) k_tupd(TDims d, LqStep st, double2* __restrict__ S,
                                               const double2* __restrict__ Pbuf, int sg_size) {
    constexpr int kTuRows = ROWS;
    extern __shared__ __align__(16) unsigned char smem[];
    const int m = d.m, mp = d.mp, nb = st.nb;
    double* Pan = reinterpret_cast<double*>(smem);                                // [nb][kTuRows]
    double2* Psm = reinterpret_cast<double2*>(smem + (size_t)nb * kTuRows * 8);  // (nb+mp) x mp
    double2* Rb = Psm + (PSM ? (nb + mp) * mp : 0);                               // [mp][kTuRows] row copy
    const int rlo = st.k0 + nb;
    const int i = rlo + blockIdx.x * kTuRows + threadIdx.x;
    const int ihi = 2 * d.n;
    const int mnb = min(m, nb);
    const int crow0 = st.k0 + nb + (m - mnb);
    for (int v = threadIdx.x; v < nb * kTuRows; v += blockDim.x) {
        const int j = v / kTuRows, rr = v - j * kTuRows;
        const int ii = rlo + blockIdx.x * kTuRows + rr;
        double a = 0.0;
        if (ii < d.n) a = d.A[st.c0 + j + (int64_t)ii * d.lda];
        else if (ii < ihi && ii - d.n == st.c0 + j) a = -1.0;
        Pan[j * kTuRows + rr] = a;
    }
    const int l0 = blockIdx.y * sg_size, l1 = min(l0 + sg_size, d.sb);
    for (int l = l0; l < l1; ++l) {
        __syncthreads();
        if (d.fail[l] >= 0) continue;
        const double2* pl = Pbuf + (int64_t)l * (nb + mp) * mp;
        if (PSM)
            for (int v = threadIdx.x; v < (nb + mp) * mp; v += blockDim.x) Psm[v] = pl[v];
        const double2* Ps = PSM ? Psm : pl;
        __syncthreads();
        if (i >= ihi) continue;
        double2* Sl = S + (int64_t)l * mp * d.LDS;
        const double2 sig = d.shifts[l];
        for (int j = 0; j < mp; ++j) Rb[j * kTuRows + threadIdx.x] = Sl[(int64_t)j * d.LDS + i];
        const int dd = i - crow0;
        for (int c0 = 0; c0 < mp; c0 += 8) {
            double2 acc[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[c] = cz();
            for (int j = 0; j < mp; ++j) {
                const double2 sj = Rb[j * kTuRows + threadIdx.x];
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (c0 + c < mp) acc[c] = cfma(sj, Ps[(nb + j) * mp + c0 + c], acc[c]);
            }
            for (int j = 0; j < nb; ++j) {
                const double a = Pan[j * kTuRows + threadIdx.x];
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (c0 + c < mp) acc[c] = rfma(a, Ps[j * mp + c0 + c], acc[c]);
            }
            if (dd >= 0 && dd < mnb) {
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (c0 + c < mp) acc[c] = csub(acc[c], cmul(sig, Ps[(nb - mnb + dd) * mp + c0 + c]));
            }
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if (c0 + c < mp) Sl[(int64_t)(c0 + c) * d.LDS + i] = acc[c];
        }
    }
}

// ---------------------------------------------------------------------------
// unblocked tail (solvers.py:470-486): one CTA per shift
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_ttail(TDims d, double2* __restrict__ S, double2* __restrict__ X,
                                               int64_t ldx) {
    __shared__ double s_c;
    __shared__ double2 s_s, s_r, s_w;
    __shared__ int s_fail;
    const int l = blockIdx.x, tid = threadIdx.x;
    const int n = d.n, m = d.m;
    double2* Sl = S + (int64_t)l * d.ms * d.LDS;
    double2* wv = Sl + (int64_t)m * d.LDS;
    const int lo = n - m, hi = 2 * n;
    if (tid == 0) s_fail = d.fail[l];
    __syncthreads();
    const double tol = d.tol[l];
    if (s_fail < 0) {
        for (int kk = 1; kk < m && s_fail < 0; ++kk) {
            const int rr = n - m + kk - 1;
            double2* hcol = Sl + (int64_t)(kk - 1) * d.LDS;
            for (int c = kk; c < m; ++c) {
                double2* tcol = Sl + (int64_t)c * d.LDS;
                if (tid == 0) {
                    double cc;
                    double2 ss, rv;
                    givens(hcol[rr], tcol[rr], cc, ss, rv);
                    s_c = cc;
                    s_s = ss;
                    s_r = rv;
                }
                __syncthreads();
                const double cc = s_c;
                const double2 ss = s_s;
                for (int i = lo + tid; i < hi; i += blockDim.x) {
                    double2 h = hcol[i], t = tcol[i];
                    rot_apply(cc, ss, h, t);
                    hcol[i] = h;
                    tcol[i] = t;
                }
                __syncthreads();
                if (tid == 0) {
                    tcol[rr] = cz();
                    hcol[rr] = s_r;
                }
                __syncthreads();
            }
            if (tid == 0) {
                const double2 piv = hcol[rr];
                if (hypot(piv.x, piv.y) <= tol) {
                    s_fail = rr;
                } else {
                    s_w = cdiv(wv[rr], piv);
                    wv[rr] = s_w;
                }
            }
            __syncthreads();
            if (s_fail >= 0) break;
            const double2 wr = s_w;
            for (int i = rr + 1 + tid; i < hi; i += blockDim.x) wv[i] = csub(wv[i], cmul(hcol[i], wr));
            __syncthreads();
        }
        if (s_fail < 0) {
            double2* hcol = Sl + (int64_t)(m - 1) * d.LDS;
            if (tid == 0) {
                const double2 piv = hcol[n - 1];
                if (hypot(piv.x, piv.y) <= tol) {
                    s_fail = n - 1;
                } else {
                    s_w = cdiv(wv[n - 1], piv);
                    wv[n - 1] = s_w;
                }
            }
            __syncthreads();
            if (s_fail < 0) {
                const double2 wr = s_w;
                for (int i = n + tid; i < hi; i += blockDim.x) wv[i] = csub(wv[i], cmul(hcol[i], wr));
            }
        }
    }
    __syncthreads();
    const bool ok = s_fail < 0;
    const double qn = __longlong_as_double(0x7ff8000000000000ULL);
    for (int i = tid; i < n; i += blockDim.x)
        X[i + (int64_t)l * ldx] = ok ? wv[n + i] : make_double2(qn, qn);
    if (tid == 0) d.fail[l] = s_fail;
}

// The same tail for m <= 32 without m^2 / 2 passes over the 2n-row columns:
// the rotations and the substitution values depend only on the m x m top
// block (rows [n - m, n)), so warp 0 runs the whole tail on that block in
// shared memory (lane = row; same operations, same order as k_ttail) and
// records every rotation and every w; then each thread replays them on its
// rows of [n, 2n) with the row's m state values in a shared-memory slice
// (x = w[n:] is the only output; the state is not written back).
constexpr int kTtMax = 32;
__host__ __device__ inline size_t ttail_s_smem(int m) {
    return (size_t)m * 256 * 16 + (size_t)kTtMax * kTtMax * 16;
}
__global__ void __launch_bounds__(256) k_ttail_s(TDims d, const double2* __restrict__ S, double2* __restrict__ X,
                                                 int64_t ldx) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int NR = kTtMax * (kTtMax - 1) / 2;
    __shared__ double rc[NR];
    __shared__ double2 rs[NR], wk[kTtMax], wt[kTtMax];
    __shared__ int s_fail;
    double2* xs = reinterpret_cast<double2*>(smem);  // [m][256]: thread t's row values at j * 256 + t
    double2* Ts = xs + (size_t)d.m * 256;           // top block [column][kTtMax]
    const int l = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
    const int n = d.n, m = d.m;
    const double2* Sl = S + (int64_t)l * d.ms * d.LDS;
    const double2* wv = Sl + (int64_t)m * d.LDS;
    if (tid < 32) {
        int fail = d.fail[l];
        const double tol = d.tol[l];
        if (lane < m) {
            for (int j = 0; j < m; ++j) Ts[j * kTtMax + lane] = Sl[(int64_t)j * d.LDS + n - m + lane];
            wt[lane] = wv[n - m + lane];
        }
        __syncwarp();
        if (fail < 0) {
            int idx = 0;
            for (int kk = 1; kk < m && fail < 0; ++kk) {
                const int rl = kk - 1;
                double2* hc = Ts + (kk - 1) * kTtMax;
                for (int c = kk; c < m; ++c, ++idx) {
                    double2* tc = Ts + c * kTtMax;
                    double cc;
                    double2 ss, rv;
                    givens(hc[rl], tc[rl], cc, ss, rv);
                    __syncwarp();
                    if (lane < m) {
                        double2 hh = hc[lane], tt = tc[lane];
                        rot_apply(cc, ss, hh, tt);
                        hc[lane] = hh;
                        tc[lane] = tt;
                    }
                    __syncwarp();
                    if (lane == 0) {
                        tc[rl] = cz();
                        hc[rl] = rv;
                        rc[idx] = cc;
                        rs[idx] = ss;
                    }
                    __syncwarp();
                }
                const double2 piv = hc[rl];
                if (hypot(piv.x, piv.y) <= tol) {
                    fail = n - m + rl;
                    break;
                }
                const double2 w = cdiv(wt[rl], piv);
                __syncwarp();
                if (lane == 0) {
                    wt[rl] = w;
                    wk[rl] = w;
                }
                if (lane > rl && lane < m) wt[lane] = csub(wt[lane], cmul(hc[lane], w));
                __syncwarp();
            }
            if (fail < 0) {
                const double2 piv = Ts[(m - 1) * kTtMax + m - 1];
                if (hypot(piv.x, piv.y) <= tol) {
                    fail = n - 1;
                } else if (lane == 0) {
                    wk[m - 1] = cdiv(wt[m - 1], piv);
                }
            }
        }
        if (lane == 0) s_fail = fail;
    }
    __syncthreads();
    const int fail = s_fail;
    const double qn = __longlong_as_double(0x7ff8000000000000ULL);
    double2* Xl = X + (int64_t)l * ldx;
    if (fail >= 0) {
        for (int i = tid; i < n; i += blockDim.x) Xl[i] = make_double2(qn, qn);
        if (tid == 0) d.fail[l] = fail;
        return;
    }
    for (int i = n + tid; i < 2 * n; i += blockDim.x) {
        for (int j = 0; j < m; ++j) xs[j * 256 + tid] = Sl[(int64_t)j * d.LDS + i];
        double2 w = wv[i];
        int idx = 0;
        for (int kk = 1; kk < m; ++kk) {
            double2 hh = xs[(kk - 1) * 256 + tid];
            for (int c = kk; c < m; ++c, ++idx) {
                double2 tt = xs[c * 256 + tid];
                rot_apply(rc[idx], rs[idx], hh, tt);
                xs[c * 256 + tid] = tt;
            }
            w = csub(w, cmul(hh, wk[kk - 1]));
        }
        w = csub(w, cmul(xs[(m - 1) * 256 + tid], wk[m - 1]));
        Xl[i - n] = w;
    }
    if (tid == 0) d.fail[l] = -1;
}

__global__ void k_tol(int sb, const double2* __restrict__ shifts, const double* __restrict__ scal,
                      int n, double rtol, double* __restrict__ tol) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= sb) return;
    const double2 sg = shifts[l];
    const double sc2 = scal[0] - 2.0 * (sg.x * scal[1]) + (sg.x * sg.x + sg.y * sg.y) * n;
    tol[l] = rtol * sqrt(sc2 > 0.0 ? sc2 : 0.0);
}

template <typename F>
cudaError_t allow_smem(ss_handle* h, F* fn) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, fn);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(h->smem_optin - fa.sharedSizeBytes));
}

constexpr int kLqMaxL = 256;  // widest window (k_lq_big with 16 threads per vector)

int launch_lq(ss_handle* h, int m, int sb, cudaStream_t st, const TDims& d, const LqStep& s,
              const double2* S, double2* P) {
    const int L = m + 1;
    const size_t big = lq_big_smem(s.nb, m);
    if (L <= 2) k_lq<2><<<sb, 32, 0, st>>>(d, s, S, P);
    else if (L <= 4) k_lq<4><<<sb, 32, 0, st>>>(d, s, S, P);
    else if (L <= 8) k_lq<8><<<sb, 32, 0, st>>>(d, s, S, P);
    else if (L <= 12) k_lq<12><<<sb, 32, 0, st>>>(d, s, S, P);
    else if (L <= 16) k_lq<16><<<sb, 32, 0, st>>>(d, s, S, P);
    else if (L <= 24) k_lq<24><<<sb, 32, 0, st>>>(d, s, S, P);
    else if (L <= 32) k_lq<32><<<sb, 32, 0, st>>>(d, s, S, P);
    else if (L <= 4 * kLqBigHW) k_lq_big<4><<<sb, kLqBigThreads, big, st>>>(d, s, S, P);
    else if (L <= 8 * kLqBigHW) k_lq_big<8><<<sb, kLqBigThreads, big, st>>>(d, s, S, P);
    else if (L <= 16 * kLqBigHW) k_lq_big<16><<<sb, kLqBigThreads, big, st>>>(d, s, S, P);
    else return ss::set_err(h, SS_EARG, "transposed solve: m + 1 must be <= 256");
    SS_LAUNCH_CHECK(h);
    return SS_OK;
}

// rows-below update: the widest variant whose shared memory fits
int launch_tupd(ss_handle* h, cudaStream_t st, const TDims& d, const LqStep& s, double2* S,
                const double2* P, int rows_total) {
    const int sg = 8, nb = s.nb, mp = d.mp;
    const size_t cap = h->smem_optin;
    const unsigned gy = (unsigned)((d.sb + sg - 1) / sg);
    auto grid = [&](int r) { return dim3((unsigned)((rows_total + r - 1) / r), gy); };
    size_t sm;
    if ((sm = tupd_smem(128, true, nb, mp)) <= cap)
        k_tupd<128, true><<<grid(128), 128, sm, st>>>(d, s, S, P, sg);
    else if ((sm = tupd_smem(64, true, nb, mp)) <= cap)
        k_tupd<64, true><<<grid(64), 64, sm, st>>>(d, s, S, P, sg);
    else if ((sm = tupd_smem(64, false, nb, mp)) <= cap)
        k_tupd<64, false><<<grid(64), 64, sm, st>>>(d, s, S, P, sg);
    else if ((sm = tupd_smem(32, false, nb, mp)) <= cap)
        k_tupd<32, false><<<grid(32), 32, sm, st>>>(d, s, S, P, sg);
    else
        return ss::set_err(h, SS_EARG, "transposed solve: m too large for the row update");
    SS_LAUNCH_CHECK(h);
    return SS_OK;
}

}  // namespace

extern "C" int ss_solve_transposed(ss_handle* h, int n, int m, const double* Ahat, int64_t lda,
                                   const double* shifts, int64_t s, const double* rhs, int64_t ldr,
                                   int nb, int64_t batch, double rtol, double* X, int64_t ldx,
                                   int32_t* fail_row, void* stream) {
    if (!h) return SS_EARG;
    if (n < 1 || m < 1 || m > n || s < 0)
        return ss::set_err(h, SS_EDIM, "inconsistent controller-Hessenberg form");
    if (lda < n || ldr < n || ldx < n) return ss::set_err(h, SS_EDIM, "leading dimension too small");
    if (nb < 1) return ss::set_err(h, SS_EARG, "window block size must be >= 1");
    if (m + 1 > kLqMaxL) return ss::set_err(h, SS_EARG, "transposed solve: m + 1 must be <= 256");
    if (s == 0) return SS_OK;
    if (!Ahat || !shifts || !rhs || !X || !fail_row) return ss::set_err(h, SS_EARG, "null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    ss::DevGuard dg(h->device);
    SS_CUDA_TRY(h, dg.err);
    const double rt = std::isnan(rtol) ? 1e3 * n * 2.220446049250313e-16 : rtol;  // NaN: default
    int nb0 = std::max(1, std::min(std::min(nb, kLqMaxNb), std::max(n - m, 1)));
    // wide windows keep the block rows in shared memory: shrink the window to fit
    while (m + 1 > 32 && nb0 > 1 && lq_big_smem(nb0, m) > h->smem_optin) --nb0;
    const int mp = m + 1;
    const int64_t LDS = ((int64_t)2 * n + 7) & ~(int64_t)7;
    // ||A||_F^2 and trace(A) for the per-shift pivot tolerances
    {
        int rc = ss::fro2_trace(h, n, Ahat, lda, st);
        if (rc) return rc;
    }
    // Composites (as the forward sweep's window composites): up to kTrK
    // columns of windows, the rows below them updated ONCE by the K-streamed
    // far kernel; the state is padded to M = 10 ceil(mp / 10) columns for its
    // register tiles (zero columns stay zero: P and W are zero there)
    // For m a multiple of 10 the far pass is split instead (no padding): z2 on
    // k_fark at exactly m columns, w on k_farkm (ss_sweep.cu tr_far_split)
    const bool split = n - m > 2 * nb0 && ss::tr_split_supported(h, m);
    const int M = split ? mp : 10 * ((mp + 9) / 10);
    const bool comp = split || (M <= 60 && ss::tr_far_supported(h, M) && n - m > 2 * nb0);
    const int ms = comp ? M : mp;
    const int G = std::max(1, std::min(64, kTrK / nb0)), Kmax = G * nb0;
    const int64_t wstride = comp ? (int64_t)(Kmax + M) * M : 0;
    const int64_t wzstride = split ? (int64_t)(Kmax + m) * m : 0;                    // W of z2
    const int64_t gstride = split ? (int64_t)(Kmax + 1) * kFkmShiftsLq : 0;          // w column, per group
    // composites keep every window's P (the composite is built from all of
    // them at its end, k_wsuffix): G slabs
    const int nslab = comp ? G : 1;
    const size_t per_shift = (size_t)LDS * ms * 16 + (size_t)nslab * (nb0 + ms) * ms * 16 + (size_t)wstride * 16 +
                             (size_t)wzstride * 16 + (size_t)(Kmax + 1) * (split ? 16 : 0) + 8 + 64;
    int64_t sb_max = std::min<int64_t>(batch > 0 ? batch : s, s);
    if (per_shift * (size_t)sb_max + 256 > h->ws_bytes) {  // query only to grow (slow driver call)
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        const size_t cap = std::max<size_t>(fr / 2 + h->ws_bytes / 2, per_shift);
        sb_max = std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(sb_max, s),
                                                        (int64_t)(cap / per_shift)));
    }
    {
        const size_t slack = split ? (size_t)kFkmShiftsLq * (Kmax + 1) * 16 : 0;  // the last group of 80
        int rc = ss::ensure_ws(h, per_shift * (size_t)sb_max + 256 + slack, 0);
        if (rc) return rc;
    }
    double2* Sb = (double2*)h->ws;
    double2* Pb = Sb + (size_t)sb_max * ms * LDS;
    const int64_t pslab = (int64_t)sb_max * (nb0 + ms) * ms;  // one window's P of the batch
    double2* Wb = Pb + (size_t)nslab * pslab;
    double2* Wzb = Wb + (size_t)sb_max * wstride;
    double2* Wwb = Wzb + (size_t)sb_max * wzstride;  // ceil(sb / 80) groups (per_shift holds Kmax + 1 each + slack)
    const size_t ngroups_max = split ? (size_t)((sb_max + kFkmShiftsLq - 1) / kFkmShiftsLq) : 0;
    double* tolb = (double*)(Wwb + ngroups_max * gstride);
    static ss::DevMask attrs;  // devices configured
    if (!attrs.has(h)) {
        SS_CUDA_TRY(h, allow_smem(h, k_tupd<128, true>));
        SS_CUDA_TRY(h, allow_smem(h, k_tupd<64, true>));
        SS_CUDA_TRY(h, allow_smem(h, k_tupd<64, false>));
        SS_CUDA_TRY(h, allow_smem(h, k_tupd<32, false>));
        SS_CUDA_TRY(h, allow_smem(h, k_lq_big<4>));
        SS_CUDA_TRY(h, allow_smem(h, k_lq_big<8>));
        SS_CUDA_TRY(h, allow_smem(h, k_lq_big<16>));
        attrs.set(h);
    }
    for (int64_t lo = 0; lo < s; lo += sb_max) {
        const int sb = (int)std::min<int64_t>(sb_max, s - lo);
        TDims d;
        d.n = n;
        d.m = m;
        d.mp = mp;
        d.ms = ms;
        d.A = Ahat;
        d.lda = lda;
        d.shifts = (const double2*)shifts + lo;
        d.sb = sb;
        d.LDS = LDS;
        d.fail = fail_row + lo;
        d.tol = tolb;
        k_tol<<<(sb + 127) / 128, 128, 0, st>>>(sb, d.shifts, h->d_scal, n, rt, tolb);
        SS_LAUNCH_CHECK(h);
        {
            dim3 g((unsigned)((LDS + 255) / 256), (unsigned)sb);
            k_tseed<<<g, 256, 0, st>>>(d, (const double2*)rhs + lo * ldr, ldr, Sb);
            SS_LAUNCH_CHECK(h);
        }
        for (int k0 = 0; comp && k0 < n - m;) {
            // ---- one composite: windows top-down, near rows, fold; far pass ----
            int k0w[64], nbw[64], g = 0;
            for (int kk = k0; kk < n - m && g < G; ++g) {
                k0w[g] = kk;
                nbw[g] = std::min(nb0, n - m - kk);
                kk += nbw[g];
            }
            const int c0 = k0 + m;                       // first panel column
            const int kend = k0w[g - 1] + nbw[g - 1];    // first far row
            const int K = kend - k0;                     // panel columns of the composite
            int xw[64];
            for (int b = 0; b < g; ++b) {
                LqStep ls;
                ls.k0 = k0w[b];
                ls.nb = nbw[b];
                ls.c0 = k0w[b] + m;
                xw[b] = k0w[b] - k0;
                double2* Pw = Pb + (size_t)b * pslab;  // this window's P slab
                cudaEvent_t ev = ss::timing_begin(h, st);
                int rc = launch_lq(h, m, sb, st, d, ls, Sb, Pw);
                if (rc) return rc;
                ss::timing_end(h, st, ev, ss::PH_RQ);
                const int rows = kend - (ls.k0 + ls.nb);  // near: the composite's rows below this window
                if (rows > 0) {
                    UpdDims u;
                    u.n = n;
                    u.m = M;
                    u.ptop = 0;
                    u.ident_top = 0;
                    u.A = Ahat;
                    u.lda = lda;
                    u.T = nullptr;
                    u.ldt = 0;
                    u.shifts = d.shifts;
                    u.sb = sb;
                    u.LDZ = LDS;
                    u.nb = ls.nb;
                    u.mnb = std::min(m, ls.nb);
                    u.r0 = kend;
                    u.c0 = ls.c0;
                    u.nc = ls.nb + M;
                    u.rlo = ls.k0 + ls.nb;
                    u.lz0 = ls.k0 + ls.nb + (m - u.mnb);
                    u.lzp = ls.nb - u.mnb;
                    ev = ss::timing_begin(h, st);
                    rc = ss::launch_update_tr(h, u, rows, Sb, Pw, st);
                    if (rc) return rc;
                    ss::timing_end(h, st, ev, ss::PH_UPDATE, 8.0 * rows * M * M * (double)sb,
                                   8.0 * rows * (double)sb * M * ls.nb, 4.0 * mp * (double)rows * ls.nb * sb);
                }
            }
            {
                cudaEvent_t ev = ss::timing_begin(h, st);
                int rc = ss::wsuffix(h, st, sb, g, xw, nbw, M, mp, K, Pb, pslab, Wb, wstride);
                if (rc) return rc;
                ss::timing_end(h, st, ev, ss::PH_BATCHED_GEMM);
            }
            // far rows: the rest of A^T's rows and the -I rows up to the
            // composite's last column
            const int rend = std::min(2 * n, n + c0 + K);
            int rc = split ? ss::tr_far_split(h, st, n, m, Ahat, lda, d.shifts, sb, Sb, LDS, kend, rend, c0, K, Wb,
                                              wstride, Wzb, wzstride, Wwb, gstride)
                           : ss::tr_far(h, st, n, m, M, Ahat, lda, d.shifts, sb, Sb, LDS, kend, rend, c0, K, Wb,
                                        wstride);
            if (rc) return rc;
            k0 = kend;
        }
        for (int k0 = 0; !comp && k0 < n - m;) {
            LqStep ls;
            ls.k0 = k0;
            ls.nb = std::min(nb0, n - m - k0);
            ls.c0 = k0 + m;
            cudaEvent_t ev = ss::timing_begin(h, st);
            int rc = launch_lq(h, m, sb, st, d, ls, Sb, Pb);
            if (rc) return rc;
            ss::timing_end(h, st, ev, ss::PH_RQ);
            // rows below the window with a nonzero state or panel entry: all of
            // A^T's, and the -I rows up to this window's last column (the rest
            // of the stacked state is still the seed's zero)
            const int rend = std::min(2 * n, n + ls.c0 + ls.nb);
            const int rows = rend - (k0 + ls.nb);
            ev = ss::timing_begin(h, st);
            {
                UpdDims u;
                u.n = n;
                u.m = mp;
                u.ptop = 0;
                u.ident_top = 0;
                u.A = Ahat;
                u.lda = lda;
                u.T = nullptr;
                u.ldt = 0;
                u.shifts = d.shifts;
                u.sb = sb;
                u.LDZ = LDS;
                u.nb = ls.nb;
                u.mnb = std::min(m, ls.nb);
                u.r0 = rend;
                u.c0 = ls.c0;
                u.nc = ls.nb + mp;
                u.rlo = k0 + ls.nb;
                u.lz0 = k0 + ls.nb + (m - u.mnb);
                u.lzp = ls.nb - u.mnb;
                // the window-update kernel covers <= 10 column blocks of 10
                // (mp <= 100); wider states keep the row-per-thread k_tupd
                if (rows <= 0) rc = SS_OK;
                else if (mp <= 100) rc = ss::launch_update_tr(h, u, rows, Sb, Pb, st);
                else rc = launch_tupd(h, st, d, ls, Sb, Pb, rows);
            }
            if (rc) return rc;
            const double fl_b = (double)sb * 8.0 * rows * mp * mp;
            const double fl_o = (double)sb * 8.0 * rows * mp * ls.nb;
            h->flops[ss::PH_BATCHED_GEMM] += fl_b;
            h->flops[ss::PH_OUTER_GEMM] += fl_o;
            ss::timing_end(h, st, ev, ss::PH_UPDATE, fl_b, fl_o, 0.0);
            k0 += ls.nb;
        }
        cudaEvent_t ev = ss::timing_begin(h, st);
        if (m <= kTtMax && ttail_s_smem(m) + 8192 <= h->smem_optin) {
            static ss::DevMask configured;
            if (!configured.has(h)) {
                SS_CUDA_TRY(h, allow_smem(h, k_ttail_s));
                configured.set(h);
            }
            k_ttail_s<<<sb, 256, ttail_s_smem(m), st>>>(d, Sb, (double2*)X + lo * ldx, ldx);
        } else {
            k_ttail<<<sb, 256, 0, st>>>(d, Sb, (double2*)X + lo * ldx, ldx);
        }
        SS_LAUNCH_CHECK(h);
        ss::timing_end(h, st, ev, ss::PH_TAIL);
    }
    return SS_OK;
}
