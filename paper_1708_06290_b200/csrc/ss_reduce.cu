// One-time reduction of (A, B, C) to controller-Hessenberg form on sm_100a.
//
// Reference: hessenberg.py:260-328 (reduce_controller_hessenberg) with the
// two-level blocked band reduction of hessenberg.py:83-245.  Same
// reflectors (kernels.py:74-99 sign convention), so Ahat/Bhat/Chat agree
// with the reference to rounding:
//
//  1. QR of B by Householder columns; the m reflectors form one compact-WY
//     block (V_B, T_B) that is applied to A from both sides and to C from
//     the right with GEMMs (the reference applies them one by one,
//     hessenberg.py:297-315; the product is the same).
//  2. Band reduction in panels of `block_size` columns.  Per panel column:
//     the column receives the right update of the panel's earlier
//     mini-blocks (Y V^T) and the left update (I - V T^T V^T), then its
//     reflector is generated and the T factor grows (reference
//     _process_panel, hessenberg.py:99-146).  These run as one persistent
//     cooperative kernel per mini-block (k_panel, ss_panel.cuh: two grid
//     barriers per column instead of six launches).  Every m columns (a
//     "mini-block", mini_boundaries hessenberg.py:83-96) Y = A V T is
//     extended by one GEMM over the trailing matrix -- the band-width trick
//     that reads the trailing matrix n/m times instead of n times.  After the
//     panel the trailing updates (tasks (a), (b), (c) of
//     hessenberg.py:149-193) and the C / Q right updates are GEMMs.
//
// All dense contractions go through k_dmma (ss_gemm.cuh), a hand-written
// FP64 tensor-core GEMM (mma.sync m16n8k8 .f64, i.e. DMMA, cp.async ring,
// deterministic split-K) -- the only place DMMA is used.  Every reduction
// runs in a fixed order, so results are run-to-run reproducible.
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "ss_internal.h"
#include "ss_gemm.cuh"
#include "ss_panel.cuh"

namespace {

__global__ void k_zero(double* p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = 0.0;
}

__global__ void k_zero_mat(double* p, int rows, int cols, int64_t ld) {
    const int64_t tot = (int64_t)rows * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / rows, r = e - c * rows;
        p[r + c * ld] = 0.0;
    }
}

__global__ void k_eye(double* p, int n, int64_t ld) {
    const int64_t tot = (int64_t)n * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / n, r = e - c * n;
        p[r + c * ld] = r == c ? 1.0 : 0.0;
    }
}

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
struct Ctx {
    ss_handle* h;
    cudaStream_t st;
    double* split = nullptr;  // split-K partial tiles
    size_t split_cap = 0;     // doubles
};

template <bool TA, bool TB, int MT, int NT, int WM, int WN, int BK = ssr::kGBK>
int gemm_launch(Ctx& x, const ssr::GemmArgs& g, dim3 grid) {
    using Cfg = ssr::GemmCfg<TA, TB, MT, NT, WM, WN, BK>;
    static ss::DevMask configured;  // devices configured
    if (!configured.has(x.h)) {
        SS_CUDA_TRY(x.h, cudaFuncSetAttribute(ssr::k_dmma<TA, TB, MT, NT, WM, WN, false, BK>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
        SS_CUDA_TRY(x.h, cudaFuncSetAttribute(ssr::k_dmma<TA, TB, MT, NT, WM, WN, true, BK>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
        configured.set(x.h);
    }
    // 16-byte copies when both operands' base pointers and leading dimensions are even
    const bool v16 = ((uintptr_t)g.A % 16 == 0) && ((uintptr_t)g.B % 16 == 0) && g.lda % 2 == 0 && g.ldb % 2 == 0;
    if (v16)
        ssr::k_dmma<TA, TB, MT, NT, WM, WN, true, BK><<<grid, ssr::kGThreads, Cfg::SMEM, x.st>>>(g);
    else
        ssr::k_dmma<TA, TB, MT, NT, WM, WN, false, BK><<<grid, ssr::kGThreads, Cfg::SMEM, x.st>>>(g);
    SS_LAUNCH_CHECK(x.h);
    return SS_OK;
}

template <bool TA, bool TB>
int gemm_t(Ctx& x, ssr::GemmArgs g) {
    // tile shape from the output shape: narrow outputs (the Y extension's
    // A0 V, M V) take narrow N tiles, short M (V^T M) a 64-row tile
    int BM = 128, BN = 64, shape = 2;
    // narrow N (the Y extension's A0 V has N = m): the N tile is the number of
    // n8 DMMA tiles the output needs
    if (g.N <= 8) { BN = 8; shape = 0; }
    else if (g.N <= 16) { BN = 16; shape = 5; }
    else if (g.N <= 24) { BN = 24; shape = 6; }
    else if (g.N <= 32) { BN = 32; shape = 1; }
    else if (g.N <= 64) { BN = 64; shape = 2; }
    else if (g.M <= 64) { BM = 64; BN = 64; shape = 4; }  // V^T M: 64 x 64 tiles (22.4 vs 12.2 TF/s with 64 x 128)
    // else 128 x 64 at two CTAs per SM (n = 20000: 1.99 s vs 2.12 s with 128 x 128 at one)
    const int64_t tiles = (int64_t)((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN);
    const int nkt = (g.K + ssr::kGBK - 1) / ssr::kGBK;
    // split K when the output has too few tiles to fill the SMs
    int ks = 1;
    const int64_t want = 2 * (int64_t)x.h->num_sms;
    if (tiles < want && nkt >= 32) {
        ks = (int)std::min<int64_t>({(want + tiles - 1) / tiles, nkt / 16, 32});
        while (ks > 1 && (size_t)ks * g.M * g.N > x.split_cap) --ks;
        ks = std::max(ks, 1);
    }
    g.ksplit = ks;
    g.part = x.split;
    dim3 grid((unsigned)((g.M + BM - 1) / BM), (unsigned)((g.N + BN - 1) / BN), (unsigned)ks);
    int rc;
    switch (shape) {
        case 0: rc = gemm_launch<TA, TB, 1, 1, 8, 1>(x, g, grid); break;
        case 1: rc = gemm_launch<TA, TB, 1, 4, 8, 1>(x, g, grid); break;
        case 4: rc = gemm_launch<TA, TB, 1, 4, 4, 2>(x, g, grid); break;
        case 5: rc = gemm_launch<TA, TB, 1, 2, 8, 1>(x, g, grid); break;
        case 6: rc = gemm_launch<TA, TB, 1, 3, 8, 1>(x, g, grid); break;
        default: rc = gemm_launch<TA, TB, 2, 4, 4, 2>(x, g, grid); break;
    }
    if (rc) return rc;
    if (ks > 1) {
        const int64_t tot = (int64_t)g.M * g.N;
        const int blocks = (int)std::min<int64_t>((tot + 255) / 256, 4 * (int64_t)x.h->num_sms);
        ssr::k_gemm_splitk_reduce<<<blocks, 256, 0, x.st>>>(g);
        SS_LAUNCH_CHECK(x.h);
    }
    return SS_OK;
}

int gemm(Ctx& x, bool ta, bool tb, int M, int N, int K, double alpha, const double* A, int64_t lda,
         const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
    if (M <= 0 || N <= 0) return SS_OK;
    ssr::GemmArgs g{M, N, K, alpha, beta, A, lda, B, ldb, C, ldc, 1, nullptr};
    if (!ta && !tb) return gemm_t<false, false>(x, g);
    if (!ta && tb) return gemm_t<false, true>(x, g);
    if (ta && !tb) return gemm_t<true, false>(x, g);
    return gemm_t<true, true>(x, g);
}

#define SS_TRY(expr)            \
    do {                        \
        int _rc = (expr);       \
        if (_rc) return _rc;    \
    } while (0)

// Apply Q = I - V T V^T (V: rows x k, ld ldv) to M from the right:
// M[:, 0:rows] <- M (I - V T V^T), M has mrows rows.  Work: W1 = M V, W2 = W1 T.
int apply_right(Ctx& x, double* M, int64_t ldm, int mrows, const double* V, int64_t ldv,
                const double* T, int64_t ldt, int rows, int k, double* W1, double* W2, int64_t ldw) {
    if (mrows <= 0 || rows <= 0 || k <= 0) return SS_OK;
    SS_TRY(gemm(x, false, false, mrows, k, rows, 1.0, M, ldm, V, ldv, 0.0, W1, ldw));
    SS_TRY(gemm(x, false, false, mrows, k, k, 1.0, W1, ldw, T, ldt, 0.0, W2, ldw));
    SS_TRY(gemm(x, false, true, mrows, rows, k, -1.0, W2, ldw, V, ldv, 1.0, M, ldm));
    return SS_OK;
}

// M[0:rows, :] <- (I - V T^T V^T) M, M has mcols columns.  W (k x mcols, ld ldw).
int apply_left(Ctx& x, double* M, int64_t ldm, int mcols, const double* V, int64_t ldv,
               const double* T, int64_t ldt, int rows, int k, double* W1, double* W2, int64_t ldw) {
    if (mcols <= 0 || rows <= 0 || k <= 0) return SS_OK;
    SS_TRY(gemm(x, true, false, k, mcols, rows, 1.0, V, ldv, M, ldm, 0.0, W1, ldw));
    SS_TRY(gemm(x, true, false, k, mcols, k, 1.0, T, ldt, W1, ldw, 0.0, W2, ldw));
    SS_TRY(gemm(x, false, false, rows, mcols, k, -1.0, V, ldv, W2, ldw, 1.0, M, ldm));
    return SS_OK;
}

// One mini-block [js, jb) of panel columns: the cooperative panel kernel
// (ss_panel.cuh), one CTA per SM.
int panel_cols(Ctx& x, ssr::Pan& p, int js, int jb) {
    static ss::DevMask configured;  // devices configured
    if (!configured.has(x.h)) {
        SS_CUDA_TRY(x.h, cudaFuncSetAttribute(ssr::k_panel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)x.h->smem_optin));
        SS_CUDA_TRY(x.h, cudaFuncSetAttribute(ssr::k_panel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)x.h->smem_optin));
        SS_CUDA_TRY(x.h, cudaFuncSetAttribute(ssr::k_panel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        configured.set(x.h);
    }
    // small panels: one cluster of kPCl CTAs (hardware cluster barriers and
    // distributed-shared-memory sums); large: every SM, grid barriers
    // (not with the in-kernel Y extension: its A0 V stream wants every SM)
    const bool cl = !p.yin && p.nk <= ssr::kPCl * ssr::kPClRows;
    const int G = cl ? ssr::kPCl : x.h->num_sms;
    // the CTAs' own rows of V and Y in shared memory when they fit
    const int nown = (p.nk + G - 1) / G;
    int stage = ssr::pan_smem_bytes(p.bw, G, nown, cl) <= x.h->smem_optin ? 1 : 0;
    const size_t smem = ssr::pan_smem_bytes(p.bw, G, stage ? nown : 0, cl);
    if (smem > x.h->smem_optin) return ss::set_err(x.h, SS_EARG, "reduction: panel too wide for shared memory");
    if (cl) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ssr::kPCl);
        cfg.blockDim = dim3(ssr::kPT);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = x.st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = ssr::kPCl;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        SS_CUDA_TRY(x.h, cudaLaunchKernelEx(&cfg, ssr::k_panel<true>, p, js, jb, stage));
    } else {
        void* args[] = {(void*)&p, (void*)&js, (void*)&jb, (void*)&stage};
        SS_CUDA_TRY(x.h, cudaLaunchCooperativeKernel((const void*)ssr::k_panel<false>, dim3(G), dim3(ssr::kPT),
                                                     args, smem, x.st));
    }
    x.h->launches++;
    return SS_OK;
}

}  // namespace

// The reduction's DMMA GEMM behind the C ABI (diagnostics / tests):
// C = alpha op(A) op(B) + beta C, column-major, op = transpose if ta / tb.
extern "C" int ss_dgemm(ss_handle* h, int ta, int tb, int M, int N, int K, double alpha, const double* A,
                        int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                        void* stream) {
    if (!h) return SS_EARG;
    if (M < 0 || N < 0 || K < 0) return ss::set_err(h, SS_EDIM, "negative dimension");
    if (ldc < std::max(M, 1) || lda < std::max(ta ? K : M, 1) || ldb < std::max(tb ? N : K, 1))
        return ss::set_err(h, SS_EDIM, "leading dimension too small");
    ss::DevGuard dg(h->device);
    SS_CUDA_TRY(h, dg.err);
    Ctx x{h, (cudaStream_t)stream};
    const size_t split_cap = (size_t)8 << 20;
    SS_TRY(ss::ensure_ws(h, split_cap * sizeof(double), 1));
    x.split = (double*)h->ws2;
    x.split_cap = split_cap;
    return gemm(x, ta != 0, tb != 0, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
}

extern "C" int ss_reduce_chf(ss_handle* h, int n, int m, int p, double* A, int64_t lda, double* B,
                             int64_t ldb, double* C, int64_t ldc, double* Q, int64_t ldq,
                             int block_size, void* stream) {
    if (!h) return SS_EARG;
    if (n < 1 || m < 1 || m >= n || p < 0)
        return ss::set_err(h, SS_EDIM, "need 1 <= m < n (inputs vs state dimension)");
    if (lda < n || ldb < n || (p > 0 && ldc < p) || (Q && ldq < n))
        return ss::set_err(h, SS_EDIM, "leading dimension too small");
    if (block_size < 1) return ss::set_err(h, SS_EARG, "block_size must be positive");
    if (!A || !B || (p > 0 && !C)) return ss::set_err(h, SS_EARG, "null pointer");
    ss::DevGuard dg(h->device);
    SS_CUDA_TRY(h, dg.err);
    cudaStream_t st = (cudaStream_t)stream;
    Ctx x{h, st};
    cudaEvent_t e0 = ss::timing_begin(h, st);
    const int b = std::min(block_size, 128);
    const int bw_max = std::max(b, m);
    // workspace: V, Y (n x bw), T (bw x bw), W1/W2 (max(n,p) x max(bw, n) as needed), partials
    const int64_t ldv = n;
    const int64_t ldw = std::max<int64_t>(std::max(n, p), 1);
    size_t need = 0;
    need += (size_t)ldv * bw_max;        // V
    need += (size_t)ldv * bw_max;        // Y (bottom)
    need += (size_t)bw_max * bw_max;     // T
    need += (size_t)ldw * bw_max * 2;    // W1, W2 for right updates (mrows x k)
    need += (size_t)bw_max * n * 2;      // W1, W2 for left updates (k x mcols)
    need += ssr::pan_ws_doubles(h->num_sms);  // panel kernel partials
    const size_t split_cap = (size_t)8 << 20;    // split-K partials (64 MB)
    need += split_cap;
    SS_TRY(ss::ensure_ws(h, need * sizeof(double), 1));
    double* V = (double*)h->ws2;
    double* Y = V + (size_t)ldv * bw_max;
    double* T = Y + (size_t)ldv * bw_max;
    const int64_t ldt = bw_max;
    double* W1 = T + (size_t)bw_max * bw_max;
    double* W2 = W1 + (size_t)ldw * bw_max;
    double* L1 = W2 + (size_t)ldw * bw_max;
    double* L2 = L1 + (size_t)bw_max * n;
    double* pws = L2 + (size_t)bw_max * n;
    x.split = pws + ssr::pan_ws_doubles(h->num_sms);
    x.split_cap = split_cap;
    const int64_t ldl = bw_max;
    if (b > ssr::kPBmax || m > ssr::kPBmax) return ss::set_err(h, SS_EARG, "reduction: block size / m > 128");

    if (Q) {
        k_eye<<<256, 256, 0, st>>>(Q, n, ldq);
        SS_LAUNCH_CHECK(h);
    }

    // ---- 1. QR of B (hessenberg.py:297-315) as one compact-WY block ----
    const int kB = std::min(m, n - 1);
    k_zero_mat<<<128, 256, 0, st>>>(V, n, kB, ldv);
    SS_LAUNCH_CHECK(h);
    k_zero_mat<<<16, 256, 0, st>>>(T, kB, kB, ldt);
    SS_LAUNCH_CHECK(h);
    {
        ssr::Pan pp;
        pp.a0 = B;
        pp.lda = ldb;
        pp.nk = n;
        pp.bw = kB;
        pp.m = kB;
        pp.yext = 0;
        pp.vrow0 = 0;
        pp.V = V;
        pp.Y = Y;
        pp.ldv = ldv;
        pp.T = T;
        pp.ldt = ldt;
        pp.ws = pws;
        pp.tr = nullptr;
        pp.yin = 0;
        SS_TRY(panel_cols(x, pp, 0, kB));
    }
    // Bhat[m:, :] = 0 exactly (hessenberg.py:315) and the columns past kB
    // (only when m == n, excluded above) need no work.
    // A <- Q_B^T A Q_B ; C <- C Q_B  (Q_B = I - V T V^T)
    SS_TRY(apply_left(x, A, lda, n, V, ldv, T, ldt, n, kB, L1, L2, ldl));
    SS_TRY(apply_right(x, A, lda, n, V, ldv, T, ldt, n, kB, W1, W2, ldw));
    if (p > 0) SS_TRY(apply_right(x, C, ldc, p, V, ldv, T, ldt, n, kB, W1, W2, ldw));
    if (Q) SS_TRY(apply_right(x, Q, ldq, n, V, ldv, T, ldt, n, kB, W1, W2, ldw));

    // ---- 2. blocked band reduction (hessenberg.py:196-245) ----
    const int ncols = std::max(n - m - 1, 0);
    for (int zc = 0; zc < ncols; zc += b) {
        const int bw = std::min(b, ncols - zc);
        const int kb = zc + m;
        const int nk = n - kb;
        k_zero_mat<<<128, 256, 0, st>>>(V, nk, bw, ldv);
        SS_LAUNCH_CHECK(h);
        k_zero_mat<<<16, 256, 0, st>>>(T, bw, bw, ldt);
        SS_LAUNCH_CHECK(h);
        ssr::Pan pp;
        pp.a0 = A + kb + (int64_t)zc * lda;
        pp.lda = lda;
        pp.nk = nk;
        pp.bw = bw;
        pp.m = m;
        pp.yext = 1;
        pp.vrow0 = zc - kb;  // V row of column j's right update: col - kb = j - m
        pp.V = V;
        pp.Y = Y;
        pp.ldv = ldv;
        pp.T = T;
        pp.ldt = ldt;
        pp.ws = pws;
        pp.tr = A + kb + (int64_t)kb * lda;
        pp.yin = m <= ssr::kPYin ? 1 : 0;
        if (pp.yin) {
            // small m: the Y extension inside the panel kernel, one launch per panel
            SS_TRY(panel_cols(x, pp, 0, bw));
        }
        int js = 0;  // first reflector of the current mini-block
        for (int j = 0; j < bw && !pp.yin; ++j) {
            const int jb = j + 1;
            if (jb % m == 0 || jb == bw) {
                // panel columns [js, jb) (right update from the complete
                // mini-blocks, reflectors i <= j - m), then Y for them
                SS_TRY(panel_cols(x, pp, js, jb));
                // Y[:, js:jb] = (A0[kb:, kb+js:] V[js:, js:jb] - Y[:, :js] (V[:, :js]^T V[:, js:jb])) T[js:jb, js:jb]
                const int cw = jb - js;
                SS_TRY(gemm(x, false, false, nk, cw, nk - js, 1.0, A + kb + (int64_t)(kb + js) * lda, lda,
                            V + js + (int64_t)js * ldv, ldv, 0.0, W1, ldw));
                if (js > 0) {
                    SS_TRY(gemm(x, true, false, js, cw, nk, 1.0, V, ldv, V + (int64_t)js * ldv, ldv, 0.0,
                                L1, ldl));
                    SS_TRY(gemm(x, false, false, nk, cw, js, -1.0, Y, ldv, L1, ldl, 1.0, W1, ldw));
                }
                SS_TRY(gemm(x, false, false, nk, cw, cw, 1.0, W1, ldw, T + js + (int64_t)js * ldt, ldt,
                            0.0, Y + (int64_t)js * ldv, ldv));
                js = jb;
            }
        }
        // task (c): rows 0..kb, right update of columns kb..n via Ytop = A[0:kb, kb:] V T
        if (kb > 0) SS_TRY(apply_right(x, A + (int64_t)kb * lda, lda, kb, V, ldv, T, ldt, nk, bw, W1, W2, ldw));
        // tasks (a)+(b): rows kb..n, trailing columns zc+bw..n
        // (a) right: columns with reflector support, max(zc+bw, kb).. (hessenberg.py:149-160)
        const int col0 = std::max(zc + bw, kb);
        if (col0 < n) {
            const int vrow0 = col0 - kb;
            SS_TRY(gemm(x, false, true, nk, n - col0, bw, -1.0, Y, ldv, V + vrow0, ldv, 1.0,
                        A + kb + (int64_t)col0 * lda, lda));
        }
        // (b) left: every column right of the panel, zc+bw..n (hessenberg.py:161-164)
        const int lcol0 = zc + bw;
        if (lcol0 < n)
            SS_TRY(apply_left(x, A + kb + (int64_t)lcol0 * lda, lda, n - lcol0, V, ldv, T, ldt, nk, bw,
                              L1, L2, ldl));
        if (p > 0) SS_TRY(apply_right(x, C + (int64_t)kb * ldc, ldc, p, V, ldv, T, ldt, nk, bw, W1, W2, ldw));
        if (Q) SS_TRY(apply_right(x, Q + (int64_t)kb * ldq, ldq, n, V, ldv, T, ldt, nk, bw, W1, W2, ldw));
    }
    // exact zero patterns (hessenberg.py:125-126, 315)
    if (m < n) {
        k_zero_mat<<<64, 256, 0, st>>>(B + m, n - m, m, ldb);
        SS_LAUNCH_CHECK(h);
    }
    ss::timing_end(h, st, e0, ss::PH_REDUCTION);
    // reference flop count: 10/3 n^3 + 5/2 n^2 b - 9/2 n^2 m + n^2 m^2/(2b)
    const double dn = n, db = b, dm = m;
    h->flops[ss::PH_REDUCTION] += 10.0 / 3.0 * dn * dn * dn + 2.5 * dn * dn * db - 4.5 * dn * dn * dm +
                                  dn * dn * dm * dm / (2.0 * db);
    return SS_OK;
}
