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
//     _process_panel, hessenberg.py:99-146).  Every m columns (a "mini-block",
//     mini_boundaries hessenberg.py:83-96) Y = A V T is extended by one GEMM
//     over the trailing matrix -- the band-width trick that reads the
//     trailing matrix n/m times instead of n times.  After the panel the
//     trailing updates (tasks (a), (b), (c) of hessenberg.py:149-193) and the
//     C / Q right updates are GEMMs.
//
// All dense contractions go through k_dgemm, a hand-written FP64 tensor-core
// GEMM (mma.sync m16n8k8 .f64, i.e. DMMA) -- the only place DMMA is used.
// Per-column vector work runs in small multi-CTA kernels with deterministic
// (fixed-order) partial reductions, so results are run-to-run reproducible.
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "ss_internal.h"

namespace {

// ---------------------------------------------------------------------------
// FP64 GEMM on DMMA:  C = alpha op(A) op(B) + beta C   (column-major)
// CTA tile 64x64x16, 4 warps each 32x32 (2 x 4 m16n8k8 tiles).
// ---------------------------------------------------------------------------
constexpr int GBM = 64, GBN = 64, GBK = 16, GS = 68;  // GS = 4 mod 16: conflict-free frags

__device__ __forceinline__ void dmma16n8k8(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(128)
    k_dgemm(int M, int N, int K, double alpha, const double* __restrict__ A, int64_t lda,
            const double* __restrict__ B, int64_t ldb, double beta, double* __restrict__ C,
            int64_t ldc) {
    __shared__ double As[2][GBK * GS];
    __shared__ double Bs[2][GBK * GS];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, tq = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
    const int m0 = blockIdx.x * GBM, n0 = blockIdx.y * GBN;
    double acc[2][4][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;

    // 64x16 tile = 1024 values, 8 per thread
    double ra[8], rb[8];
    auto load = [&](int k0) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = tid + u * 128;
            int mi, kk;
            if (!TA) { mi = e & 63; kk = e >> 6; } else { kk = e & 15; mi = e >> 4; }
            const int gm = m0 + mi, gk = k0 + kk;
            double v = 0.0;
            if (gm < M && gk < K) v = TA ? A[gk + (int64_t)gm * lda] : A[gm + (int64_t)gk * lda];
            ra[u] = v;
            int ni, kb;
            if (!TB) { kb = e & 15; ni = e >> 4; } else { ni = e & 63; kb = e >> 6; }
            const int gn = n0 + ni, gk2 = k0 + kb;
            double w = 0.0;
            if (gn < N && gk2 < K) w = TB ? B[gn + (int64_t)gk2 * ldb] : B[gk2 + (int64_t)gn * ldb];
            rb[u] = w;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = tid + u * 128;
            int mi, kk;
            if (!TA) { mi = e & 63; kk = e >> 6; } else { kk = e & 15; mi = e >> 4; }
            As[buf][kk * GS + mi] = ra[u];
            int ni, kb;
            if (!TB) { kb = e & 15; ni = e >> 4; } else { ni = e & 63; kb = e >> 6; }
            Bs[buf][kb * GS + ni] = rb[u];
        }
    };
    const int nk = (K + GBK - 1) / GBK;
    if (nk > 0) {
        load(0);
        store(0);
    }
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < nk) load((kt + 1) * GBK);
#pragma unroll
        for (int ks = 0; ks < GBK; ks += 8) {
            double af[2][4], bf[4][2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int mb = wm + i * 16;
                af[i][0] = As[buf][(ks + tq) * GS + mb + g];
                af[i][1] = As[buf][(ks + tq) * GS + mb + g + 8];
                af[i][2] = As[buf][(ks + tq + 4) * GS + mb + g];
                af[i][3] = As[buf][(ks + tq + 4) * GS + mb + g + 8];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int nb = wn + j * 8;
                bf[j][0] = Bs[buf][(ks + tq) * GS + nb + g];
                bf[j][1] = Bs[buf][(ks + tq + 4) * GS + nb + g];
            }
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma16n8k8(acc[i][j], af[i], bf[j]);
        }
        if (kt + 1 < nk) store(buf ^ 1);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int gm = m0 + wm + i * 16 + g + ((v >> 1) << 3);
                const int gn = n0 + wn + j * 8 + 2 * tq + (v & 1);
                if (gm < M && gn < N) {
                    double* cp = C + gm + (int64_t)gn * ldc;
                    double r = alpha * acc[i][j][v];
                    if (beta != 0.0) r = fma(beta, *cp, r);
                    *cp = r;
                }
            }
}

// ---------------------------------------------------------------------------
// per-column panel kernels.  The working column a = A[kb:, col] (nk rows).
// V is nk x b (ld ldv), T is b x b (ld ldt), Y is nk x b (ld ldy).
// ---------------------------------------------------------------------------
constexpr int CT = 256;  // threads per CTA of the row-parallel kernels

struct Col {
    double* a;   // column (nk rows)
    int nk;      // rows
    int j;       // reflector index within the panel
    int jr;      // right-update width (reflectors 0..jr-1 of Y)
    int vrow;    // row of V multiplying the right update (col - kb)
    const double* V;
    int64_t ldv;
    const double* T;
    int64_t ldt;
    const double* Y;
    int64_t ldy;
    double* part;  // per-CTA partials, stride b
    int b;
    double* scal;  // [0] tau [1] beta [2] scale [3] alpha [4..] w / dots
};

// warp w of the CTA accumulates dot(V[rows, t], x[rows]) for t = w, w+8, ...
__device__ __forceinline__ void cta_vdots(const Col& c, const double* xs, int i0, int cnt, int nt,
                                          double* out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int t = warp; t < nt; t += CT / 32) {
        const double* vc = c.V + (int64_t)t * c.ldv + i0;
        double s = 0.0;
        for (int r = lane; r < cnt; r += 32) s = fma(vc[r], xs[r], s);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) out[t] = s;
    }
}

// (1) right update from earlier mini-blocks, then partial V^T a
__global__ void __launch_bounds__(CT) k_col_right_dots(Col c) {
    __shared__ double xs[CT];
    const int i0 = blockIdx.x * CT, i = i0 + threadIdx.x;
    const int cnt = min(CT, c.nk - i0);
    if (i < c.nk) {
        double v = c.a[i];
        for (int t = 0; t < c.jr; ++t) v = fma(-c.Y[i + (int64_t)t * c.ldy], c.V[c.vrow + (int64_t)t * c.ldv], v);
        c.a[i] = v;
        xs[threadIdx.x] = v;
    }
    __syncthreads();
    cta_vdots(c, xs, i0, cnt, c.j, c.part + (int64_t)blockIdx.x * c.b);
}

// (2) w = T^T (sum of partials)   (left update coefficients)
__global__ void k_col_w(Col c, int nparts) {
    extern __shared__ double w0[];  // j entries
    for (int t = threadIdx.x; t < c.j; t += blockDim.x) {
        double s = 0.0;
        for (int p = 0; p < nparts; ++p) s += c.part[(int64_t)p * c.b + t];
        w0[t] = s;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < c.j; t += blockDim.x) {
        double s = 0.0;
        for (int k = 0; k <= t; ++k) s = fma(c.T[k + (int64_t)t * c.ldt], w0[k], s);  // (T^T w0)_t
        c.scal[8 + t] = s;
    }
}

// (3) a -= V w; partial sum of squares of a[j+1:], alpha = a[j]
__global__ void __launch_bounds__(CT) k_col_left(Col c) {
    __shared__ double red[CT / 32];
    const int i = blockIdx.x * CT + threadIdx.x;
    double sq = 0.0;
    if (i < c.nk) {
        double v = c.a[i];
        for (int t = 0; t < c.j; ++t) v = fma(-c.V[i + (int64_t)t * c.ldv], c.scal[8 + t], v);
        c.a[i] = v;
        if (i > c.j) sq = v * v;
    }
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < CT / 32; ++w) s += red[w];
        c.part[(int64_t)blockIdx.x * c.b] = s;
    }
}

// (4) householder_vector scalars (kernels.py:74-99, real case)
__global__ void k_col_house(Col c, int nparts) {
    if (threadIdx.x != 0) return;
    double sigma = 0.0;
    for (int p = 0; p < nparts; ++p) sigma += c.part[(int64_t)p * c.b];
    const double alpha = c.a[c.j];
    double tau, beta, scale;
    if (sigma == 0.0) {
        tau = 0.0;
        beta = alpha;
        scale = 0.0;
    } else {
        const double anorm = sqrt(alpha * alpha + sigma);
        beta = alpha >= 0.0 ? -anorm : anorm;
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
    }
    c.scal[0] = tau;
    c.scal[1] = beta;
    c.scal[2] = scale;
    c.scal[3] = alpha;
}

// (5) write v_j into V, finalize the column, partial V^T v
__global__ void __launch_bounds__(CT) k_col_vec(Col c, double* Vw) {
    __shared__ double xs[CT];
    const int i0 = blockIdx.x * CT, i = i0 + threadIdx.x;
    const int cnt = min(CT, c.nk - i0);
    if (i < c.nk) {
        double v;
        const double tau = c.scal[0];
        if (i < c.j) v = 0.0;
        else if (i == c.j) v = 1.0;
        else v = tau == 0.0 ? 0.0 : c.a[i] * c.scal[2];
        Vw[i + (int64_t)c.j * c.ldv] = v;
        xs[threadIdx.x] = v;
        if (i == c.j) c.a[i] = c.scal[1];
        else if (i > c.j) c.a[i] = 0.0;
    }
    __syncthreads();
    cta_vdots(c, xs, i0, cnt, c.j, c.part + (int64_t)blockIdx.x * c.b);
}

// (6) T[:j, j] = -tau T[:j,:j] (V[:, :j]^T v_j), T[j, j] = tau  (kernels.py:156-160)
__global__ void k_col_tcol(Col c, double* Tw, int nparts) {
    extern __shared__ double d[];  // j entries
    const double tau = c.scal[0];
    for (int t = threadIdx.x; t < c.j; t += blockDim.x) {
        double s = 0.0;
        for (int p = 0; p < nparts; ++p) s += c.part[(int64_t)p * c.b + t];
        d[t] = s;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < c.j; r += blockDim.x) {
        double s = 0.0;
        for (int k = r; k < c.j; ++k) s = fma(c.T[r + (int64_t)k * c.ldt], d[k], s);
        Tw[r + (int64_t)c.j * c.ldt] = -tau * s;
    }
    if (threadIdx.x == 0) Tw[c.j + (int64_t)c.j * c.ldt] = tau;
}

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
};

int gemm(Ctx& x, bool ta, bool tb, int M, int N, int K, double alpha, const double* A, int64_t lda,
         const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
    if (M <= 0 || N <= 0) return SS_OK;
    dim3 grid((M + GBM - 1) / GBM, (N + GBN - 1) / GBN);
    if (!ta && !tb) k_dgemm<false, false><<<grid, 128, 0, x.st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    else if (!ta && tb) k_dgemm<false, true><<<grid, 128, 0, x.st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    else if (ta && !tb) k_dgemm<true, false><<<grid, 128, 0, x.st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    else k_dgemm<true, true><<<grid, 128, 0, x.st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    SS_LAUNCH_CHECK(x.h);
    return SS_OK;
}

#define SS_TRY(expr)            \
    do {                        \
        int _rc = (expr);       \
        if (_rc) return _rc;    \
    } while (0)

// Factor one column of a panel: right update (jr reflectors of Y), left
// update with the panel's j earlier reflectors, Householder, T column.
int panel_column(Ctx& x, Col c, double* V, double* T) {
    const int nparts = (c.nk + CT - 1) / CT;
    k_col_right_dots<<<nparts, CT, 0, x.st>>>(c);
    SS_LAUNCH_CHECK(x.h);
    if (c.j > 0) {
        k_col_w<<<1, 256, (size_t)c.j * sizeof(double), x.st>>>(c, nparts);
        SS_LAUNCH_CHECK(x.h);
    }
    k_col_left<<<nparts, CT, 0, x.st>>>(c);
    SS_LAUNCH_CHECK(x.h);
    k_col_house<<<1, 32, 0, x.st>>>(c, nparts);
    SS_LAUNCH_CHECK(x.h);
    k_col_vec<<<nparts, CT, 0, x.st>>>(c, V);
    SS_LAUNCH_CHECK(x.h);
    k_col_tcol<<<1, 256, (size_t)std::max(c.j, 1) * sizeof(double), x.st>>>(c, T, nparts);
    SS_LAUNCH_CHECK(x.h);
    return SS_OK;
}

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

}  // namespace

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
    const int nparts_max = (n + CT - 1) / CT;
    size_t need = 0;
    need += (size_t)ldv * bw_max;        // V
    need += (size_t)ldv * bw_max;        // Y (bottom)
    need += (size_t)bw_max * bw_max;     // T
    need += (size_t)ldw * bw_max * 2;    // W1, W2 for right updates (mrows x k)
    need += (size_t)bw_max * n * 2;      // W1, W2 for left updates (k x mcols)
    need += (size_t)nparts_max * bw_max; // partials
    need += 16 + 2 * (size_t)bw_max;     // scalars + w
    SS_TRY(ss::ensure_ws(h, need * sizeof(double), 1));
    double* V = (double*)h->ws2;
    double* Y = V + (size_t)ldv * bw_max;
    double* T = Y + (size_t)ldv * bw_max;
    const int64_t ldt = bw_max;
    double* W1 = T + (size_t)bw_max * bw_max;
    double* W2 = W1 + (size_t)ldw * bw_max;
    double* L1 = W2 + (size_t)ldw * bw_max;
    double* L2 = L1 + (size_t)bw_max * n;
    double* part = L2 + (size_t)bw_max * n;
    double* scal = part + (size_t)nparts_max * bw_max;
    const int64_t ldl = bw_max;

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
    for (int j = 0; j < kB; ++j) {
        Col c;
        c.a = B + (int64_t)j * ldb;
        c.nk = n;
        c.j = j;
        c.jr = 0;
        c.vrow = 0;
        c.V = V;
        c.ldv = ldv;
        c.T = T;
        c.ldt = ldt;
        c.Y = Y;
        c.ldy = ldv;
        c.part = part;
        c.b = bw_max;
        c.scal = scal;
        SS_TRY(panel_column(x, c, V, T));
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
        int js = 0;  // first reflector of the current mini-block
        for (int j = 0; j < bw; ++j) {
            const int col = zc + j;
            Col c;
            c.a = A + kb + (int64_t)col * lda;
            c.nk = nk;
            c.j = j;
            // right update from complete mini-blocks: reflectors i <= j - m
            c.jr = std::min(js, std::max(j - m + 1, 0));
            c.vrow = col - kb;  // = j - m (only used when jr > 0)
            c.V = V;
            c.ldv = ldv;
            c.T = T;
            c.ldt = ldt;
            c.Y = Y;
            c.ldy = ldv;
            c.part = part;
            c.b = bw_max;
            c.scal = scal;
            SS_TRY(panel_column(x, c, V, T));
            const int jb = j + 1;
            if (jb % m == 0 || jb == bw) {
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
