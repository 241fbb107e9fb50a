// FP64 tensor-core GEMM for the reduction's trailing updates (north_star:
// the only dense contraction, the only DMMA use):
//     C = alpha op(A) op(B) + beta C        (column-major, op = N or T)
//
// sm_100a mapping: mma.sync.m16n8k8.f64 (DMMA) with 8 warps per CTA, CTA
// tile BM x BN (BM = 16 MT WM, BN = 8 NT WN), K in steps of BK = 16 through
// a kGS-stage cp.async ring (8-byte copies: the reduction's sub-matrices
// start at arbitrary rows, so 16-byte alignment is not guaranteed).  Each
// operand tile is stored in the layout its global copy is contiguous in
// (k-contiguous rows or m/n-contiguous rows), padded so that the DMMA
// fragment loads (lanes (g, tq)) hit 32 distinct banks.
// Long-K products with a small output (V^T M, M V, the Y extension's
// A0 V) run split-K: every split writes its partial tile to scratch and
// k_gemm_splitk_reduce sums the splits in split order (deterministic).
#pragma once

namespace ssr {

constexpr int kGBK = 16;    // K per stage
constexpr int kGS = 3;      // stages
constexpr int kGThreads = 256;

__device__ __forceinline__ void dmma(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

__device__ __forceinline__ void cpa8(double* s, const double* g, bool valid) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(valid ? 8 : 0));
}
// 16-byte copy of the pair (g[0], g[1]); `bytes` 16, 8 (second element past
// the matrix edge: zero-filled) or 0
__device__ __forceinline__ void cpa16(double* s, const double* g, int bytes) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(bytes));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Operand tile of R rows (m or n) x BK: "row-contiguous" (global contiguous
// along m/n): s[k][r], stride R + 4; "k-contiguous": s[r][k], stride BK + 4.
// Both strides are 4 mod 16 doubles: fragment loads are conflict-free.
template <int R, bool KC, int BK = kGBK>
struct Tile {
    static constexpr int STRIDE = KC ? BK + 4 : R + 4;
    static constexpr int ELEMS = KC ? R * STRIDE : BK * STRIDE;
    __device__ static __forceinline__ int idx(int r, int k) { return KC ? r * STRIDE + k : k * STRIDE + r; }
};

template <bool TA, bool TB, int MT, int NT, int WM, int WN, int BK_ = kGBK>
struct GemmCfg {
    static constexpr int BM = 16 * MT * WM, BN = 8 * NT * WN, BK = BK_;
    // A (m, k): !TA -> A[m + k lda] m-contiguous; TA -> A[k + m lda] k-contiguous
    using TA_ = Tile<BM, TA, BK>;
    // B (k, n): !TB -> B[k + n ldb] k-contiguous; TB -> B[n + k ldb] n-contiguous
    using TB_ = Tile<BN, !TB, BK>;
    static constexpr int STAGE = TA_::ELEMS + TB_::ELEMS;
    static constexpr size_t SMEM = (size_t)kGS * STAGE * 8;
};

struct GemmArgs {
    int M, N, K;
    double alpha, beta;
    const double* A;
    int64_t lda;
    const double* B;
    int64_t ldb;
    double* C;
    int64_t ldc;
    int ksplit;       // > 1: partial tiles to `part` (K range split evenly in BK steps)
    double* part;     // [ksplit][M x N] (ld M)
};

// two CTAs per SM for warp tiles of <= 8 DMMA tiles (acc 32 doubles): one
// CTA's epilogue / pipeline fill overlaps the other's DMMAs
// V16: both operands' contiguous dimensions are 16-byte aligned (base
// pointers and leading dimensions even): pairs of elements per cp.async
// (half the copy instructions; the 8-byte path serves odd row offsets).
template <bool TA, bool TB, int MT, int NT, int WM, int WN, bool V16 = false, int BK = kGBK>
__global__ void __launch_bounds__(kGThreads, MT * NT <= 8 ? 2 : 1) k_dmma(GemmArgs g) {
    using Cfg = GemmCfg<TA, TB, MT, NT, WM, WN, BK>;
    constexpr int BM = Cfg::BM, BN = Cfg::BN;
    using TAt = typename Cfg::TA_;
    using TBt = typename Cfg::TB_;
    extern __shared__ __align__(16) double gsm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int gq = lane >> 2, tq = lane & 3;
    const int wm = (warp % WM) * 16 * MT, wn = (warp / WM) * 8 * NT;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    const int nkt_all = (g.K + BK - 1) / BK;
    const int split = blockIdx.z;
    const int kt0 = (int)((int64_t)nkt_all * split / g.ksplit), kt1 = (int)((int64_t)nkt_all * (split + 1) / g.ksplit);
    const int nkt = kt1 - kt0;

    auto load = [&](int kt, int buf) {
        double* As = gsm + (size_t)buf * Cfg::STAGE;
        double* Bs = As + TAt::ELEMS;
        const int k0 = kt * BK;
        if (V16) {
            // pairs along each operand's contiguous dimension
            for (int e = tid; e < BM * BK / 2; e += kGThreads) {
                int r, k;
                if (!TA) { r = 2 * (e % (BM / 2)); k = e / (BM / 2); } else { k = 2 * (e % (BK / 2)); r = e / (BK / 2); }
                const int gm = m0 + r, gk = k0 + k;
                const int lim = !TA ? g.M - gm : g.K - gk;   // elements left along the pair
                const bool ok = (!TA ? gk < g.K : gm < g.M) && lim > 0;
                const double* src = g.A + (ok ? (TA ? gk + (int64_t)gm * g.lda : gm + (int64_t)gk * g.lda) : 0);
                cpa16(As + TAt::idx(r, k), src, ok ? (lim >= 2 ? 16 : 8) : 0);
            }
            for (int e = tid; e < BN * BK / 2; e += kGThreads) {
                int r, k;
                if (TB) { r = 2 * (e % (BN / 2)); k = e / (BN / 2); } else { k = 2 * (e % (BK / 2)); r = e / (BK / 2); }
                const int gn = n0 + r, gk = k0 + k;
                const int lim = TB ? g.N - gn : g.K - gk;
                const bool ok = (TB ? gk < g.K : gn < g.N) && lim > 0;
                const double* src = g.B + (ok ? (TB ? gn + (int64_t)gk * g.ldb : gk + (int64_t)gn * g.ldb) : 0);
                cpa16(Bs + TBt::idx(r, k), src, ok ? (lim >= 2 ? 16 : 8) : 0);
            }
            return;
        }
        // A tile: BM x BK
        for (int e = tid; e < BM * BK; e += kGThreads) {
            int r, k;
            if (!TA) { r = e % BM; k = e / BM; } else { k = e % BK; r = e / BK; }
            const int gm = m0 + r, gk = k0 + k;
            const bool ok = gm < g.M && gk < g.K;
            const double* src = g.A + (ok ? (TA ? gk + (int64_t)gm * g.lda : gm + (int64_t)gk * g.lda) : 0);
            cpa8(As + TAt::idx(r, k), src, ok);
        }
        for (int e = tid; e < BN * BK; e += kGThreads) {
            int r, k;
            if (TB) { r = e % BN; k = e / BN; } else { k = e % BK; r = e / BK; }
            const int gn = n0 + r, gk = k0 + k;
            const bool ok = gn < g.N && gk < g.K;
            const double* src = g.B + (ok ? (TB ? gn + (int64_t)gk * g.ldb : gk + (int64_t)gn * g.ldb) : 0);
            cpa8(Bs + TBt::idx(r, k), src, ok);
        }
    };

    double acc[MT][NT][4];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;

#pragma unroll
    for (int s = 0; s < kGS - 1; ++s) {
        if (s < nkt) load(kt0 + s, s);
        cpa_commit();
    }
    for (int it = 0; it < nkt; ++it) {
        cpa_wait<kGS - 2>();
        __syncthreads();
        // prefetch stage it + kGS - 1 (its buffer was consumed at it - 1)
        if (it + kGS - 1 < nkt) load(kt0 + it + kGS - 1, (it + kGS - 1) % kGS);
        cpa_commit();
        const double* As = gsm + (size_t)(it % kGS) * Cfg::STAGE;
        const double* Bs = As + TAt::ELEMS;
#pragma unroll
        for (int ks = 0; ks < BK; ks += 8) {
            double af[MT][4], bf[NT][2];
#pragma unroll
            for (int i = 0; i < MT; ++i) {
                const int mb = wm + i * 16;
                af[i][0] = As[TAt::idx(mb + gq, ks + tq)];
                af[i][1] = As[TAt::idx(mb + gq + 8, ks + tq)];
                af[i][2] = As[TAt::idx(mb + gq, ks + tq + 4)];
                af[i][3] = As[TAt::idx(mb + gq + 8, ks + tq + 4)];
            }
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const int nb = wn + j * 8;
                bf[j][0] = Bs[TBt::idx(nb + gq, ks + tq)];
                bf[j][1] = Bs[TBt::idx(nb + gq, ks + tq + 4)];
            }
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma(acc[i][j], af[i], bf[j]);
        }
    }
    cpa_wait<0>();
    // epilogue: C(m, n) for rows gq, gq + 8 and columns 2 tq, 2 tq + 1 of each
    // tile.  All C loads are issued before any store (C is not restrict: a
    // load-fma-store per element would serialise 4 MT NT global round trips)
    if (g.ksplit > 1) {
        double* out = g.part + (size_t)split * g.M * g.N;
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const int gm = m0 + wm + i * 16 + gq + ((v >> 1) << 3);
                    const int gn = n0 + wn + j * 8 + 2 * tq + (v & 1);
                    if (gm < g.M && gn < g.N) out[gm + (int64_t)gn * g.M] = acc[i][j][v];
                }
        return;
    }
    if (g.beta != 0.0) {
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const int gm = m0 + wm + i * 16 + gq + ((v >> 1) << 3);
                    const int gn = n0 + wn + j * 8 + 2 * tq + (v & 1);
                    const double c = (gm < g.M && gn < g.N) ? __ldg(g.C + gm + (int64_t)gn * g.ldc) : 0.0;
                    acc[i][j][v] = fma(g.beta, c, g.alpha * acc[i][j][v]);
                }
    } else {
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[i][j][v] *= g.alpha;
    }
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int gm = m0 + wm + i * 16 + gq + ((v >> 1) << 3);
                const int gn = n0 + wn + j * 8 + 2 * tq + (v & 1);
                if (gm < g.M && gn < g.N) g.C[gm + (int64_t)gn * g.ldc] = acc[i][j][v];
            }
}

// C = alpha sum_s part[s] + beta C  (splits summed in order)
__global__ void __launch_bounds__(256) k_gemm_splitk_reduce(GemmArgs g) {
    const int64_t tot = (int64_t)g.M * g.N;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int q = 0; q < g.ksplit; ++q) s += g.part[(size_t)q * tot + e];
        const int64_t n = e / g.M, mm = e - n * g.M;
        double* cp = g.C + mm + n * g.ldc;
        double r = g.alpha * s;
        if (g.beta != 0.0) r = fma(g.beta, *cp, r);
        *cp = r;
    }
}

}  // namespace ssr
