// Window update kernel (the dominant FP64 kernel of the sweep).
//
//   Zout_l[i, :] = Zin_l[i, :] P_l[nb:nb+m, :] + Pan[i, :] P_l[0:nb, :]
//                  - sigma_l P_l[i - (r0 - m), :]        (lazy-shift rows only)
//
// reference solvers.py:186-199 (update_shift + gemm_acc).  Pan is the real,
// shift-independent panel [top; Ahat][0:r0, c0:c0+nb]; P_l is j-major.
//
// Tiling (sized from measured B200 shared-memory costs: a per-lane LDS.128
// is 4 LSU cycles, a broadcast LDS.128 2 cycles, 64 DFMA/clk/SM):
//  * a CTA owns one 64-row tile of the panel, staged once (cp.async) and
//    reused by every shift of its group (SG shifts, chunks of S);
//  * per chunk, P_l and the 64 x m tile of Zin_l of the S shifts are staged
//    with cp.async (zero-filled past r0);
//  * a warp owns one (shift, column block of G*C columns) unit; lane =
//    (row group rg, column group q): R = 2G consecutive rows x C columns in
//    registers.  For m = 10: G = 2, C = 5, R = 4 -> per panel column j a
//    warp issues 2 panel LDS.128 (pair-interleaved layout, 2 wavefronts
//    each), 5 P LDS.128 (two broadcast addresses) and 40 DFMA: 14 LSU
//    cycles per 20 FP64-pipe cycles.
#pragma once

#include "ss_device.cuh"

namespace ssd {

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit_wait_all() {
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::);
}

constexpr int kUpdRows = 64;  // rows per tile

struct UpdDims {
    int n, m, ptop, ident_top;
    const double* A;
    int64_t lda;
    const double* T;
    int64_t ldt;
    const double2* shifts;
    int sb;
    int64_t LDZ;
    // step
    int nb, mnb, r0, c0, nc;
    // tiling
    int rlo;  // first row of tile 0
    int S;    // shifts per chunk
    int SG;   // shifts per CTA
    int nws;     // column blocks per shift
    int ksplit;  // warps per (shift, column block): 1, or 2 = panel K range split
    int jh;      // ksplit == 2: warp half 0 takes panel columns [0, jh) + the Z2 part
    int jq[3];   // k_far4: role boundaries of the four-way K split
    // P source (warp-specialised kernel): per shift, P12 = pstride*l + p12off
    // (nb x m, j-major), P22 = pstride*l + p22off (m x m) unless zid (P22 = I:
    // the far-row passes of the two-level sweep after the first)
    int64_t pstride, p12off, p22off;
    int zid;
    int flags;  // experiment knobs (bit 0: producer spins instead of parking)
    // transposed sweep (k_update<..., TR = true>, ss_lq.cu): the panel is
    // [A^T; -I] (rows i < n: A(c0 + j, i), rows n + r: -[r == c0 + j]); the
    // lazy -sigma rows are [lz0, lz0 + mnb) with P12 rows lzp + (i - lz0)
    int lz0 = 0, lzp = 0;
};

__host__ __device__ inline size_t upd_smem_bytes(int nb, int m, int S, bool pg = false) {
    const int nc = nb + m;
    return (size_t)nb * kUpdRows * 8 + (pg ? 0 : (size_t)S * nc * m * 16) + (size_t)S * m * kUpdRows * 16;
}

// panel position of tile row `row` (0..63) inside one panel column: rows of
// a lane's row group are stored as R/2 pairs; pair p of every row group is
// contiguous across row groups so one LDS.128 touches 256 contiguous bytes.
template <int G>
__device__ __forceinline__ int pan_index(int row) {
    constexpr int R = 2 * G, RG = 32 / G;
    const int rg = row / R, w = row - rg * R, p = w >> 1, e = w & 1;
    return p * (2 * RG) + rg * 2 + e;
}

// PG: P_l is read from global memory (L1 / L2; every lane of a row group
// reads the same entries) instead of being staged -- windows so wide
// (m >~ 90) that the staged P does not fit shared memory.
template <int G, int C, bool EXACT, int MAXT = 256, bool PG = false, bool TR = false>
__global__ void __launch_bounds__(MAXT)
    k_update(UpdDims u, const double2* __restrict__ Zin, double2* __restrict__ Zout,
             const double2* __restrict__ Pbuf) {
    constexpr int R = 2 * G, RG = 32 / G;
    extern __shared__ __align__(16) unsigned char smem[];
    const int nb = u.nb, m = u.m, nc = u.nc, r0 = u.r0;
    double* Pan = (double*)smem;                                        // [nb][64] (pair-interleaved)
    double2* Pst = (double2*)(smem + (size_t)nb * kUpdRows * 8);        // [S][nc*m], j-major
    double2* Zst = Pst + (PG ? 0 : (size_t)u.S * nc * m);               // [S][m][64]
    const int i0 = u.rlo + blockIdx.x * kUpdRows;
    const int l0 = blockIdx.y * u.SG;
    const int lend = min(l0 + u.SG, u.sb);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    // ---- panel tile (once per CTA) ----
    for (int v = tid; v < nb * kUpdRows; v += blockDim.x) {
        // transposed: consecutive threads along a row of A^T (= a column of
        // A, contiguous) instead of down a column
        const int j = TR ? v % nb : v >> 6, rr = TR ? v / nb : v & 63;
        const int i = i0 + rr, col = u.c0 + j;
        double* dst = Pan + j * kUpdRows + pan_index<G>(rr);
        if (TR) {
            if (i >= r0) *dst = 0.0;
            else if (i < u.n) cp_async8(dst, u.A + col + (int64_t)i * u.lda, true);
            else *dst = (i - u.n == col) ? -1.0 : 0.0;
        } else if (i >= r0) {
            *dst = 0.0;
        } else if (i >= u.ptop) {
            cp_async8(dst, u.A + (i - u.ptop) + (int64_t)col * u.lda, true);
        } else if (u.ident_top) {
            *dst = (i == col) ? 1.0 : 0.0;
        } else {
            cp_async8(dst, u.T + i + (int64_t)col * u.ldt, true);
        }
    }

    const int unit = warp / u.ksplit, half = warp - unit * u.ksplit;
    const int s_w = unit / u.nws, blk = unit - s_w * u.nws;  // this warp's (shift, column block)
    // adjacent lanes share a row group (q = lane % G): measured on B200 an
    // LDS.128 costs one cycle per half-warp per 128 distinct bytes, so the
    // pair-sharing pattern keeps both panel and P loads at 2 cycles
    const int rg = lane / G, q = lane - rg * G;
    const int cb = blk * (G * C) + q * C;                     // first output column of this lane
    const int ncol = EXACT ? C : max(0, min(C, m - cb));
    const int rbase = rg * R;                                 // first tile row of this lane
    const int dlo = TR ? u.lz0 : r0 - m;  // first lazy-shift row
    const int dp = TR ? u.lzp : 0;         // its P12 row
    const int jlo = half == 0 ? 0 : u.jh;
    const int jhi = (u.ksplit == 1 || half == 1) ? nb : u.jh;

    for (int lc = l0; lc < lend; lc += u.S) {
        const int nsc = min(u.S, lend - lc);
        __syncthreads();  // previous chunk's readers are done with the stage
        {
            const double2* src = Pbuf + (int64_t)lc * nc * m;
            const int tot = nsc * nc * m;
            if (!PG)
                for (int v = tid; v < tot; v += blockDim.x) cp_async16(Pst + v, src + v, true);
            const int ztot = nsc * m * kUpdRows;
            for (int v = tid; v < ztot; v += blockDim.x) {
                const int ii = v & 63, sc = v >> 6;  // sc = s*m + c
                const int s = sc / m, c = sc - s * m;
                const int i = i0 + ii;
                const bool ok = i < r0;
                const double2* zp = Zin + ((int64_t)(lc + s) * m + c) * u.LDZ + (ok ? i : 0);
                // row ii = rg*R + w lives at w*RG + rg: a lane's R rows are R
                // conflict-free LDS.128 at stride RG
                const int zrg = ii / R, zw = ii - zrg * R;
                cp_async16(Zst + (v - ii) + zw * RG + zrg, zp, ok);
            }
        }
        cp_async_commit_wait_all();
        __syncthreads();
        {
            // pull the next chunk's P and Z2 tiles into L2 while this chunk
            // computes, so its cp.async staging hits L2 instead of HBM
            const int lnx = lc + u.S;
            if (lnx < lend) {
                const int nnx = min(u.S, lend - lnx);
                const char* pb = reinterpret_cast<const char*>(Pbuf + (int64_t)lnx * nc * m);
                const int plines = (nnx * nc * m * 16 + 127) >> 7;
                for (int v = tid; v < plines; v += blockDim.x)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(pb + (size_t)v * 128));
                const int zcols = nnx * m;  // one 64-row tile = 1 KB = 8 lines per column
                for (int v = tid; v < zcols * 8; v += blockDim.x) {
                    const int sc = v >> 3, ln = v & 7;
                    const int s = sc / m, c = sc - s * m;
                    const double2* zp = Zin + ((int64_t)(lnx + s) * m + c) * u.LDZ + i0 + ln * 8;
                    if (i0 + ln * 8 < r0) asm volatile("prefetch.global.L2 [%0];" ::"l"(zp));
                }
            }
        }
        if (s_w >= nsc) continue;
        const int l = lc + s_w;
        const double2* Pl = PG ? Pbuf + (int64_t)l * nc * m + cb : Pst + (size_t)s_w * nc * m + cb;
        double2* Zs = Zst + (size_t)s_w * m * kUpdRows;
        const double2* Zl = Zs + rg;
        double2 acc[R][C];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < C; ++c) acc[r][c] = cz();
        // Z1 (real panel) part -- the reference's outer GEMM
        const double* pan_l = Pan + rg * 2;
#pragma unroll 2
        for (int j = jlo; j < jhi; ++j) {
            double a[R];
#pragma unroll
            for (int p = 0; p < R / 2; ++p) {
                const double2 v = *reinterpret_cast<const double2*>(pan_l + j * kUpdRows + p * (2 * RG));
                a[2 * p] = v.x;
                a[2 * p + 1] = v.y;
            }
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (EXACT || c < ncol) {
                    const double2 pv = Pl[j * m + c];
#pragma unroll
                    for (int r = 0; r < R; ++r) acc[r][c] = rfma(a[r], pv, acc[r][c]);
                }
            }
        }
        // Z2 part -- the reference's per-shift batched GEMM (warp half 0)
        if (half == 0) {
            for (int j = 0; j < m; ++j) {
                double2 z[R];
#pragma unroll
                for (int r = 0; r < R; ++r) z[r] = Zl[j * kUpdRows + r * RG];
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    if (EXACT || c < ncol) {
                        const double2 pv = Pl[(nb + j) * m + c];
#pragma unroll
                        for (int r = 0; r < R; ++r) acc[r][c] = cfma(z[r], pv, acc[r][c]);
                    }
                }
            }
        }
        if (u.ksplit == 2) {
            // half 1 hands its partial sums to half 0 through this shift's (now
            // consumed) Z2 staging tile: [c][64 rows] per column block.  With
            // several column blocks every block's half 0 reads all m columns
            // of Zs, so the whole shift group syncs (64 nws threads; one named
            // barrier per shift of the CTA)
            const int bar = u.nws == 1 ? 1 + unit : 1 + s_w;
            const int cnt = 64 * u.nws;
            asm volatile("bar.sync %0, %1;\n" ::"r"(bar), "r"(cnt));   // every half 0 done reading Zs
            // scratch [(r*C + c)][lane] per column block: conflict-free 16-byte stores / loads
            double2* red = Zs + blk * (R * C * 32) + lane;
            if (half == 1) {
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int c = 0; c < C; ++c)
                        if (EXACT || c < ncol) red[(r * C + c) * 32] = acc[r][c];
            }
            asm volatile("bar.sync %0, %1;\n" ::"r"(bar), "r"(cnt));   // partials visible
            if (half == 1) continue;
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < C; ++c)
                    if (EXACT || c < ncol) acc[r][c] = cadd(acc[r][c], red[(r * C + c) * 32]);
        }
        const double2 sig = u.shifts[l];
        double2* zo = Zout + ((int64_t)l * m + cb) * u.LDZ;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int row = i0 + rbase + r;
            if (row >= r0) continue;
            const int dd = row - dlo;
            const bool corr = dd >= 0 && dd < u.mnb;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (EXACT || c < ncol) {
                    double2 v = acc[r][c];
                    if (corr) v = csub(v, cmul(sig, Pl[(dp + dd) * m + c]));
                    zo[(int64_t)c * u.LDZ + row] = v;
                }
            }
        }
    }
}

}  // namespace ssd
