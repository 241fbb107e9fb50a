// Window update kernel (the dominant FP64 kernel of the sweep).
//
//   Zout_l[i, :] = Zin_l[i, :] P_l[nb:nb+m, :] + Pan[i, :] P_l[0:nb, :]
//                  - sigma_l P_l[i - (r0 - m), :]        (lazy-shift rows only)
//
// reference solvers.py:186-199 (update_shift + gemm_acc).  Pan is the real,
// shift-independent panel [top; Ahat][0:r0, c0:c0+nb].
//
// Tiling: a CTA owns one 64-row tile of the panel (staged once in shared
// memory, reused by all SG shifts the CTA processes) and walks its shifts in
// chunks of S.  Per chunk, P_l (nc x m) and the 64 x m tile of Zin_l for the
// S shifts are staged with cp.async (zero-filled past r0).  Warp w owns one
// (shift, C-column group) unit of the chunk: lane L computes rows
// (2L, 2L+1) x C complex columns in registers; P_l entries are warp-uniform shared
// memory broadcasts, panel / Zin entries are per-lane conflict-free loads.
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

constexpr int kUpdRows = 64;  // rows per tile: 2 per lane

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
};

__host__ __device__ inline size_t upd_smem_bytes(int nb, int m, int S) {
    const int nc = nb + m;
    return (size_t)nb * kUpdRows * 8 + (size_t)S * nc * m * 16 + (size_t)S * m * kUpdRows * 16;
}

template <int C, bool EXACT>
__global__ void __launch_bounds__(256)
    k_update(UpdDims u, const double2* __restrict__ Zin, double2* __restrict__ Zout,
             const double2* __restrict__ Pbuf) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int nb = u.nb, m = u.m, nc = u.nc, r0 = u.r0;
    double* Pan = (double*)smem;                                        // [nb][64]
    double2* Pst = (double2*)(smem + (size_t)nb * kUpdRows * 8);        // [S][nc*m]
    double2* Zst = Pst + (size_t)u.S * nc * m;                          // [S][m][64]
    const int i0 = u.rlo + blockIdx.x * kUpdRows;
    const int l0 = blockIdx.y * u.SG;
    const int lend = min(l0 + u.SG, u.sb);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ncg = (m + C - 1) / C;

    // ---- panel tile (once per CTA) ----
    for (int v = tid; v < nb * kUpdRows; v += blockDim.x) {
        const int j = v >> 6, ii = v & 63;
        const int i = i0 + ii, col = u.c0 + j;
        if (i >= r0) {
            Pan[v] = 0.0;
        } else if (i >= u.ptop) {
            cp_async8(Pan + v, u.A + (i - u.ptop) + (int64_t)col * u.lda, true);
        } else if (u.ident_top) {
            Pan[v] = (i == col) ? 1.0 : 0.0;
        } else {
            cp_async8(Pan + v, u.T + i + (int64_t)col * u.ldt, true);
        }
    }

    const int s_w = warp / ncg, g = warp - s_w * ncg;  // this warp's unit
    const int cb = g * C;
    const int row_a = i0 + 2 * lane, row_b = row_a + 1;  // adjacent rows: 16-byte panel loads
    const int dlo = r0 - m;

    for (int lc = l0; lc < lend; lc += u.S) {
        const int nsc = min(u.S, lend - lc);
        __syncthreads();  // previous chunk's readers are done with the stage
        {
            const double2* src = Pbuf + (int64_t)lc * nc * m;
            const int tot = nsc * nc * m;
            for (int v = tid; v < tot; v += blockDim.x) cp_async16(Pst + v, src + v, true);
            const int ztot = nsc * m * kUpdRows;
            for (int v = tid; v < ztot; v += blockDim.x) {
                const int ii = v & 63, sc = v >> 6;  // sc = s*m + c
                const int s = sc / m, c = sc - s * m;
                const int i = i0 + ii;
                const bool ok = i < r0;
                const double2* zp = Zin + ((int64_t)(lc + s) * m + c) * u.LDZ + (ok ? i : 0);
                cp_async16(Zst + v, zp, ok);
            }
        }
        cp_async_commit_wait_all();
        __syncthreads();
        if (s_w >= nsc) continue;
        const int l = lc + s_w;
        const double2* Pl = Pst + (size_t)s_w * nc * m;
        const double2* Zl = Zst + (size_t)s_w * m * kUpdRows;
        const int ncol = EXACT ? C : min(C, m - cb);
        double2 acc0[C], acc1[C];
#pragma unroll
        for (int c = 0; c < C; ++c) acc0[c] = acc1[c] = cz();
        // Z1 (real panel) part -- the reference's outer GEMM
#pragma unroll 4
        for (int j = 0; j < nb; ++j) {
            const double2 a01 = *reinterpret_cast<const double2*>(Pan + j * kUpdRows + 2 * lane);
            const double a0 = a01.x, a1 = a01.y;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (EXACT || c < ncol) {
                    const double2 p = Pl[j * m + cb + c];
                    acc0[c] = rfma(a0, p, acc0[c]);
                    acc1[c] = rfma(a1, p, acc1[c]);
                }
            }
        }
        // Z2 part -- the reference's per-shift batched GEMM
#pragma unroll 2
        for (int j = 0; j < m; ++j) {
            const double2 z0 = Zl[j * kUpdRows + 2 * lane], z1 = Zl[j * kUpdRows + 2 * lane + 1];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (EXACT || c < ncol) {
                    const double2 p = Pl[(nb + j) * m + cb + c];
                    acc0[c] = cfma(z0, p, acc0[c]);
                    acc1[c] = cfma(z1, p, acc1[c]);
                }
            }
        }
        const double2 sig = u.shifts[l];
        double2* zo = Zout + ((int64_t)l * m + cb) * u.LDZ;
        const int da = row_a - dlo, db = row_b - dlo;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (EXACT || c < ncol) {
                if (row_a < r0) {
                    double2 v = acc0[c];
                    if (da >= 0 && da < u.mnb) v = csub(v, cmul(sig, Pl[da * m + cb + c]));
                    zo[(int64_t)c * u.LDZ + row_a] = v;
                }
                if (row_b < r0) {
                    double2 v = acc1[c];
                    if (db >= 0 && db < u.mnb) v = csub(v, cmul(sig, Pl[db * m + cb + c]));
                    zo[(int64_t)c * u.LDZ + row_b] = v;
                }
            }
        }
    }
}

}  // namespace ssd
