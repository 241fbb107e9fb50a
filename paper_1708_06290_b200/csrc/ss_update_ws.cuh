// Warp-specialised window update (TMA bulk copies + mbarrier ring).
//
// Same math as k_update (ss_update.cuh):
//   Zout_l[i, :] = Zin_l[i, :] P_l[nb:nb+m, :] + Pan[i, :] P_l[0:nb, :]
//                  - sigma_l P_l[i - (r0 - m), :]
// (reference solvers.py:186-199), restructured so the FP64 warps never wait
// on staging:
//  * warp 0 (producer, one elected lane) streams, per shift, P_l (one
//    contiguous bulk copy) and the m columns of the 64-row Zin_l tile (m bulk
//    copies) into a ring of NST stages with cp.async.bulk ...
//    mbarrier::complete_tx; it refills a stage as soon as both consumers of
//    that stage have released it (empty mbarrier, count 2);
//  * warps 1..8 are 4 consumer pairs; pair p takes the CTA's shifts p, p+4,
//    ...; within a pair warp half 0 computes panel columns [0, jh) plus the
//    Z2 x P22 part, half 1 panel columns [jh, nb), and half 1 hands its
//    partial sums to half 0 through the (consumed) Zin tile of the stage;
//  * the 64 x nb real panel tile is staged once per CTA (cp.async,
//    pair-interleaved so one panel LDS.128 is 2 wavefronts).
// Register tile per lane: 4 rows x 5 complex columns (m = 10: G = 2, C = 5).
#pragma once

#include "ss_update.cuh"

namespace ssd {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// Producer-side wait: the suspend-time hint parks the polling thread in the
// barrier unit instead of spinning (a spinning producer took ~10% of the
// kernel's issue slots from the consumers sharing its SMSP).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAITS_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
    unsigned r;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(r)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return r != 0;
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes,
                                             uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Row map of the warp-specialised kernel: lane row group rg owns tile rows
// rg + RG*w (w = 0..R-1), so for fixed w the lanes of a half-warp touch
// consecutive rows (conflict-free Z-tile LDS.128, coalesced stores).  The
// panel keeps rows (rg + RG*2p, rg + RG*(2p+1)) adjacent for 16-byte loads.
template <int G>
__device__ __forceinline__ int pan_index_ws(int row) {
    constexpr int RG = 32 / G;
    const int rg = row % RG, w = row / RG, p = w >> 1, e = w & 1;
    return p * (2 * RG) + rg * 2 + e;
}

#ifndef SS_WS_STAGES
#define SS_WS_STAGES 8
#endif
constexpr int kWsStages = SS_WS_STAGES;
constexpr int kWsPairs = 4;
constexpr int kWsThreads = 32 * (1 + 2 * kWsPairs);

__host__ __device__ inline size_t ws_smem_bytes(int nb, int m) {
    const int nc = nb + m;
    const size_t stage = ((size_t)nc * m + (size_t)m * kUpdRows) * 16;
    return 128 + (size_t)nb * kUpdRows * 8 + kWsStages * stage;
}

// ZID: the Z2 part is the identity (Zout = Zin + Pan P12): the second and
// later far-row passes of the two-level sweep.  Zin may alias Zout (in-place:
// every (row tile, shift) is read and written by one CTA only).
template <int G, int C, bool ZID>
__global__ void __launch_bounds__(kWsThreads, 1)
    k_update_ws(UpdDims u, const double2* Zin, double2* Zout, const double2* __restrict__ Pbuf) {
    constexpr int R = 2 * G, RG = 32 / G, M = G * C;  // one warp pair covers all m = M columns
    extern __shared__ __align__(16) unsigned char smem[];
    const int nb = u.nb, nc = u.nc, r0 = u.r0;
    constexpr int m = M;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);       // [kWsStages]
    uint64_t* empty = full + kWsStages;                         // [kWsStages]
    double* Pan = reinterpret_cast<double*>(smem + 128);        // [nb][64] pair-interleaved
    double2* Stg = reinterpret_cast<double2*>(smem + 128 + (size_t)nb * kUpdRows * 8);
    const size_t stage_el = (size_t)nc * m + (size_t)m * kUpdRows;  // P then Z tile [c][64]
    const int i0 = u.rlo + blockIdx.x * kUpdRows;
    const int l0 = blockIdx.y * u.SG;
    const int nsh = min(u.SG, u.sb - l0);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int rows_valid = min(kUpdRows, r0 - i0);

    if (tid == 0) {
        for (int s = 0; s < kWsStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 2);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // panel tile: all threads, generic-proxy cp.async (permuted layout)
    for (int v = tid; v < nb * kUpdRows; v += blockDim.x) {
        const int j = v >> 6, rr = v & 63;
        const int i = i0 + rr, col = u.c0 + j;
        double* dst = Pan + j * kUpdRows + pan_index_ws<G>(rr);
        if (i >= r0) {
            *dst = 0.0;
        } else if (i >= u.ptop) {
            cp_async8(dst, u.A + (i - u.ptop) + (int64_t)col * u.lda, true);
        } else if (u.ident_top) {
            *dst = (i == col) ? 1.0 : 0.0;
        } else {
            cp_async8(dst, u.T + i + (int64_t)col * u.ldt, true);
        }
    }
    cp_async_commit_wait_all();
    __syncthreads();

    if (warp == 0) {
        // ---------------- producer ----------------
        if (lane == 0) {
            const unsigned p12bytes = (unsigned)(nb * m * 16);
            const unsigned p22bytes = ZID ? 0u : (unsigned)(m * m * 16);
            const unsigned zbytes = (unsigned)(rows_valid * 16);
            for (int k = 0; k < nsh; ++k) {
                const int s = k % kWsStages, use = k / kWsStages;
                if (use > 0) mbar_wait_sleep(empty + s, (use - 1) & 1);
                double2* st = Stg + (size_t)s * stage_el;
                const int l = l0 + k;
                const double2* pl = Pbuf + (int64_t)l * u.pstride;
                mbar_expect_tx(full + s, p12bytes + p22bytes + (unsigned)m * zbytes);
                tma_bulk_g2s(st, pl + u.p12off, p12bytes, full + s);
                if (!ZID) tma_bulk_g2s(st + (size_t)nb * m, pl + u.p22off, p22bytes, full + s);
                double2* zt = st + (size_t)nc * m;
                for (int c = 0; c < m; ++c)
                    tma_bulk_g2s(zt + c * kUpdRows, Zin + ((int64_t)l * m + c) * u.LDZ + i0, zbytes,
                                 full + s);
            }
        }
        return;
    }

    // ---------------- consumers ----------------
    const int cw = warp - 1, pair = cw >> 1, half = cw & 1;
    const int rg = lane / G, q = lane - rg * G;
    const int cb = q * C;
    const int dlo = r0 - m;
    // interior tiles need neither the r0 row guard nor the lazy-shift rows
    const bool interior = i0 + kUpdRows <= (u.mnb > 0 ? dlo : r0);
    const int jlo = half == 0 ? 0 : u.jh;
    const int jhi = half == 1 ? nb : u.jh;
    const double* pan_l = Pan + rg * 2;
    for (int k = pair; k < nsh; k += kWsPairs) {
        const int s = k % kWsStages, use = k / kWsStages;
        mbar_wait(full + s, use & 1);
        const double2* st = Stg + (size_t)s * stage_el;
        const double2* Pl = st + cb;
        double2* Zs = const_cast<double2*>(st) + (size_t)nc * m;
        double2 acc[R][C];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < C; ++c) acc[r][c] = cz();
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
                const double2 pv = Pl[j * m + c];
#pragma unroll
                for (int r = 0; r < R; ++r) acc[r][c] = rfma(a[r], pv, acc[r][c]);
            }
        }
        if (half == 0) {
            if (ZID) {
#pragma unroll
                for (int c = 0; c < C; ++c)
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        acc[r][c] = cadd(acc[r][c], Zs[(cb + c) * kUpdRows + rg + RG * r]);
            } else {
                for (int j = 0; j < m; ++j) {
                    double2 z[R];
#pragma unroll
                    for (int r = 0; r < R; ++r) z[r] = Zs[j * kUpdRows + rg + RG * r];
#pragma unroll
                    for (int c = 0; c < C; ++c) {
                        const double2 pv = Pl[(nb + j) * m + c];
#pragma unroll
                        for (int r = 0; r < R; ++r) acc[r][c] = cfma(z[r], pv, acc[r][c]);
                    }
                }
            }
        }
        // pair hand-off through the consumed Z tile ([(r*C+c)][lane], R*C*32 <= m*64)
        const int bar = 1 + pair;
        asm volatile("bar.sync %0, 64;" ::"r"(bar) : "memory");
        double2* red = Zs + lane;
        if (half == 1) {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < C; ++c) red[(r * C + c) * 32] = acc[r][c];
        }
        asm volatile("bar.sync %0, 64;" ::"r"(bar) : "memory");
        if (half == 0) {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < C; ++c) acc[r][c] = cadd(acc[r][c], red[(r * C + c) * 32]);
            const int l = l0 + k;
            const double2 sig = u.shifts[l];
            double2* zo = Zout + ((int64_t)l * m + cb) * u.LDZ + i0 + rg;
            if (interior) {
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int c = 0; c < C; ++c) zo[(int64_t)c * u.LDZ + RG * r] = acc[r][c];
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int row = i0 + rg + RG * r;
                    if (row >= r0) continue;
                    const int dd = row - dlo;
                    const bool corr = dd >= 0 && dd < u.mnb;
#pragma unroll
                    for (int c = 0; c < C; ++c) {
                        double2 v = acc[r][c];
                        if (corr) v = csub(v, cmul(sig, Pl[dd * m + c]));
                        zo[(int64_t)c * u.LDZ + RG * r] = v;
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
    }
}

}  // namespace ssd
