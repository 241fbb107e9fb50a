// Far-row update with 128-column passes and a four-way K split (m = G C, one
// column block): k_far's math and data flow (ss_far.cuh), re-balanced for
// the shared-memory budget.
//
// Measured on B200 (config 2): a pass's fixed costs -- the Z tile's trip
// through HBM, the stage wait, the partial-sum hand-off, the epilogue -- are
// ~25% of k_far's consumer time at 64-column passes, and one consumer warp
// per SM sub-partition working on 128-column passes got within 3% of two
// warps on 64-column ones.  Four pairs with two 128-column stages each do
// not fit in shared memory; here FOUR warps share one unit (each a quarter
// of the K range), so two units in flight (two groups, two stages each) keep
// two consumer warps per sub-partition with half the stages:
//   smem = 64 x 128 panel tile (64 KB) + 4 stages x (W (138 x 10) + Z tile)
//          (126 KB) + one 10 KB partial-sum buffer per group (20 KB).
// The partial sums meet without a full barrier: role 1 parks its sums over
// the consumed Z tile, role 2 in the group buffer, role 3 adds its own into
// that buffer, role 0 (the Z2 W22 part / Z2 read, then its panel columns)
// collects both and stores; mbarriers order each hand-off, and the group
// buffer is released by role 0 before role 2 of the next unit writes it.
#pragma once

#include "ss_far.cuh"

namespace ssd {

constexpr int kFar4Groups = 2, kFar4Stages = 4;
constexpr int kFar4Hdr = 256;  // 18 mbarriers
constexpr int kFar4Threads = 32 * (1 + 4 * kFar4Groups);

template <int G, int C, int R>
__host__ __device__ inline size_t far4_smem_bytes(int nb, int m) {
    const int TILE = (32 / G) * R;
    const size_t stage = ((size_t)(nb + m) * m + (size_t)m * TILE) * 16;
    return kFar4Hdr + (size_t)nb * TILE * 8 + kFar4Stages * stage + (size_t)kFar4Groups * R * C * 32 * 16;
}

template <int G, int C, int R, bool ZID>
__global__ void __launch_bounds__(kFar4Threads, 1)
    k_far4(UpdDims u, double2* Z, const double2* __restrict__ Pbuf) {
    constexpr int RG = 32 / G, M = G * C, TILE = RG * R;
    constexpr int NG = kFar4Groups, NST = kFar4Stages;
    constexpr int m = M;
    static_assert(R % 2 == 0 && NST % NG == 0, "k_far4: shape");
    extern __shared__ __align__(16) unsigned char smem[];
    const int nb = u.nb, nc = u.nc, r0 = u.r0, sb = u.sb;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [NST]
    uint64_t* empty = full + NST;                         // [NST] (count 4)
    uint64_t* zfree = empty + NST;                        // [NG] role 0 consumed Z
    uint64_t* p1 = zfree + NG;                            // [NG] role 1 partials in the Z tile
    uint64_t* pa = p1 + NG;                               // [NG] role 2 partials in the group buffer
    uint64_t* pa2 = pa + NG;                              // [NG] role 3 added into it
    uint64_t* afree = pa2 + NG;                           // [NG] role 0 read the group buffer
    double* Pan = reinterpret_cast<double*>(smem + kFar4Hdr);
    double2* Stg = reinterpret_cast<double2*>(smem + kFar4Hdr + (size_t)nb * TILE * 8);
    const size_t stage_el = (size_t)nc * m + (size_t)m * TILE;
    double2* Abuf = Stg + NST * stage_el;  // [NG][R*C][32]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ntiles = (r0 - u.rlo + TILE - 1) / TILE;
    const int64_t units = (int64_t)ntiles * sb;
    const int64_t ua = units * blockIdx.x / gridDim.x, ub = units * (blockIdx.x + 1) / gridDim.x;
    const int nun = (int)(ub - ua);

    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 4);
        }
        for (int g = 0; g < NG; ++g) {
            mbar_init(zfree + g, 1);
            mbar_init(p1 + g, 1);
            mbar_init(pa + g, 1);
            mbar_init(pa2 + g, 1);
            mbar_init(afree + g, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (nun <= 0) return;

    if (warp == 0) {
        // ---------------- producer (as k_far's) ----------------
        if (lane == 0) {
            const unsigned p12bytes = (unsigned)(nb * m * 16);
            const unsigned p22bytes = ZID ? 0u : (unsigned)(m * m * 16);
            int next[NG];
            int last[NST];
#pragma unroll
            for (int g = 0; g < NG; ++g) next[g] = g;
#pragma unroll
            for (int q = 0; q < NST; ++q) last[q] = q - NST;
            int left = nun;
            while (left > 0) {
                bool any = false;
#pragma unroll
                for (int g = 0; g < NG; ++g) {
                    const int k = next[g];
                    if (k >= nun) continue;
                    const int s = k % NST, use = k / NST;
                    int lk = 0;
#pragma unroll
                    for (int q = 0; q < NST; ++q) lk = (q == s) ? last[q] : lk;
                    if (lk != k - NST) continue;
                    if (use > 0 && !mbar_test(empty + s, (use - 1) & 1)) continue;
#pragma unroll
                    for (int q = 0; q < NST; ++q) last[q] = (q == s) ? k : last[q];
                    const int64_t unit = ua + k;
                    const int tile = (int)(unit / sb), l = (int)(unit - (int64_t)tile * sb);
                    const int i0 = u.rlo + tile * TILE;
                    const unsigned zbytes = (unsigned)(min(TILE, r0 - i0) * 16);
                    double2* st = Stg + (size_t)s * stage_el;
                    double2* zt = st + (size_t)nc * m;
                    const double2* pl = Pbuf + (int64_t)l * u.pstride;
                    mbar_expect_tx(full + s, p12bytes + p22bytes + (unsigned)m * zbytes);
                    tma_bulk_g2s(st, pl + u.p12off, p12bytes, full + s);
                    if (!ZID) tma_bulk_g2s(st + (size_t)nb * m, pl + u.p22off, p22bytes, full + s);
                    for (int c = 0; c < m; ++c)
                        tma_bulk_g2s(zt + c * TILE, Z + ((int64_t)l * m + c) * u.LDZ + i0, zbytes, full + s);
                    next[g] = k + NG;
                    --left;
                    any = true;
                }
                if (!any) __nanosleep(128);
            }
        }
        return;
    }

    // ---------------- consumers: group g, role q ----------------
    const int cw = warp - 1, grp = cw >> 2, role = cw & 3;
    const int rg = lane / G, qg = lane - rg * G;
    const int cb = qg * C;  // first output column of this lane
    const int dlo = r0 - m;
    const int jb0 = role == 0 ? 0 : u.jq[role - 1];
    const int jb1 = role == 3 ? nb : u.jq[role];
    const double* pan_l = Pan + rg * 2;
    int nu = 0;  // units this group has processed
    const int tfirst = (int)(ua / sb), tlast = (int)((ub - 1) / sb);
    for (int tile = tfirst; tile <= tlast; ++tile) {
        asm volatile("bar.sync 1, %0;" ::"r"(32 * 4 * NG) : "memory");
        {
            const int i0n = u.rlo + tile * TILE;
            for (int v = tid - 32; v < nb * TILE; v += 32 * 4 * NG) {
                const int j = v / TILE, rr = v - j * TILE;
                const int i = i0n + rr, col = u.c0 + j;
                double* dst = Pan + j * TILE + far_pan_index<G>(rr);
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
        }
        asm volatile("bar.sync 1, %0;" ::"r"(32 * 4 * NG) : "memory");
        const int ka = (int)(max(ua, (int64_t)tile * sb) - ua);
        const int kb = (int)(min(ub, (int64_t)(tile + 1) * sb) - ua);
        const int l0t = (int)(ua + ka - (int64_t)tile * sb) - ka;
        for (int k = ka + (((grp - ka) % NG) + NG) % NG; k < kb; k += NG) {
            const int l = l0t + k;
            const int i0 = u.rlo + tile * TILE;
            const bool interior = i0 + TILE <= (u.mnb > 0 ? dlo : r0);
            const int s = k % NST, use = k / NST;
            const unsigned ph = (unsigned)nu & 1u;
            mbar_wait(full + s, use & 1);
            double2* st = Stg + (size_t)s * stage_el;
            const double2* Pl = st + cb;
            double2* Zs = st + (size_t)nc * m;
            double2 acc[R][C];
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < C; ++c) acc[r][c] = cz();
            if (role == 0) {
                if (ZID) {
#pragma unroll
                    for (int c = 0; c < C; ++c)
#pragma unroll
                        for (int r = 0; r < R; ++r) acc[r][c] = Zs[(cb + c) * TILE + rg + RG * r];
                } else {
                    for (int j = 0; j < m; ++j) {
                        double2 z[R];
#pragma unroll
                        for (int r = 0; r < R; ++r) z[r] = Zs[j * TILE + rg + RG * r];
#pragma unroll
                        for (int c = 0; c < C; ++c) {
                            const double2 pv = Pl[(nb + j) * m + c];
#pragma unroll
                            for (int r = 0; r < R; ++r) acc[r][c] = cfma(z[r], pv, acc[r][c]);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(zfree + grp);
            }
#pragma unroll 2
            for (int j = jb0; j < jb1; ++j) {
                double a[R];
#pragma unroll
                for (int p = 0; p < R / 2; ++p) {
                    const double2 v = *reinterpret_cast<const double2*>(pan_l + j * TILE + p * (2 * RG));
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
            double2* redz = Zs + lane;                           // role 1: over the consumed Z tile
            double2* reda = Abuf + (size_t)grp * (R * C * 32) + lane;  // roles 2, 3: the group buffer
            if (role == 1) {
                mbar_wait(zfree + grp, ph);
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int c = 0; c < C; ++c) redz[(r * C + c) * 32] = acc[r][c];
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(p1 + grp);
                    mbar_arrive(empty + s);
                }
            } else if (role == 2) {
                if (nu > 0) mbar_wait(afree + grp, ph ^ 1u);  // role 0 read the previous unit's sums
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int c = 0; c < C; ++c) reda[(r * C + c) * 32] = acc[r][c];
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(pa + grp);
                    mbar_arrive(empty + s);
                }
            } else if (role == 3) {
                mbar_wait(pa + grp, ph);
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int c = 0; c < C; ++c)
                        reda[(r * C + c) * 32] = cadd(reda[(r * C + c) * 32], acc[r][c]);
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(pa2 + grp);
                    mbar_arrive(empty + s);
                }
            } else {
                mbar_wait(p1 + grp, ph);
                mbar_wait(pa2 + grp, ph);
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int c = 0; c < C; ++c)
                        acc[r][c] = cadd(acc[r][c], cadd(redz[(r * C + c) * 32], reda[(r * C + c) * 32]));
                __syncwarp();
                if (lane == 0) mbar_arrive(afree + grp);
                const double2 sig = u.shifts[l];
                double2* zo = Z + ((int64_t)l * m + cb) * u.LDZ + i0 + rg;
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
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + s);
            }
            ++nu;
        }
    }
}

}  // namespace ssd
