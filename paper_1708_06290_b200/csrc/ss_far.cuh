// Persistent warp-specialised far-row update of the two-level sweep.
//
// Same math as k_update_ws (ss_update_ws.cuh) -- per shift l and far row i
//   Zout_l[i, :] = Zin_l[i, :] P22_l + Pan[i, :] P12_l - sigma_l P12_l[i - (r0 - m), :]
// (reference solvers.py:186-199 with the outer block's composite W in place
// of one window's P) -- restructured after ncu showed ~19% of the consumer
// warps' time waiting in k_update_ws:
//  * persistent: one CTA per SM walks a contiguous range of (64-row tile,
//    shift) units in tile-major order, so the stage ring never drains between
//    CTAs and the 64 x nb panel tile is restaged only when the range crosses
//    a tile boundary (consumer-only named barrier; the producer keeps
//    prefetching across it);
//  * asynchronous pair hand-off: in a consumer pair, half 0 does the Z2 part
//    FIRST and signals "Z tile consumed" (mbarrier), then its panel columns;
//    half 1 does its panel columns, waits for that signal, writes its partial
//    sums over the Z tile and signals "partials ready"; only half 0 waits for
//    the partials, after its own work -- no pair-wide bar.sync;
//  * the producer parks on the empty barriers with a suspend-time hint.
#pragma once

#include "ss_update_ws.cuh"

namespace ssd {

#ifndef SS_FAR_NAP
#define SS_FAR_NAP 128  // producer back-off (ns) when no stage is free
#endif

// Tile shape (template): lane = (row group rg < 32/G, column group q < G),
// R rows x C columns per lane, tile = (32/G) R rows.  NPAIR consumer pairs,
// NST ring stages.
__host__ __device__ constexpr int far_threads(int npair) { return 32 * (1 + 2 * npair); }

__host__ __device__ inline size_t far_smem_bytes(int nb, int m, int tile, int nst) {
    const int nc = nb + m;
    const size_t stage = ((size_t)nc * m + (size_t)m * tile) * 16;
    return 256 + (size_t)nb * tile * 8 + nst * stage;
}

// panel position of tile row `row`: lane row group rg owns rows rg + RG*w;
// rows (rg + RG*2p, rg + RG*(2p+1)) are adjacent so one LDS.128 feeds two
template <int G>
__device__ __forceinline__ int far_pan_index(int row) {
    constexpr int RG = 32 / G;
    const int rg = row % RG, w = row / RG, p = w >> 1, e = w & 1;
    return p * (2 * RG) + rg * 2 + e;
}

// NCB column blocks: a unit's m = NCB G C columns are split over a group of
// NCB pairs (pair cbk owns columns [cbk G C, (cbk + 1) G C)); the group shares
// the unit's stage (P for all m columns, the 64 x m Z tile: every pair's Z2
// part needs all m state columns).
//
// MSH (m = 1 only): the M = G C NCB "columns" of a unit are M different
// shifts (one state column each); the stage holds their P vectors [q][nb+1]
// and Z tiles [q][TILE], the Z2 part is the per-shift scalar W22 and the
// lazy-shift correction uses each column's own sigma.  Turns the
// LSU-bound one-column update of config 3 into the m = 10 register tile.
template <int G, int C, int R, int NPAIR, int NST, bool ZID, int NCB = 1, bool MSH = false>
__global__ void __launch_bounds__(far_threads(NPAIR), 1)
    k_far(UpdDims u, double2* Z, const double2* __restrict__ Pbuf) {
    constexpr int RG = 32 / G, MB = G * C, M = MB * NCB, TILE = RG * R;
    constexpr int NG = NPAIR / NCB;  // consumer groups (one unit each at a time)
    constexpr int m = M;
    // every group owns NST / NG stages outright: a stage shared by several
    // groups would let a fast group pass a full-barrier parity test two uses
    // ahead (phase aliasing)
    static_assert(R % 2 == 0 && 2 * NST + 2 * NPAIR <= 32 && NPAIR % NCB == 0 && NST % NG == 0,
                  "k_far: shape");
    extern __shared__ __align__(16) unsigned char smem[];
    const int nb = u.nb, nc = u.nc, r0 = u.r0, sb = u.sb;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [NST]
    uint64_t* empty = full + NST;                          // [NST]
    uint64_t* zfree = empty + NST;                         // [NG] (count NCB)
    uint64_t* partr = zfree + NPAIR;                       // [NPAIR]
    double* Pan = reinterpret_cast<double*>(smem + 256);   // [nb][TILE] pair-interleaved
    double2* Stg = reinterpret_cast<double2*>(smem + 256 + (size_t)nb * TILE * 8);
    const size_t stage_el = (size_t)nc * m + (size_t)m * TILE;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ntiles = (r0 - u.rlo + TILE - 1) / TILE;
    const int su = MSH ? (sb + M - 1) / M : sb;  // units per row tile
    const int64_t units = (int64_t)ntiles * su;
    const int64_t ua = units * blockIdx.x / gridDim.x, ub = units * (blockIdx.x + 1) / gridDim.x;
    const int nun = (int)(ub - ua);

    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 2 * NCB);
        }
        for (int p = 0; p < NPAIR; ++p) {
            mbar_init(zfree + p, NCB);
            mbar_init(partr + p, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (nun <= 0) return;

    if (warp == 0) {
        // ---------------- producer ----------------
        // Unit k belongs to pair k % NPAIR and stage k % NST.  The producer
        // refills whichever pair's next stage is free first (non-blocking
        // polls), so one slow pair does not hold back the others' prefetch.
        if (lane == 0) {
            const unsigned p12bytes = (unsigned)(nb * m * 16);
            const unsigned p22bytes = ZID ? 0u : (unsigned)(m * m * 16);
            // a stage may serve several pairs in turn (NST % NPAIR != 0): its
            // uses must be issued in unit order, or the parity test on its
            // empty barrier could alias two phases ahead
            int next[NG];
            int last[NST];  // last unit issued into each stage
#pragma unroll
            for (int p = 0; p < NG; ++p) next[p] = p;
#pragma unroll
            for (int q = 0; q < NST; ++q) last[q] = q - NST;
            int left = nun;
            while (left > 0) {
                bool any = false;
#pragma unroll
                for (int p = 0; p < NG; ++p) {
                    const int k = next[p];
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
                    const int tile = (int)(unit / su), l = (int)(unit - (int64_t)tile * su);
                    const int i0 = u.rlo + tile * TILE;
                    const unsigned zbytes = (unsigned)(min(TILE, r0 - i0) * 16);
                    double2* st = Stg + (size_t)s * stage_el;
                    double2* zt = st + (size_t)nc * m;
                    if (MSH) {
                        const int nq = min(M, sb - l * M);
                        const unsigned pq = (unsigned)((ZID ? nb : nb + 1) * 16);
                        mbar_expect_tx(full + s, (unsigned)nq * (pq + zbytes));
                        for (int q = 0; q < nq; ++q) {
                            const int64_t lq = (int64_t)l * M + q;
                            tma_bulk_g2s(st + (size_t)q * nc, Pbuf + lq * u.pstride + u.p12off, pq,
                                         full + s);
                            tma_bulk_g2s(zt + q * TILE, Z + lq * u.LDZ + i0, zbytes, full + s);
                        }
                    } else {
                        const double2* pl = Pbuf + (int64_t)l * u.pstride;
                        mbar_expect_tx(full + s, p12bytes + p22bytes + (unsigned)m * zbytes);
                        tma_bulk_g2s(st, pl + u.p12off, p12bytes, full + s);
                        if (!ZID) tma_bulk_g2s(st + (size_t)nb * m, pl + u.p22off, p22bytes, full + s);
                        for (int c = 0; c < m; ++c)
                            tma_bulk_g2s(zt + c * TILE, Z + ((int64_t)l * m + c) * u.LDZ + i0, zbytes,
                                         full + s);
                    }
                    next[p] = k + NG;
                    --left;
                    any = true;
                }
                if (!any) __nanosleep(SS_FAR_NAP);
            }
        }
        return;
    }

    // ---------------- consumers ----------------
    const int cw = warp - 1, pair = cw >> 1, half = cw & 1;
    const int grp = pair / NCB, cbk = pair - grp * NCB;
    const int rg = lane / G, q = lane - rg * G;
    const int cb = cbk * MB + q * C;  // first output column of this lane
    const int dlo = r0 - (MSH ? 1 : m);
    const int jlo = half == 0 ? 0 : u.jh;
    const int jhi = half == 1 ? nb : u.jh;
    const double* pan_l = Pan + rg * 2;
    int npair = 0;  // units this pair has processed (mbarrier phase of zfree / partr)
    const int tfirst = (int)(ua / su), tlast = (int)((ub - 1) / su);
    for (int tile = tfirst; tile <= tlast; ++tile) {
        // (re)stage the panel tile: every consumer is done with the old one
        asm volatile("bar.sync 1, %0;" ::"r"(32 * 2 * NPAIR) : "memory");
        {
            const int i0n = u.rlo + tile * TILE;
            for (int v = tid - 32; v < nb * TILE; v += 32 * 2 * NPAIR) {
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
        asm volatile("bar.sync 1, %0;" ::"r"(32 * 2 * NPAIR) : "memory");
        // this tile's units of the CTA range: k in [ka, kb); pair p takes k = p mod 4
        const int ka = (int)(max(ua, (int64_t)tile * su) - ua);
        const int kb = (int)(min(ub, (int64_t)(tile + 1) * su) - ua);
        const int l0t = (int)(ua + ka - (int64_t)tile * su) - ka;  // l = l0t + k
        for (int k = ka + (((grp - ka) % NG) + NG) % NG; k < kb; k += NG) {
        const int l = l0t + k;
        const int i0 = u.rlo + tile * TILE;
        const bool interior = i0 + TILE <= (u.mnb > 0 ? dlo : r0);
        const int s = k % NST, use = k / NST;
        mbar_wait(full + s, use & 1);
        double2* st = Stg + (size_t)s * stage_el;
        const double2* Pl = st + cb;
        double2* Zs = st + (size_t)nc * m;
        double2 acc[R][C];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < C; ++c) acc[r][c] = cz();
        if (half == 0) {
            // Z2 part first, then release the Z tile to the partner
            if (ZID) {
#pragma unroll
                for (int c = 0; c < C; ++c)
#pragma unroll
                    for (int r = 0; r < R; ++r) acc[r][c] = Zs[(cb + c) * TILE + rg + RG * r];
            } else if (MSH) {
                // per-shift scalar W22
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const double2 w22 = st[(cb + c) * nc + nb];
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        acc[r][c] = cmul(Zs[(cb + c) * TILE + rg + RG * r], w22);
                }
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
        for (int j = jlo; j < jhi; ++j) {
            double a[R];
#pragma unroll
            for (int p = 0; p < R / 2; ++p) {
                const double2 v = *reinterpret_cast<const double2*>(pan_l + j * TILE + p * (2 * RG));
                a[2 * p] = v.x;
                a[2 * p + 1] = v.y;
            }
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const double2 pv = MSH ? st[(cb + c) * nc + j] : Pl[j * m + c];
#pragma unroll
                for (int r = 0; r < R; ++r) acc[r][c] = rfma(a[r], pv, acc[r][c]);
            }
        }
        double2* red = Zs + cbk * (MB * TILE) + lane;  // [(r*C + c)][lane] over the consumed Z tile
        if (half == 1) {
            mbar_wait(zfree + grp, npair & 1);
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < C; ++c) red[(r * C + c) * 32] = acc[r][c];
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(partr + pair);
                mbar_arrive(empty + s);
            }
        } else {
            mbar_wait(partr + pair, npair & 1);
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < C; ++c) acc[r][c] = cadd(acc[r][c], red[(r * C + c) * 32]);
            if (MSH) {
                // column c is shift l M + cb + c (state column 0)
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const int64_t lq = (int64_t)l * M + cb + c;
                    if (lq >= sb) continue;
                    const double2 sgq = u.shifts[lq];
                    double2* zq = Z + lq * u.LDZ + i0 + rg;
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int row = i0 + rg + RG * r;
                        if (!interior && row >= r0) continue;
                        double2 v = acc[r][c];
                        if (!interior && row == dlo && u.mnb > 0)
                            v = csub(v, cmul(sgq, st[(cb + c) * nc]));
                        zq[RG * r] = v;
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + s);
                ++npair;
                continue;
            }
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
        ++npair;
        }
    }
}

}  // namespace ssd
