// Far-row update in ONE pass per composite: the K-streamed far kernel.
//
// Math (reference solvers.py:186-199 with the outer blocks' composite W in
// place of one window's P; same as k_far / k_far4):
//   Z_l[i, :] <- Z_l[i, :] W22_l + Pan[i, :] W12_l - sigma_l W12_l[i - (r0 - m), :]
// for the far rows i in [rlo, r0), Pan = [Chat; Ahat](:, c0 : c0 + K).
//
// k_far / k_far4 stream each (row tile, shift) unit's Z tile through HBM once
// per 64- / 128-column pass: at config 4 (m = 20) four passes per 256-column
// composite move ~25 GB of Z state per composite against ~0.5 ms of FP64
// work per GB -- ncu showed the far kernel at 44% of HBM bandwidth beside
// 55% FP64-pipe.  Here the unit's K range is streamed instead:
//  * units run shift-group-major (all row tiles of one group of S shifts,
//    then the next group), so each CTA keeps ONE group's W (S (K + m) m
//    complex, ~350 KB at m = 20) hot in L2 while it walks the tiles: the
//    148 CTAs' groups (~52 MB) plus the packed panel (~20 MB) stay L2
//    resident (tile-major order had every CTA on a different shift and
//    re-read W from HBM: 3.4x the Z traffic);
//    Teams of spl CTAs share each shift group (interleaved tiles), cutting
//    the live W working set by spl;
//  * unit = (64-row tile, S shifts); NW = S * NCB consumer warps, warp w owns
//    shift w / NCB and 10 state columns ((w % NCB) * 10 ..), its register tile
//    is 4 rows x 5 complex columns per lane over the WHOLE K range -- no
//    partial-sum hand-off, Z read once and written once per composite;
//  * the unit is a sequence of chunks through an NST-stage ring filled by one
//    producer lane with cp.async.bulk + mbarrier complete_tx:
//      nz "Z chunks"   (jz state columns of the S Z tiles + the matching jz
//                       rows of W22, for the Z W22 part), then
//      nk panel chunks (KC = 32 panel columns of the packed 64-row panel tile
//                       + the S shifts' KC rows of W12);
//  * the panel tile is packed once per composite by k_pack_panel into the
//    lane-interleaved layout (rows rg + 16 w, pairs adjacent: one LDS.128
//    feeds two rows), Chat / identity / zero rows merged, so every chunk is
//    one contiguous bulk copy regardless of ldA, p or row alignment.
#pragma once

#include "ss_far.cuh"

namespace ssd {

constexpr int kFkTile = 64;  // rows per unit
constexpr int kFarkUnroll = 4;  // panel columns unrolled in the main loop (2 / 8: same / -0.6%)
#ifndef SS_FKKC
#define SS_FKKC 32  // comparison builds vary it (tools/build_variant.sh)
#endif
constexpr int kFkKC = SS_FKKC;    // panel columns per chunk

struct FarKDims {
    int m, ptop, ident_top;
    const double* A;
    int64_t lda;
    const double* T;  // dense top rows (Chat), ptop x n
    int64_t ldt;
    const double2* shifts;
    int sb;
    int64_t LDZ;
    int r0, rlo, c0, K;  // far rows [rlo, r0), panel columns [c0, c0 + K)
    int mnb;             // lazy-shift rows: W12 rows [0, mnb) correct rows r0 - m + dd
    int64_t wstride;     // W of shift l: W + l * wstride + woff * m; rows [0, K) W12, [K, K + m) W22
    int woff;
    int nk, jz, nz, ntiles;
    int spl;  // CTAs per team (grid is a multiple of spl)
    const double* pan;  // packed panel [ntiles][nk][KC][64]
    // lazy -sigma rows: [lz0, lz0 + mnb) take W12 rows lzp + (i - lz0).
    // lzset = 0: the forward sweep's rows r0 - m .. r0 - 1 with W12 rows 0 .. m-1
    // (lz0 = r0 - M, lzp = 0); the transposed sweep sets them (its diagonal
    // entries sit at the top of the far rows, in the composite's last columns)
    int lz0 = 0, lzp = 0, lzset = 0;
    int n = 0;  // k_pack_panel_tr: rows >= n are the -I block
    // Z of shift l: Z + l zstride + zoff (0: l M LDZ / l LDZ for k_farkm) --
    // the transposed sweep runs the far pass over its z2 columns (stride
    // (m + 1) LDZ per shift) and, on k_farkm, over its w column (zoff m LDZ)
    int64_t zstride = 0, zoff = 0;
};

// The transposed sweep's panel [A^T; -I]: rows i < n are A(c, i) (row i of
// A^T; contiguous along c, so threads run along the 32 columns of a chunk),
// rows n + r are -[r == c]; zero outside [rlo, r0) x [c0, c0 + K).
__global__ void __launch_bounds__(256) k_pack_panel_tr(FarKDims u, double* __restrict__ pan) {
    const int tile = blockIdx.x / u.nk, kc = blockIdx.x - tile * u.nk;
    double* dst = pan + (size_t)blockIdx.x * kFkKC * kFkTile;
    for (int e = threadIdx.x; e < kFkKC * kFkTile; e += blockDim.x) {
        const int j = e % kFkKC, rr = e / kFkKC;
        const int i = u.rlo + tile * kFkTile + rr, jc = kc * kFkKC + j, col = u.c0 + jc;
        double v = 0.0;
        if (i < u.r0 && jc < u.K) {
            if (i < u.n) v = u.A[col + (int64_t)i * u.lda];
            else v = (i - u.n == col) ? -1.0 : 0.0;
        }
        dst[j * kFkTile + far_pan_index<2>(rr)] = v;
    }
}

template <int NCB, int S>
__host__ __device__ constexpr size_t fark_stage_bytes() {
    return (size_t)kFkKC * kFkTile * 8 + (size_t)S * kFkKC * (10 * NCB) * 16;
}
template <int NCB, int S, int NST>
__host__ __device__ constexpr size_t fark_smem_bytes() {
    return 256 + NST * fark_stage_bytes<NCB, S>();
}
// state columns per Z chunk: the S Z tiles' jz columns + jz rows of W22 fit a stage
template <int NCB, int S>
__host__ __device__ constexpr int fark_jz() {
    return (int)(fark_stage_bytes<NCB, S>() / ((size_t)S * (kFkTile + 10 * NCB) * 16));
}

// Packs Pan(:, c0 + kc*KC .. ) rows [rlo + 64 t, +64) of [top; A] into the
// chunk (t, kc): [KC columns][64 rows, lane-interleaved]; zero outside
// [rlo, r0) x [c0, c0 + K).
__global__ void __launch_bounds__(256) k_pack_panel(FarKDims u, double* __restrict__ pan) {
    const int tile = blockIdx.x / u.nk, kc = blockIdx.x - tile * u.nk;
    double* dst = pan + (size_t)blockIdx.x * kFkKC * kFkTile;
    for (int e = threadIdx.x; e < kFkKC * kFkTile; e += blockDim.x) {
        const int j = e >> 6, rr = e & 63;
        const int i = u.rlo + tile * kFkTile + rr, jc = kc * kFkKC + j, col = u.c0 + jc;
        double v = 0.0;
        if (i < u.r0 && jc < u.K) {
            if (i >= u.ptop)
                v = u.A[(i - u.ptop) + (int64_t)col * u.lda];
            else if (u.ident_top)
                v = (i == col) ? 1.0 : 0.0;
            else
                v = u.T[i + (int64_t)col * u.ldt];
        }
        dst[j * kFkTile + far_pan_index<2>(rr)] = v;
    }
}

template <int NCB, int S, int NST>
__global__ void __launch_bounds__(32 * (1 + NCB * S), 1)
    k_fark(FarKDims u, double2* Z, const double2* __restrict__ W) {
    constexpr int NW = NCB * S, M = 10 * NCB, R = 4, C = 5, RG = 16, TILE = kFkTile, KC = kFkKC;
    constexpr size_t SB = fark_stage_bytes<NCB, S>();
    constexpr size_t PANB = (size_t)KC * TILE * 8;
    static_assert(fark_jz<NCB, S>() >= 1, "k_fark: a Z chunk must fit a stage");
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [NST]
    uint64_t* empty = full + NST;                         // [NST] (count NW)
    unsigned char* stages = smem + 256;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int r0 = u.r0, sb = u.sb, K = u.K, jz = u.jz, nz = u.nz, nk = u.nk;
    const int nsu = (sb + S - 1) / S;  // shift groups per row tile
    const int64_t units = (int64_t)u.ntiles * nsu;
    // teams of u.spl CTAs share one unit range and take every spl-th unit:
    // fewer shift groups are live at once (W working set / spl)
    const int spl = u.spl, team = blockIdx.x / spl, h = blockIdx.x - team * spl, nteams = gridDim.x / spl;
    const int64_t ua0 = units * team / nteams, ub = units * (team + 1) / nteams;
    const int64_t ua = ua0 + h;
    const int nun = ua < ub ? (int)((ub - ua + spl - 1) / spl) : 0;
    const int CH = nz + nk;
    const int64_t zst = u.zstride ? u.zstride : (int64_t)M * u.LDZ;  // per-shift Z stride

    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (nun <= 0) return;

    if (warp == 0) {
        // ---------------- producer: one lane streams every chunk in order ----------------
        if (lane == 0) {
            int g = 0;
            for (int k = 0; k < nun; ++k) {
                const int64_t unit = ua + (int64_t)k * spl;
                const int grp = (int)(unit / u.ntiles), tile = (int)(unit - (int64_t)grp * u.ntiles), l0 = grp * S;
                const int ns = min(S, sb - l0);
                const int i0 = u.rlo + tile * TILE;
                const unsigned zb = (unsigned)(min(TILE, r0 - i0) * 16);
                for (int ch = 0; ch < CH; ++ch, ++g) {
                    const int s = g % NST, use = g / NST;
                    if (use > 0) mbar_wait_sleep(empty + s, (use - 1) & 1);
                    unsigned char* st = stages + (size_t)s * SB;
                    if (ch < nz) {
                        const int j0 = ch * jz, jn = min(jz, M - j0);
                        mbar_expect_tx(full + s, (unsigned)ns * (jn * zb + (unsigned)(jn * M * 16)));
                        for (int sh = 0; sh < ns; ++sh) {
                            const int64_t l = l0 + sh;
                            double2* zs = reinterpret_cast<double2*>(st) + (size_t)sh * jz * (TILE + M);
                            for (int j = 0; j < jn; ++j)
                                tma_bulk_g2s(zs + j * TILE, Z + l * zst + (int64_t)(j0 + j) * u.LDZ + i0, zb, full + s);
                            tma_bulk_g2s(zs + jz * TILE, W + l * u.wstride + (int64_t)(u.woff + K + j0) * M,
                                         (unsigned)(jn * M * 16), full + s);
                        }
                    } else {
                        const int kc = ch - nz, kcols = min(KC, K - kc * KC);
                        mbar_expect_tx(full + s, (unsigned)PANB + (unsigned)(ns * kcols * M * 16));
                        tma_bulk_g2s(st, u.pan + ((size_t)tile * nk + kc) * KC * TILE, (unsigned)PANB, full + s);
                        double2* ws = reinterpret_cast<double2*>(st + PANB);
                        for (int sh = 0; sh < ns; ++sh) {
                            const int64_t l = l0 + sh;
                            tma_bulk_g2s(ws + (size_t)sh * KC * M,
                                         W + l * u.wstride + (int64_t)(u.woff + kc * KC) * M,
                                         (unsigned)(kcols * M * 16), full + s);
                        }
                    }
                }
            }
        }
        return;
    }

    // ---------------- consumers ----------------
    const int cw = warp - 1, sw = cw / NCB, cbk = cw - sw * NCB;
    const int rg = lane >> 1, q = lane & 1;
    const int cb = cbk * 10 + q * C;  // first output column of this lane
    const int dlo = u.lzset ? u.lz0 : r0 - M;  // first lazy row
    const int dp = u.lzset ? u.lzp : 0;         // its W12 row
    int g = 0;
    for (int k = 0; k < nun; ++k) {
        const int64_t unit = ua + (int64_t)k * spl;
        const int grp = (int)(unit / u.ntiles), tile = (int)(unit - (int64_t)grp * u.ntiles), l0 = grp * S;
        const bool valid = l0 + sw < sb;
        const int64_t l = valid ? l0 + sw : 0;
        const int i0 = u.rlo + tile * TILE;
        // boundary tile: rows r0 - m + dd (dd < mnb) carry the lazy shift
        const bool interior = u.mnb == 0 || i0 + TILE <= dlo || i0 >= dlo + u.mnb;
        const double2 sig = interior ? cz() : u.shifts[l];
        double2 acc[R][C];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < C; ++c) acc[r][c] = cz();
        for (int ch = 0; ch < CH; ++ch, ++g) {
            const int s = g % NST, use = g / NST;
            mbar_wait(full + s, use & 1);
            const unsigned char* st = stages + (size_t)s * SB;
            if (valid) {
                if (ch < nz) {
                    const int j0 = ch * jz, jn = min(jz, M - j0);
                    const double2* zs = reinterpret_cast<const double2*>(st) + (size_t)sw * jz * (TILE + M);
                    const double2* w22 = zs + jz * TILE + cb;
                    for (int j = 0; j < jn; ++j) {
                        double2 z[R];
#pragma unroll
                        for (int r = 0; r < R; ++r) z[r] = zs[j * TILE + rg + RG * r];
#pragma unroll
                        for (int c = 0; c < C; ++c) {
                            const double2 pv = w22[j * M + c];
#pragma unroll
                            for (int r = 0; r < R; ++r) acc[r][c] = cfma(z[r], pv, acc[r][c]);
                        }
                    }
                } else {
                    const int kc = ch - nz, kcols = min(KC, K - kc * KC);
                    const double* pan = reinterpret_cast<const double*>(st) + rg * 2;
                    const double2* ws = reinterpret_cast<const double2*>(st + PANB) + (size_t)sw * KC * M + cb;
                    if (!interior && dp < kc * KC + kcols && dp + u.mnb > kc * KC) {
                        // acc -= sigma W12[dp + dd, :] for the lazy rows whose W12 row
                        // is in this chunk (they may span two chunks)
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            const int dd = i0 + rg + RG * r - dlo;
                            const int wr = dp + dd - kc * KC;  // chunk-local W12 row
                            if (dd >= 0 && dd < u.mnb && wr >= 0 && wr < kcols) {
#pragma unroll
                                for (int c = 0; c < C; ++c) acc[r][c] = csub(acc[r][c], cmul(sig, ws[wr * M + c]));
                            }
                        }
                    }
                    if (kcols == KC) {
#pragma unroll (kFarkUnroll)
                        for (int j = 0; j < KC; ++j) {
                            double a[R];
#pragma unroll
                            for (int p = 0; p < R / 2; ++p) {
                                const double2 v = *reinterpret_cast<const double2*>(pan + j * TILE + p * (2 * RG));
                                a[2 * p] = v.x;
                                a[2 * p + 1] = v.y;
                            }
                            // the lane's 5 W12 entries first, then rows outer: measured
                            // 4.87k vs 4.84k shifts/s at config 4 (column-outer order)
                            double2 pv[C];
#pragma unroll
                            for (int c = 0; c < C; ++c) pv[c] = ws[j * M + c];
#pragma unroll
                            for (int r = 0; r < R; ++r)
#pragma unroll
                                for (int c = 0; c < C; ++c) acc[r][c] = rfma(a[r], pv[c], acc[r][c]);
                        }
                    } else {
                        for (int j = 0; j < kcols; ++j) {
                            double a[R];
#pragma unroll
                            for (int p = 0; p < R / 2; ++p) {
                                const double2 v = *reinterpret_cast<const double2*>(pan + j * TILE + p * (2 * RG));
                                a[2 * p] = v.x;
                                a[2 * p + 1] = v.y;
                            }
#pragma unroll
                            for (int c = 0; c < C; ++c) {
                                const double2 pv = ws[j * M + c];
#pragma unroll
                                for (int r = 0; r < R; ++r) acc[r][c] = rfma(a[r], pv, acc[r][c]);
                            }
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
        }
        if (!valid) continue;
        double2* zo = Z + l * zst + (int64_t)cb * u.LDZ + i0 + rg;
        if (i0 + TILE <= r0) {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < C; ++c) zo[(int64_t)c * u.LDZ + RG * r] = acc[r][c];
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (i0 + rg + RG * r >= r0) continue;
#pragma unroll
                for (int c = 0; c < C; ++c) zo[(int64_t)c * u.LDZ + RG * r] = acc[r][c];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// m = 1 (config 3's pseudospectrum grid): the composite's far pass with the
// shifts as columns.  A unit is (64-row tile, group of kFkmShifts = 80
// shifts); consumer warp w owns shifts 10 w .. 10 w + 9 of the group (lane
// q = lane & 1 five of them) with the same 4 x 5 register tile and the same
// packed panel as k_fark.  Per shift the composite is W12 (K entries) and the
// scalar W22, stored group-major [group][row][80] (k_wsuffix1) so a KC-row chunk
// of the group's W is ONE contiguous bulk copy.  W22 is diagonal across the
// unit's columns: z <- z W22 + Pan W12 is applied in the epilogue from the Z
// values read there (no Z chunks through the ring).
// ---------------------------------------------------------------------------
constexpr int kFkmShifts = 80;
__host__ __device__ constexpr size_t farkm_stage_bytes() {
    return (size_t)kFkKC * kFkTile * 8 + (size_t)kFkKC * kFkmShifts * 16;
}
template <int NST>
__host__ __device__ constexpr size_t farkm_smem_bytes() {
    return 256 + NST * farkm_stage_bytes();
}

template <int NST>
__global__ void __launch_bounds__(32 * 9, 1) k_farkm(FarKDims u, double2* Z, const double2* __restrict__ W) {
    constexpr int S = kFkmShifts, R = 4, C = 5, RG = 16, TILE = kFkTile, KC = kFkKC;
    constexpr size_t SB = farkm_stage_bytes();
    constexpr size_t PANB = (size_t)KC * TILE * 8;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [NST]
    uint64_t* empty = full + NST;                         // [NST] (count 8)
    unsigned char* stages = smem + 256;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int r0 = u.r0, sb = u.sb, K = u.K, nk = u.nk;
    const int nsu = (sb + S - 1) / S;  // shift groups
    const int64_t units = (int64_t)u.ntiles * nsu;
    const int64_t gstride = (int64_t)u.wstride;  // complex per group: (Kmax + 1) x 80
    const int spl = u.spl, team = blockIdx.x / spl, h = blockIdx.x - team * spl, nteams = gridDim.x / spl;
    const int64_t ua0 = units * team / nteams, ub = units * (team + 1) / nteams;
    const int64_t ua = ua0 + h;
    const int nun = ua < ub ? (int)((ub - ua + spl - 1) / spl) : 0;

    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (nun <= 0) return;

    if (warp == 0) {
        if (lane == 0) {
            int g = 0;
            for (int k = 0; k < nun; ++k) {
                const int64_t unit = ua + (int64_t)k * spl;
                const int grp = (int)(unit / u.ntiles), tile = (int)(unit - (int64_t)grp * u.ntiles);
                for (int kc = 0; kc < nk; ++kc, ++g) {
                    const int s = g % NST, use = g / NST;
                    if (use > 0) mbar_wait_sleep(empty + s, (use - 1) & 1);
                    unsigned char* st = stages + (size_t)s * SB;
                    const int kcols = min(KC, K - kc * KC);
                    mbar_expect_tx(full + s, (unsigned)PANB + (unsigned)(kcols * S * 16));
                    tma_bulk_g2s(st, u.pan + ((size_t)tile * nk + kc) * KC * TILE, (unsigned)PANB, full + s);
                    tma_bulk_g2s(st + PANB, W + grp * gstride + (int64_t)kc * KC * S, (unsigned)(kcols * S * 16),
                                 full + s);
                }
            }
        }
        return;
    }

    const int cw = warp - 1;  // shifts 10 cw .. 10 cw + 9 of the group
    const int rg = lane >> 1, q = lane & 1;
    const int cb = cw * 10 + q * C;  // first of this lane's 5 shifts (group-local)
    const int dlo = u.lzset ? u.lz0 : r0 - 1;  // first lazy row
    const int dp = u.lzset ? u.lzp : 0;         // its W12 row
    const int64_t zst = u.zstride ? u.zstride : u.LDZ;
    int g = 0;
    for (int k = 0; k < nun; ++k) {
        const int64_t unit = ua + (int64_t)k * spl;
        const int grp = (int)(unit / u.ntiles), tile = (int)(unit - (int64_t)grp * u.ntiles);
        const int l0 = grp * S;
        const int i0 = u.rlo + tile * TILE;
        const bool interior = u.mnb == 0 || i0 + TILE <= dlo || i0 >= dlo + u.mnb;
        double2 acc[R][C];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < C; ++c) acc[r][c] = cz();
        for (int kc = 0; kc < nk; ++kc, ++g) {
            const int s = g % NST, use = g / NST;
            mbar_wait(full + s, use & 1);
            const unsigned char* st = stages + (size_t)s * SB;
            const int kcols = min(KC, K - kc * KC);
            const double* pan = reinterpret_cast<const double*>(st) + rg * 2;
            const double2* ws = reinterpret_cast<const double2*>(st + PANB) + cb;
            if (!interior && dp < kc * KC + kcols && dp + u.mnb > kc * KC) {
                // lazy shift: rows dlo + dd carry -sigma_l W12_l[dp + dd]
                // (forward m = 1: the one row r0 - 1 with W12 row 0)
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int dd = i0 + rg + RG * r - dlo;
                    const int wr = dp + dd - kc * KC;
                    if (dd >= 0 && dd < u.mnb && wr >= 0 && wr < kcols) {
#pragma unroll
                        for (int c = 0; c < C; ++c) {
                            const int l = min(l0 + cb + c, sb - 1);
                            acc[r][c] = csub(acc[r][c], cmul(u.shifts[l], ws[wr * S + c]));
                        }
                    }
                }
            }
#pragma unroll 4
            for (int j = 0; j < kcols; ++j) {
                double a[R];
#pragma unroll
                for (int p = 0; p < R / 2; ++p) {
                    const double2 v = *reinterpret_cast<const double2*>(pan + j * TILE + p * (2 * RG));
                    a[2 * p] = v.x;
                    a[2 * p + 1] = v.y;
                }
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const double2 pv = ws[j * S + c];
#pragma unroll
                    for (int r = 0; r < R; ++r) acc[r][c] = rfma(a[r], pv, acc[r][c]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
        }
        // epilogue: z <- z W22 + acc for the lane's 4 rows x 5 shifts
        // (every load before any store: Z is not restrict)
        const double2* w22 = W + grp * gstride + (int64_t)K * S + cb;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int64_t l = l0 + cb + c;
            if (l >= sb) continue;
            const double2 wz = w22[c];
            const double2* zc = Z + l * zst + u.zoff + i0 + rg;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (i0 + rg + RG * r < r0) acc[r][c] = cfma(__ldg(zc + RG * r), wz, acc[r][c]);
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int64_t l = l0 + cb + c;
            if (l >= sb) continue;
            double2* zc = Z + l * zst + u.zoff + i0 + rg;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (i0 + rg + RG * r < r0) zc[RG * r] = acc[r][c];
        }
    }
}

}  // namespace ssd
