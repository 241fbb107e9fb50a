// K-streamed far kernel on the FP64 tensor cores (DMMA): k_farkd.
//
// Same math, units, producer and ring as k_fark (ss_fark.cuh):
//   Z_l[i, :] <- Z_l[i, :] W22_l + Pan[i, :] W12_l - sigma_l W12_l[lazy row of i, :]
// but the consumer warps run mma.sync.m16n8k8.f64 instead of DFMA.  Viewing
// the complex m-column state as 2m interleaved real columns (the double2
// storage order), both products are REAL GEMMs:
//   * panel part: Z(64 x 2m) += Pan(64 x K, real) W12(K x 2m, real view);
//   * state part: Z(64 x 2m) = Z_old(64 x 2m) W22e(2m x 2m), with W22e the
//     real 2 x 2 block expansion [[re, im], [-im, re]] of each W22 entry.
// A DMMA instruction carries 16x as many FMAs per issue slot as a DFMA, so
// the consumer no longer spends its issue bandwidth on operand loads and
// fixed-latency waits (k_fark: 64% of the FP64 pipe with issue 44% active).
//
// Warp layout: WR x WC warps per shift, warp (shift sw, wr, wc) owns the
// m16 row tiles wr, wr + WR, .. (MT = 4 / WR) and a range of NTW of the
// NT = ceil(m / 4) n8 column tiles (the last one partial when m % 4 != 0,
// its missing columns predicated to zero).  The accumulators must fit the
// register budget of 9 warps per CTA (168 per thread: one SM sub-partition
// holds 3 of them), hence column-split warps for wide m.  Accumulator fragment (i, nt): c0 + i c1 is
// the complex entry (row gq, column 4 nt + tq), c2 + i c3 the one 8 rows
// below.
//
// The panel chunk is packed by k_pack_panel_d in DMMA fragment order: for
// k-step ks (8 panel columns) and m16 tile mt, the 32 lanes' (a0, a1) pairs
// then their (a2, a3) pairs -- two conflict-free LDS.128 per fragment.
#pragma once

#include "ss_fark.cuh"

namespace ssd {

__device__ __forceinline__ void dmma8(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

// packed index of panel element (column j of the chunk, tile row rr)
__host__ __device__ inline int farkd_pan_index(int j, int rr) {
    const int ks = j >> 3, kk = j & 7, mt = rr >> 4, rl = rr & 15;
    const int gq = rl & 7, hi = rl >> 3, tq = kk & 3, khi = kk >> 2;
    const int v = hi + 2 * khi, lane = gq * 4 + tq;
    return (((ks * 4 + mt) * 2 + (v >> 1)) * 32 + lane) * 2 + (v & 1);
}

// k_pack_panel in fragment order (zero outside [rlo, r0) x [c0, c0 + K))
__global__ void __launch_bounds__(256) k_pack_panel_d(FarKDims u, double* __restrict__ pan) {
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
        dst[farkd_pan_index(j, rr)] = v;
    }
}

// k_pack_panel_tr in fragment order: rows i < n are A(c, i), rows n + r are
// -[r == c]; zero outside [rlo, r0) x [c0, c0 + K)
__global__ void __launch_bounds__(256) k_pack_panel_tr_d(FarKDims u, double* __restrict__ pan) {
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
        dst[farkd_pan_index(j, rr)] = v;
    }
}

// state columns per Z chunk: k_fark's, rounded down to a multiple of 4 (one
// k8 step = 4 complex columns)
template <int NCB, int S>
__host__ __device__ constexpr int farkd_jz() {
    return fark_jz<NCB, S>() & ~3;
}

template <int NCB, int S, int NST, int WR, int WC>
__global__ void __launch_bounds__(32 * (1 + WR * WC * S), 1)
    k_farkd(FarKDims u, double2* Z, const double2* __restrict__ W) {
    // WR x WC warps per shift; warp (wr, wc) owns the m16 row tiles wr,
    // wr + WR, .. and the n8 column tiles [wc NTW, wc NTW + NTW) (the last
    // one partial when 2m % 8 != 0)
    constexpr int WPS = WR * WC, NW = WPS * S, M = 10 * NCB, TILE = kFkTile, KC = kFkKC;
    constexpr int MT = 4 / WR, M2 = 2 * M, NT = (M2 + 7) / 8, NTW = (NT + WC - 1) / WC;
    static_assert(WR == 1 || WR == 2 || WR == 4, "k_farkd: 4 row tiles per unit");
    constexpr size_t SB = fark_stage_bytes<NCB, S>();
    constexpr size_t PANB = (size_t)KC * TILE * 8;
    static_assert(farkd_jz<NCB, S>() >= 4, "k_farkd: a Z chunk must hold one k8 step");
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [NST]
    uint64_t* empty = full + NST;                         // [NST] (count NW)
    unsigned char* stages = smem + 256;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int r0 = u.r0, sb = u.sb, K = u.K, jz = u.jz, nz = u.nz, nk = u.nk;
    const int nsu = (sb + S - 1) / S;
    const int64_t units = (int64_t)u.ntiles * nsu;
    const int spl = u.spl, team = blockIdx.x / spl, h = blockIdx.x - team * spl, nteams = gridDim.x / spl;
    const int64_t ua0 = units * team / nteams, ub = units * (team + 1) / nteams;
    const int64_t ua = ua0 + h;
    const int nun = ua < ub ? (int)((ub - ua + spl - 1) / spl) : 0;
    const int CH = nz + nk;
    const int64_t zst = u.zstride ? u.zstride : (int64_t)M * u.LDZ;

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
        // ---------------- producer (as k_fark) ----------------
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
    const int cw = warp - 1, sw = cw / WPS, wr = (cw - sw * WPS) % WR, wc = (cw - sw * WPS) / WR;
    const int gq = lane >> 2, tq = lane & 3;
    const int t0 = WC == 1 ? 0 : wc * NTW;  // first n8 tile of this warp
    // every tile full and every warp's tile range in bounds: no predicates
    constexpr bool EXACT = (M2 % 8 == 0) && (NT % WC == 0);
    // m % 4 == 0: every k8 step of the state part is full (jz % 4 == 0)
    constexpr bool ZEX = M % 4 == 0;
    const int dlo = u.lzset ? u.lz0 : r0 - M;
    const int dp = u.lzset ? u.lzp : 0;
    // the lane's B column (real) of its n8 tile t: 8 (t0 + t) + gq; complex
    // output column of its accumulators: 4 (t0 + t) + tq
    auto bcol_ok = [&](int t) { return EXACT || 8 * (t0 + t) + gq < M2; };
    auto ccol_ok = [&](int t) { return EXACT || 4 * (t0 + t) + tq < M; };
    auto tile_ok = [&](int t) { return EXACT || t0 + t < NT; };
    // the lane's element of the 2 x 2 expansion of a W22 entry (state part):
    // row parity pj = tq & 1, column parity pc = gq & 1
    const int wsel = ((tq ^ gq) & 1);                                    // 0: re, 1: im
    const long long wneg = ((tq & 1) && !(gq & 1)) ? (long long)0x8000000000000000ULL : 0;  // -im
    int g = 0;
    for (int k = 0; k < nun; ++k) {
        const int64_t unit = ua + (int64_t)k * spl;
        const int grp = (int)(unit / u.ntiles), tile = (int)(unit - (int64_t)grp * u.ntiles), l0 = grp * S;
        const bool valid = l0 + sw < sb;
        const int64_t l = valid ? l0 + sw : 0;
        const int i0 = u.rlo + tile * TILE;
        const bool interior = u.mnb == 0 || i0 + TILE <= dlo || i0 >= dlo + u.mnb;
        const double2 sig = interior ? cz() : u.shifts[l];
        double acc[MT][NTW][4];
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int t = 0; t < NTW; ++t)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[i][t][v] = 0.0;
        for (int ch = 0; ch < CH; ++ch, ++g) {
            const int s = g % NST, use = g / NST;
            mbar_wait(full + s, use & 1);
            const unsigned char* st = stages + (size_t)s * SB;
            if (valid) {
                if (ch < nz) {
                    // state part: A = Z_old (real view), B = W22e; k8 step = 4
                    // complex state columns (the chunk's last step may be partial)
                    const int j0 = ch * jz, jn = min(jz, M - j0);
                    const double* zsd = reinterpret_cast<const double*>(st) + (size_t)sw * jz * (TILE + M) * 2;
                    const double* w22d = zsd + (size_t)jz * TILE * 2;
                    for (int kb = 0; kb < jn; kb += 4) {
                        const int kn = jn - kb;  // complex columns left in this step
                        double a[MT][4], b[NTW][2];
#pragma unroll
                        for (int i = 0; i < MT; ++i)
#pragma unroll
                            for (int v = 0; v < 4; ++v) {
                                const int row = 16 * (wr + WR * i) + gq + 8 * (v & 1), kk = tq + 4 * (v >> 1);
                                a[i][v] = ZEX || (kk >> 1) < kn ? zsd[((kb + (kk >> 1)) * TILE + row) * 2 + (kk & 1)] : 0.0;
                            }
#pragma unroll
                        for (int t = 0; t < NTW; ++t)
#pragma unroll
                            for (int v = 0; v < 2; ++v) {
                                const int kk = tq + 4 * v;
                                double bv = 0.0;
                                if ((ZEX || (kk >> 1) < kn) && bcol_ok(t)) {
                                    // W22e[2j + pj][2c + pc] = pj == pc ? re : (pj ? -im : im):
                                    // one 8-byte load at a lane-constant offset, sign by XOR
                                    const double w =
                                        w22d[((kb + (kk >> 1)) * M + 4 * (t0 + t) + (gq >> 1)) * 2 + wsel];
                                    bv = __longlong_as_double(__double_as_longlong(w) ^ wneg);
                                }
                                b[t][v] = bv;
                            }
#pragma unroll
                        for (int i = 0; i < MT; ++i)
#pragma unroll
                            for (int t = 0; t < NTW; ++t)
                                if (tile_ok(t)) dmma8(acc[i][t], a[i], b[t]);
                    }
                } else {
                    const int kc = ch - nz, kcols = min(KC, K - kc * KC);
                    const double* pan = reinterpret_cast<const double*>(st);
                    const double* wsd = reinterpret_cast<const double*>(st + PANB) + (size_t)sw * KC * M2;
                    if (!interior && dp < kc * KC + kcols && dp + u.mnb > kc * KC) {
                        // acc -= sigma W12[dp + dd, :] for the lazy rows in this chunk
                        const double2* ws = reinterpret_cast<const double2*>(wsd);
#pragma unroll
                        for (int i = 0; i < MT; ++i)
#pragma unroll
                            for (int hh = 0; hh < 2; ++hh) {
                                const int dd = i0 + 16 * (wr + WR * i) + gq + 8 * hh - dlo;
                                const int wrow = dp + dd - kc * KC;
                                if (dd >= 0 && dd < u.mnb && wrow >= 0 && wrow < kcols) {
#pragma unroll
                                    for (int t = 0; t < NTW; ++t) {
                                        if (!ccol_ok(t)) continue;
                                        const double2 d = cmul(sig, ws[wrow * M + 4 * (t0 + t) + tq]);
                                        acc[i][t][2 * hh] -= d.x;
                                        acc[i][t][2 * hh + 1] -= d.y;
                                    }
                                }
                            }
                    }
                    const int nks = (kcols + 7) >> 3;
                    for (int ks = 0; ks < nks; ++ks) {
                        double a[MT][4], b[NTW][2];
#pragma unroll
                        for (int i = 0; i < MT; ++i) {
                            const double* pa = pan + ((ks * 4 + wr + WR * i) * 2) * 64 + lane * 2;
                            const double2 lo = *reinterpret_cast<const double2*>(pa);
                            const double2 hi = *reinterpret_cast<const double2*>(pa + 64);
                            a[i][0] = lo.x;
                            a[i][1] = lo.y;
                            a[i][2] = hi.x;
                            a[i][3] = hi.y;
                        }
                        const int k0 = ks * 8 + tq, k1 = k0 + 4;
                        // W12 rows past the composite are not copied (stale): zero them
                        const bool full8 = ks * 8 + 8 <= kcols;
#pragma unroll
                        for (int t = 0; t < NTW; ++t) {
                            const bool cok = bcol_ok(t);
                            const int c = 8 * (t0 + t) + gq;
                            b[t][0] = cok && (full8 || k0 < kcols) ? wsd[k0 * M2 + c] : 0.0;
                            b[t][1] = cok && (full8 || k1 < kcols) ? wsd[k1 * M2 + c] : 0.0;
                        }
#pragma unroll
                        for (int i = 0; i < MT; ++i)
#pragma unroll
                            for (int t = 0; t < NTW; ++t)
                                if (tile_ok(t)) dmma8(acc[i][t], a[i], b[t]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
        }
        if (!valid) continue;
        double2* zo = Z + l * zst;
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const int row = i0 + 16 * (wr + WR * i) + gq + 8 * hh;
                if (row >= r0) continue;
#pragma unroll
                for (int t = 0; t < NTW; ++t)
                    if (ccol_ok(t))
                        zo[(int64_t)(4 * (t0 + t) + tq) * u.LDZ + row] =
                            make_double2(acc[i][t][2 * hh], acc[i][t][2 * hh + 1]);
            }
    }
}

// ---------------------------------------------------------------------------
// k_farkm on the tensor cores (m = 1: config 3's far pass; the transposed
// sweep's w column): the group's 80 shifts are the 160 interleaved real
// columns of one real GEMM  Z(64 x 160) += Pan(64 x K) W12(K x 160)  (the
// group-major W rows are exactly that matrix), W22 diagonal across the
// columns in the epilogue.  8 consumer warps: 2 row groups (2 m16 tiles
// each) x 4 column groups (5 n8 tiles = 20 shifts each).
template <int NST>
__global__ void __launch_bounds__(32 * 9, 1) k_farkmd(FarKDims u, double2* Z, const double2* __restrict__ W) {
    constexpr int S = kFkmShifts, TILE = kFkTile, KC = kFkKC, WR = 2, MT = 2, NTW = 5, S2 = 2 * S;
    constexpr size_t SB = farkm_stage_bytes();
    constexpr size_t PANB = (size_t)KC * TILE * 8;
    static_assert(4 * NTW * 8 == S2, "k_farkmd: 4 column groups of 5 n8 tiles");
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [NST]
    uint64_t* empty = full + NST;                         // [NST] (count 8)
    unsigned char* stages = smem + 256;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int r0 = u.r0, sb = u.sb, K = u.K, nk = u.nk;
    const int nsu = (sb + S - 1) / S;
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

    const int cw = warp - 1, wr = cw % WR, wc = cw / WR;
    const int gq = lane >> 2, tq = lane & 3;
    const int t0 = wc * NTW;
    const int dlo = u.lzset ? u.lz0 : r0 - 1;
    const int dp = u.lzset ? u.lzp : 0;
    const int64_t zst = u.zstride ? u.zstride : u.LDZ;
    int g = 0;
    for (int k = 0; k < nun; ++k) {
        const int64_t unit = ua + (int64_t)k * spl;
        const int grp = (int)(unit / u.ntiles), tile = (int)(unit - (int64_t)grp * u.ntiles);
        const int l0 = grp * S;
        const int i0 = u.rlo + tile * TILE;
        const bool interior = u.mnb == 0 || i0 + TILE <= dlo || i0 >= dlo + u.mnb;
        double acc[MT][NTW][4];
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int t = 0; t < NTW; ++t)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[i][t][v] = 0.0;
        for (int kc = 0; kc < nk; ++kc, ++g) {
            const int s = g % NST, use = g / NST;
            mbar_wait(full + s, use & 1);
            const unsigned char* st = stages + (size_t)s * SB;
            const int kcols = min(KC, K - kc * KC);
            const double* pan = reinterpret_cast<const double*>(st);
            const double* wsd = reinterpret_cast<const double*>(st + PANB);
            if (!interior && dp < kc * KC + kcols && dp + u.mnb > kc * KC) {
                // lazy shift: rows dlo + dd carry -sigma_l W12_l[dp + dd]
                const double2* ws = reinterpret_cast<const double2*>(wsd);
#pragma unroll
                for (int i = 0; i < MT; ++i)
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const int dd = i0 + 16 * (wr + WR * i) + gq + 8 * hh - dlo;
                        const int wrow = dp + dd - kc * KC;
                        if (dd >= 0 && dd < u.mnb && wrow >= 0 && wrow < kcols) {
#pragma unroll
                            for (int t = 0; t < NTW; ++t) {
                                const int c = 4 * (t0 + t) + tq;
                                const int l = min(l0 + c, sb - 1);
                                const double2 d = cmul(u.shifts[l], ws[wrow * S + c]);
                                acc[i][t][2 * hh] -= d.x;
                                acc[i][t][2 * hh + 1] -= d.y;
                            }
                        }
                    }
            }
            const int nks = (kcols + 7) >> 3;
            for (int ks = 0; ks < nks; ++ks) {
                double a[MT][4], b[NTW][2];
#pragma unroll
                for (int i = 0; i < MT; ++i) {
                    const double* pa = pan + ((ks * 4 + wr + WR * i) * 2) * 64 + lane * 2;
                    const double2 lo = *reinterpret_cast<const double2*>(pa);
                    const double2 hi = *reinterpret_cast<const double2*>(pa + 64);
                    a[i][0] = lo.x;
                    a[i][1] = lo.y;
                    a[i][2] = hi.x;
                    a[i][3] = hi.y;
                }
                const int k0 = ks * 8 + tq, k1 = k0 + 4;
                const bool full8 = ks * 8 + 8 <= kcols;
#pragma unroll
                for (int t = 0; t < NTW; ++t) {
                    const int c = 8 * (t0 + t) + gq;
                    b[t][0] = full8 || k0 < kcols ? wsd[k0 * S2 + c] : 0.0;
                    b[t][1] = full8 || k1 < kcols ? wsd[k1 * S2 + c] : 0.0;
                }
#pragma unroll
                for (int i = 0; i < MT; ++i)
#pragma unroll
                    for (int t = 0; t < NTW; ++t) dmma8(acc[i][t], a[i], b[t]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
        }
        // epilogue: z <- z W22 + acc (every load before any store: Z is not restrict)
        const double2* w22 = W + grp * gstride + (int64_t)K * S;
#pragma unroll
        for (int t = 0; t < NTW; ++t) {
            const int c = 4 * (t0 + t) + tq;
            const int64_t l = l0 + c;
            if (l >= sb) continue;
            const double2 wz = w22[c];
            const double2* zc = Z + l * zst + u.zoff;
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int row = i0 + 16 * (wr + WR * i) + gq + 8 * hh;
                    if (row < r0) {
                        const double2 z = __ldg(zc + row);
                        const double2 r = cfma(z, wz, make_double2(acc[i][t][2 * hh], acc[i][t][2 * hh + 1]));
                        acc[i][t][2 * hh] = r.x;
                        acc[i][t][2 * hh + 1] = r.y;
                    }
                }
        }
#pragma unroll
        for (int t = 0; t < NTW; ++t) {
            const int c = 4 * (t0 + t) + tq;
            const int64_t l = l0 + c;
            if (l >= sb) continue;
            double2* zc = Z + l * zst + u.zoff;
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int row = i0 + 16 * (wr + WR * i) + gq + 8 * hh;
                    if (row < r0) zc[row] = make_double2(acc[i][t][2 * hh], acc[i][t][2 * hh + 1]);
                }
        }
    }
}

}  // namespace ssd
