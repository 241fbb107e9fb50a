// Window block RQ for wide blocks, m + 1 > 32 (config 5: m = 50), by row
// Householder reflectors -- the B200 replacement of the reference's scheduled
// Givens batch (batched.py:64-122) where k_rq_house's one-lane-per-row
// register window (L <= 32) does not fit.
//
// Same math as k_rq_house / k_block (kernels.py:74-99's sign rule, the
// unnormalised form H = I - kappa v v^H): bottom-up over the nb rows of the
// window, row t's reflector maps its active columns t..t+m to (0,..,0,beta);
// rows above are updated; P = H_{nb-1}(...(H_0 E)) by reverse accumulation.
// One CTA (8 warps) per shift; the nb x L active windows live in shared
// memory as circular buffers (slot = column mod L: the column retiring at
// step t, t + m, and the one entering, t - 1, share a slot), the reflectors
// v_t in shared memory for the accumulation.  Per step: warp 0 builds the
// reflector (warp reductions), then every warp updates rows i = warp mod 8
// (each lane two entries of the row, a warp reduction for the dot product)
// and slides the next panel entry into the retired slot.  The reverse
// accumulation keeps each column of P as a full (nb + m)-vector in shared
// memory (no sliding), one warp per column.
//
// With the reflectors not limited by a register window, the one-level sweep
// can use wider windows for large m (nb = 96: the window-update overhead
// 2m/nb drops from 156% at nb = 64 to 104%).
#pragma once

#include "ss_rq_house.cuh"

namespace ssd {

constexpr int kRqBigThreads = 256;

// accumulation vectors (one per warp) reuse the windows' space when it is large enough
__host__ __device__ inline bool rq_big_acc_in_win(int nb, int m) {
    return (size_t)(kRqBigThreads / 32) * (nb + m) <= (size_t)nb * (m + 1);
}
__host__ __device__ inline size_t rq_big_smem_bytes(int nb, int m) {
    const int L = m + 1;
    const size_t win = (size_t)2 * nb * L + nb;  // windows, reflectors, kappa
    const size_t acc = (size_t)(kRqBigThreads / 32) * (nb + m);
    return (win + (rq_big_acc_in_win(nb, m) ? 0 : acc)) * 16;
}

__device__ __forceinline__ double2 warp_csum(double2 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    return v;
}

__global__ void __launch_bounds__(kRqBigThreads)
    k_rq_big(RqDims d, const double2* __restrict__ Z2, double2* __restrict__ Pbuf) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int nb = d.nb, m = d.m, L = m + 1;  // L <= 64
    double2* Zw = reinterpret_cast<double2*>(smem);  // [nb][L] circular windows
    double2* V = Zw + (size_t)nb * L;                // [nb][L] reflectors v_t
    double2* Kap = V + (size_t)nb * L;               // [nb]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int l = blockIdx.x;
    const double2 sig = d.shifts[l];
    const int64_t arow0 = (int64_t)d.k - nb;
    const double* A = d.A;
    auto panel = [&](int i, int c) -> double2 {  // window entry of panel column c, row i
        double2 v = make_double2(A[arow0 + i + (int64_t)(d.c0 + c) * d.lda], 0.0);
        if (i + m == c) v = csub(v, sig);  // lazy -sigma on Ahat's diagonal
        return v;
    };
    // initial windows: columns nb-1 .. nb-1+m (the panel's last column, then
    // the m state columns)
    for (int e = tid; e < nb * L; e += kRqBigThreads) {
        const int i = e / L, s = e - i * L;
        const int col = nb - 1 + ((s - (nb - 1) % L) % L + L) % L;
        Zw[e] = col == nb - 1 ? panel(i, nb - 1)
                              : Z2[(int64_t)l * m * d.LDZ + (int64_t)(col - nb) * d.LDZ + d.r0 + i];
    }
    __syncthreads();

    const int j0 = lane, j1 = lane + 32;  // this lane's reflector-space entries
    __shared__ double pcol[2][128];  // panel column t - 1 of the window rows, staged per step
    for (int t = nb - 1; t >= 0; --t) {
        const double2* row_t = Zw + (size_t)t * L;
        double2* vt = V + (size_t)t * L;
        // stage the entering panel column (contiguous rows: coalesced) while
        // warp 0 builds the reflector
        if (warp > 0 && t >= 1)
            for (int i = tid - 32; i < t; i += kRqBigThreads - 32)
                pcol[t & 1][i] = A[arow0 + i + (int64_t)(d.c0 + t - 1) * d.lda];
        if (warp == 0) {
            // y = conj(row t over columns t..t+m); alpha = y[m]
            double2 y0 = cz(), y1 = cz();
            if (j0 < L) { const double2 z = row_t[(t + j0) % L]; y0 = make_double2(z.x, -z.y); }
            if (j1 < L) { const double2 z = row_t[(t + j1) % L]; y1 = make_double2(z.x, -z.y); }
            double s2 = 0.0;
            if (j0 < m) s2 = fma(y0.x, y0.x, y0.y * y0.y);
            if (j1 < m) s2 = fma(y1.x, y1.x, fma(y1.y, y1.y, s2));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
            const double2 am = row_t[(t + m) % L];
            const double2 alpha = make_double2(am.x, -am.y);
            const bool ident = s2 == 0.0 && alpha.y == 0.0;
            const double nrm2 = ident ? 1.0 : fma(alpha.x, alpha.x, fma(alpha.y, alpha.y, s2));
            const double rn = rsqrt_pos(nrm2);
            const double sg = alpha.x >= 0.0 ? -1.0 : 1.0;
            const double beta = sg * nrm2 * rn, ib = sg * rn;
            const double zx = beta - alpha.x;
            const double f = ib * rcp_pos(fma(zx, zx, alpha.y * alpha.y));
            const double2 kap = ident ? cz() : make_double2(zx * f, -alpha.y * f);
            const double2 vl = make_double2(alpha.x - beta, alpha.y);
            if (j0 < L) vt[j0] = j0 == m ? vl : y0;
            if (j1 < L) vt[j1] = j1 == m ? vl : y1;
            if (lane == 0) Kap[t] = kap;
        }
        __syncthreads();
        const double2 kap = Kap[t];
        const double2 v0 = j0 < L ? vt[j0] : cz(), v1 = j1 < L ? vt[j1] : cz();
        const int s0 = (t + j0) % L, s1 = (t + j1) % L;
        // two rows per iteration: independent reductions interleave
        constexpr int NW = kRqBigThreads / 32;
        for (int i = warp; i < t; i += 2 * NW) {
            const int i2 = i + NW;
            const bool two = i2 < t;
            double2* za = Zw + (size_t)i * L;
            double2* zb = Zw + (size_t)(two ? i2 : i) * L;
            double2 a0 = j0 < L ? za[s0] : cz(), a1 = j1 < L ? za[s1] : cz();
            double2 b0 = j0 < L ? zb[s0] : cz(), b1 = j1 < L ? zb[s1] : cz();
            double2 da = cfma(a1, v1, cmul(a0, v0)), db = cfma(b1, v1, cmul(b0, v0));  // z . v
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                da.x += __shfl_xor_sync(0xffffffffu, da.x, o);
                da.y += __shfl_xor_sync(0xffffffffu, da.y, o);
                db.x += __shfl_xor_sync(0xffffffffu, db.x, o);
                db.y += __shfl_xor_sync(0xffffffffu, db.y, o);
            }
            const double2 ta = cmul(kap, da), tb = cmul(kap, db);
            // z_j -= tw conj(v_j)
            auto upd = [](double2 z, double2 tw, double2 v) {
                return make_double2(z.x - (tw.x * v.x + tw.y * v.y), z.y - (tw.y * v.x - tw.x * v.y));
            };
            a0 = upd(a0, ta, v0);
            a1 = upd(a1, ta, v1);
            b0 = upd(b0, tb, v0);
            b1 = upd(b1, tb, v1);
            if (j0 < L) za[s0] = a0;
            if (j1 < L) za[s1] = a1;
            if (two) {
                if (j0 < L) zb[s0] = b0;
                if (j1 < L) zb[s1] = b1;
            }
            __syncwarp();
            // column t + m retires; panel column t - 1 enters its slot
            if (lane == 0 && t >= 1) {
                double2 pa = make_double2(pcol[t & 1][i], 0.0);
                if (i + m == t - 1) pa = csub(pa, sig);
                za[(t + m) % L] = pa;
                if (two) {
                    double2 pb = make_double2(pcol[t & 1][i2], 0.0);
                    if (i2 + m == t - 1) pb = csub(pb, sig);
                    zb[(t + m) % L] = pb;
                }
            }
        }
        __syncthreads();
    }

    // reverse accumulation: column c of P is H_{nb-1}(...(H_0 e_c)) over rows
    // 0..nb+m-1; step s touches rows s..s+m; one warp per column
    const int nrow = nb + m;
    double2* w = reinterpret_cast<double2*>(smem) +
                 (rq_big_acc_in_win(nb, m) ? 0 : (size_t)2 * nb * L + nb) + (size_t)warp * nrow;
    double2* dstP = Pbuf + (int64_t)l * d.nc * m;                          // P[row * m + c]
    for (int c = warp; c < m; c += kRqBigThreads / 32) {
        for (int r = lane; r < nrow; r += 32) w[r] = make_double2(r == c ? 1.0 : 0.0, 0.0);
        __syncwarp();
        for (int s = 0; s < nb; ++s) {
            const double2* vs = V + (size_t)s * L;
            const double2 kap = Kap[s];
            const double2 v0 = j0 < L ? vs[j0] : cz(), v1 = j1 < L ? vs[j1] : cz();
            double2 w0 = j0 < L ? w[s + j0] : cz(), w1 = j1 < L ? w[s + j1] : cz();
            // dp = v^H w
            double2 dp = make_double2(fma(v0.x, w0.x, v0.y * w0.y), fma(v0.x, w0.y, -v0.y * w0.x));
            dp.x = fma(v1.x, w1.x, fma(v1.y, w1.y, dp.x));
            dp.y = fma(v1.x, w1.y, fma(-v1.y, w1.x, dp.y));
            dp = warp_csum(dp);
            const double2 td = cmul(kap, dp);
            w0 = csub(w0, cmul(v0, td));
            w1 = csub(w1, cmul(v1, td));
            if (j0 < L) w[s + j0] = w0;
            if (j1 < L) w[s + j1] = w1;
            __syncwarp();
        }
        for (int r = lane; r < nrow; r += 32) dstP[(int64_t)r * m + c] = w[r];
        __syncwarp();
    }
}

}  // namespace ssd
