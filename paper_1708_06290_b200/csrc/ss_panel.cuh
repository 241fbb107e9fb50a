// Panel columns of the blocked controller-Hessenberg reduction as ONE
// persistent cooperative kernel per mini-block (reference hessenberg.py:99-146
// _process_panel, mini_boundaries :83-96; kernels.py:74-99
// householder_vector, :156-160 the T column).
//
// The per-column vector work of the reference (right update from the
// panel's completed mini-blocks, left update with the panel's earlier
// reflectors, the Householder vector, the T column) is a chain of small
// dependent reductions over the panel's nk trailing rows.  As separate
// launches it cost six kernels per column (80-210 us per column measured on
// B200: 81% of the reduction at n = 1500, 420 ms of config 3's 2000
// columns).  Here the trailing rows are split into contiguous slices, one per
// CTA (one CTA per SM, co-resident by cooperative launch), and a column
// costs two grid-wide barriers:
//
//   S2(j)  w = T^T (V^T a) from every CTA's partials (summed in CTA order by
//          every CTA: identical values everywhere), a -= V w on the own rows,
//          partial sum of squares below row j;
//   --- grid sync ---
//   S3(j)  Householder scalars (every CTA, same order), v_j = a / (alpha -
//          beta) below row j, V[:, j] = v_j, a finalised; partials of V^T v_j
//          (T column) and -- the next column's S1 fused in -- the right update
//          of column j+1 from the completed mini-blocks (a -= Y V[vrow]^T) and
//          the partials of V^T a_{j+1};
//   --- grid sync ---
//   T[:, j] = -tau T (V^T v_j), T[j, j] = tau: every CTA, in shared memory.
//
// The kernel covers the columns of one mini-block [js, jb); the Y extension
// between mini-blocks is a DMMA GEMM over the trailing matrix (ss_reduce.cu).
// All reductions run in a fixed order (per-warp lane-strided sums, warp
// shuffles, CTA partials summed in CTA order): run-to-run reproducible.
#pragma once

#include <cooperative_groups.h>

namespace ssr {

namespace cg = cooperative_groups;

constexpr int kPT = 256;     // threads per CTA
constexpr int kPBmax = 128;  // widest panel (block_size is capped at 128)
constexpr int kPTC = kPT / 4;  // t's per gathered chunk of cross-CTA partials (64)

struct Pan {
    double* a0;    // panel column j: a0 + j * lda, rows [0, nk)
    int64_t lda;
    int nk, bw, m;
    int yext;      // band panel (1): right updates from Y; B's QR (0)
    int vrow0;     // V row of column j's right update: j + vrow0 (= j - m)
    double* V;     // nk x bw, ld ldv (zero above the diagonal)
    double* Y;     // nk x bw, ld ldv
    int64_t ldv;
    double* T;     // bw x bw, ld ldt: columns < js in, [js, jb) out
    int64_t ldt;
    double* ws;    // scratch: pan_ws_doubles(G)
    // small m (mini-blocks of <= kPYin columns): the Y extension runs inside
    // the kernel (tr = A0[kb:, kb:], ld lda) and one launch covers the panel
    const double* tr;
    int yin;
};
constexpr int kPYin = 4;

__host__ __device__ inline size_t pan_ws_doubles(int G) {
    return (size_t)G * kPBmax * 2 + (size_t)G + 8 + (size_t)G * kPBmax * kPYin;  // + V^T V partials
}
__host__ __device__ inline size_t pan_smem_bytes(int bw, int G, int nown_staged, bool cl = false) {
    return ((size_t)bw * bw + 3 * kPBmax + kPT / 32 + 8 + (cl ? 0 : (size_t)kPTC * G) + (size_t)kPBmax * kPYin +
            (size_t)(kPT / 32) * 32 * kPYin + (cl ? (size_t)kPBmax * (2 + kPYin) + 8 : 0) +
            (size_t)2 * nown_staged * bw) * 8;
}

// The CTA's own rows of V and Y, staged in shared memory when they fit
// (rows [rlo, rhi): element (i, t) at base[(i - off) + t * ld]; global
// otherwise: off = 0, ld = ldv)
struct Own {
    const double* v;
    const double* y;
    int off;
    int64_t ld;
};

// out[t * ostride] = sum over own rows i of V[i, t] x[i], t < nt (warp per t,
// lanes over rows); partials are stored t-major (the G CTAs' values of one t
// contiguous) so the cross-CTA sums below read them coalesced
__device__ __forceinline__ void own_vdots(const Own& o, int rlo, int rhi, const double* x, int nt, double* out,
                                          int ostride) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int t = warp; t < nt; t += kPT / 32) {
        const double* vc = o.v + (int64_t)t * o.ld - o.off;
        double s = 0.0;
        for (int i = rlo + lane; i < rhi; i += 32) s = fma(vc[i], x[i], s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) out[(size_t)t * ostride] = s;
    }
}

// d[t] = sum over CTAs c of part[t * G + c], t < nt.  The nt x G partials
// (contiguous) are gathered into shared memory with cp.async -- every load
// in flight at once: one L2 round trip instead of one per t (the per-t warp
// loop measured ~1 us per t, 60% of the kernel) -- then four threads per t
// sum strided quarters and combine them with a fixed shuffle tree
// (deterministic: the same order in every CTA and run).
__device__ __forceinline__ void cta_sums(const double* part, int G, int nt, double* d, double* buf) {
    const int tid = threadIdx.x;
    for (int t0 = 0; t0 < nt; t0 += kPTC) {
        const int nc = min(kPTC, nt - t0);
        const double* src = part + (size_t)t0 * G;
        for (int e = tid; e < nc * G; e += kPT) cpa8(buf + e, src + e, true);
        cpa_commit();
        cpa_wait<0>();
        __syncthreads();
        const int t = tid >> 2, q = tid & 3;
        double s = 0.0;
        if (t < nc)
            for (int c = q; c < G; c += 4) s += buf[t * G + c];
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        if (q == 0 && t < nc) d[t0 + t] = s;
        __syncthreads();  // buf is reused by the next chunk / call
    }
}

// S1(j): right update of column j from the completed mini-blocks (Y columns
// t < jr), own rows; then the partials of V^T a_j (t < j)
__device__ __forceinline__ void s1_right(const Pan& p, const Own& o, double* vrs, int j, int js, int rlo, int rhi,
                                         double* ppart_c, int pstride) {
    double* a = p.a0 + (int64_t)j * p.lda;
    const int jr = p.yext ? min(js, max(j - p.m + 1, 0)) : 0;
    if (jr > 0) {
        // V row j - m (another CTA's row) into shared memory once
        const double* vr = p.V + (j + p.vrow0);
        for (int t = threadIdx.x; t < jr; t += kPT) vrs[t] = vr[(int64_t)t * p.ldv];
        __syncthreads();
        for (int i = rlo + (int)threadIdx.x; i < rhi; i += kPT) {
            const double* yr = o.y + (i - o.off);
            double v0 = a[i], v1 = 0.0;
            int t = 0;
            for (; t + 1 < jr; t += 2) {
                v0 = fma(-yr[(int64_t)t * o.ld], vrs[t], v0);
                v1 = fma(-yr[(int64_t)(t + 1) * o.ld], vrs[t + 1], v1);
            }
            if (t < jr) v0 = fma(-yr[(int64_t)t * o.ld], vrs[t], v0);
            a[i] = v0 + v1;
        }
        __syncthreads();
    }
    own_vdots(o, rlo, rhi, a, j, ppart_c, pstride);
}

// Cross-CTA communication of the panel kernel.  GRID: every SM (cooperative
// launch), partials in global scratch ([t][G]) gathered with cp.async, grid
// barriers (1.2 us each on B200).  CLUSTER: one cluster of kPCl CTAs for
// small panels (nk <= kPCl kPClRows): partials in each CTA's shared memory,
// summed over the cluster through distributed shared memory in rank order,
// hardware cluster barriers (0.24 us).  Both sum in a fixed order: every CTA
// gets identical values and runs are reproducible.
constexpr int kPCl = 16;        // CTAs in the cluster variant
constexpr int kPClRows = 128;   // rows per CTA it covers (own V / Y rows staged in shared memory)

template <bool CL>
struct PanComm {
    int G, cta;
    double* gpart;  // GRID: global partials base of this array ([t][G]); CLUSTER: this CTA's smem array
    double* pbuf;   // GRID: gather buffer (smem)
    __device__ __forceinline__ void sync() const {
        if constexpr (CL) cg::this_cluster().sync();
        else cg::this_grid().sync();
    }
    // where this CTA writes partial t: out[t * stride()]
    __device__ __forceinline__ double* out() const { return CL ? gpart : gpart + cta; }
    __device__ __forceinline__ int stride() const { return CL ? 1 : G; }
    // d[t] = sum over CTAs of partial t (after sync())
    __device__ __forceinline__ void sums(int nt, double* d) const {
        if constexpr (CL) {
            cg::cluster_group cl = cg::this_cluster();
            for (int t = threadIdx.x; t < nt; t += blockDim.x) {
                double s = 0.0;
                for (int r = 0; r < G; ++r) s += cl.map_shared_rank(gpart, r)[t];
                d[t] = s;
            }
        } else {
            cta_sums(gpart, G, nt, d, pbuf);
        }
    }
};

// Y[:, ms:me] = (A0 V[:, ms:me] - Y[:, :ms] (V[:, :ms]^T V[:, ms:me])) T[ms:me, ms:me]
// for the own rows (hessenberg.py:83-96 mini_boundaries; me - ms <= kPYin):
// V^T V across CTAs (partials, one grid barrier, gathered sums), A0 V with
// the warps splitting the trailing columns and lanes on rows (a fixed-order
// combine in shared memory), the rest row-local.
template <bool CL>
__device__ void yext_inline(const Pan& p, const Own& o, int ms, int me, int rlo, int rhi, const PanComm<CL>& vc,
                            const double* Ts, int bw, double* vtv, double* avs) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int cw = me - ms, ne = ms * cw;
    double* vpo = vc.out();
    const int vst = vc.stride();
    // (1) V^T V partials: entry e = t + u ms (t < ms, u < cw), stored [e][G]
    for (int e = warp; e < ne; e += kPT / 32) {
        const int t = e % ms, u = e / ms;
        const double* vt = o.v + (int64_t)t * o.ld - o.off;
        const double* vu = o.v + (int64_t)(ms + u) * o.ld - o.off;
        double s = 0.0;
        for (int i = rlo + lane; i < rhi; i += 32) s = fma(vt[i], vu[i], s);
#pragma unroll
        for (int q = 16; q > 0; q >>= 1) s += __shfl_xor_sync(0xffffffffu, s, q);
        if (lane == 0) vpo[(size_t)e * vst] = s;
    }
    // (2) A0 V for the own rows, 8 rows at a time: every thread takes trailing
    // columns c = tid, tid + 256, ... (the 8 rows of a column are contiguous:
    // two sectors, and every lane's loads are independent -- the CTA's slice
    // of A0 streams at L2 bandwidth instead of one latency per column), then
    // a fixed shuffle tree over the lanes and a fixed-order sum over warps
    const int ncol = p.nk - ms;
    for (int r0 = rlo; r0 < rhi; r0 += 8) {
        const int nr = min(8, rhi - r0);
        double acc[8][kPYin];
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int u = 0; u < kPYin; ++u) acc[r][u] = 0.0;
        for (int c = tid; c < ncol; c += kPT) {
            double vv[kPYin];
#pragma unroll
            for (int u = 0; u < kPYin; ++u) vv[u] = u < cw ? p.V[(ms + c) + (int64_t)(ms + u) * p.ldv] : 0.0;
            const double* col = p.tr + r0 + (int64_t)(ms + c) * p.lda;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                if (r < nr) {
                    const double av = col[r];
#pragma unroll
                    for (int u = 0; u < kPYin; ++u) acc[r][u] = fma(av, vv[u], acc[r][u]);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int u = 0; u < kPYin; ++u) {
                double v = acc[r][u];
#pragma unroll
                for (int q = 16; q > 0; q >>= 1) v += __shfl_xor_sync(0xffffffffu, v, q);
                if (lane == 0) avs[(warp * 8 + r) * kPYin + u] = v;
            }
        __syncthreads();
        if (tid < nr * cw) {
            const int r = tid / cw, u = tid - (tid / cw) * cw;
            double v = 0.0;
            for (int w = 0; w < kPT / 32; ++w) v += avs[(w * 8 + r) * kPYin + u];
            p.Y[r0 + r + (int64_t)(ms + u) * p.ldv] = v;  // A0 V, before the corrections
        }
        __syncthreads();
    }
    vc.sync();
    if (ne > 0) {
        vc.sums(ne, vtv);
        __syncthreads();
    }
    // (3) own rows: (A0 V - Y VtV) T, written to Y (and the staged copy)
    for (int i = rlo + tid; i < rhi; i += kPT) {
        double z[kPYin];
#pragma unroll
        for (int u = 0; u < kPYin; ++u) {
            z[u] = 0.0;
            if (u < cw) {
                double v = p.Y[i + (int64_t)(ms + u) * p.ldv];
                for (int t = 0; t < ms; ++t) v = fma(-o.y[(i - o.off) + (int64_t)t * o.ld], vtv[t + u * ms], v);
                z[u] = v;
            }
        }
#pragma unroll
        for (int u = 0; u < kPYin; ++u) {
            if (u < cw) {
                double y = 0.0;
#pragma unroll
                for (int k = 0; k < kPYin; ++k)
                    if (k <= u) y = fma(z[k], Ts[(ms + k) + (ms + u) * bw], y);
                p.Y[i + (int64_t)(ms + u) * p.ldv] = y;
                if (o.y != p.Y) const_cast<double*>(o.y)[(i - o.off) + (int64_t)(ms + u) * o.ld] = y;
            }
        }
    }
    __syncthreads();
}

template <bool CL>
__global__ void __launch_bounds__(kPT, 1) k_panel(Pan p, int js, int jb, int stage) {
    extern __shared__ double sm[];
    const int bw = p.bw, nk = p.nk;
    double* Ts = sm;               // bw x bw, col-major (ld bw)
    double* w = Ts + bw * bw;      // [kPBmax]
    double* d = w + kPBmax;        // [kPBmax]
    double* red = d + kPBmax;      // [kPT / 32]
    double* sc = red + kPT / 32;   // [8] tau, beta, scale
    double* vrs = sc + 8;          // [kPBmax] V row of the right update
    double* pbuf = vrs + kPBmax;   // [kPTC * G] cross-CTA partials (cta_sums)
    double* vtv = pbuf + (CL ? 0 : (size_t)kPTC * gridDim.x);  // [kPBmax * kPYin] V^T V of the Y extension
    double* avs = vtv + kPBmax * kPYin;             // [8 warps][32 rows][kPYin] A0 V partials
    const int G = gridDim.x, tid = threadIdx.x, lane = tid & 31;
    const int cta = CL ? (int)cg::this_cluster().block_rank() : blockIdx.x;
    const int rlo = (int)((int64_t)nk * cta / G), rhi = (int)((int64_t)nk * (cta + 1) / G);
    const int nown = rhi - rlo;
    Own o{p.V, p.Y, 0, p.ldv};
    double* Vs = nullptr;
    if (stage) {
        // own rows of V (columns < jb; column j written here as it is formed)
        // and Y (columns < js, read-only in this kernel)
        Vs = avs + (kPT / 32) * 32 * kPYin + (CL ? kPBmax * (2 + kPYin) + 8 : 0);
        double* Ys = Vs + (size_t)nown * bw;
        for (int e = tid; e < nown * jb; e += kPT) {
            const int r = e % nown, t = e / nown;
            Vs[e] = t < js ? p.V[rlo + r + (int64_t)t * p.ldv] : 0.0;
        }
        if (p.yext)
            for (int e = tid; e < nown * js; e += kPT) {
                const int r = e % nown, t = e / nown;
                Ys[e] = p.Y[rlo + r + (int64_t)t * p.ldv];
            }
        o = Own{Vs, Ys, rlo, nown};
    }
    // partial sums: GRID in global scratch ([t][G]), CLUSTER in shared memory
    double* gp = p.ws;
    double* scal = gp + (size_t)G * kPBmax * 2 + G;  // [8]: alpha (global in both variants)
    double* cp = avs + (kPT / 32) * 32 * kPYin;      // CLUSTER: [kPBmax] p, [kPBmax] q, [8] s, [kPBmax kPYin] v
    const PanComm<CL> pc{G, cta, CL ? cp : gp, pbuf};
    const PanComm<CL> qc{G, cta, CL ? cp + kPBmax : gp + (size_t)G * kPBmax, pbuf};
    const PanComm<CL> sc_{G, cta, CL ? cp + 2 * kPBmax : gp + (size_t)G * kPBmax * 2, pbuf};
    const PanComm<CL> vc{G, cta, CL ? cp + 2 * kPBmax + 8 : scal + 8, pbuf};
    // T columns of the earlier mini-blocks (upper triangle)
    for (int e = tid; e < bw * bw; e += kPT) {
        const int r = e % bw, c = e / bw;
        Ts[e] = (c < js && r <= c) ? p.T[r + (int64_t)c * p.ldt] : 0.0;
    }
    __syncthreads();
    int ms = js;  // first column of the current mini-block
    s1_right(p, o, vrs, js, ms, rlo, rhi, pc.out(), pc.stride());
    pc.sync();
    for (int j = js; j < jb; ++j) {
        double* a = p.a0 + (int64_t)j * p.lda;
        // ---- S2: w = T^T (sum of partials); a -= V w; squares below row j ----
        pc.sums(j, d);
        __syncthreads();
        for (int t = tid; t < j; t += kPT) {
            double s = 0.0;
            for (int k = 0; k <= t; ++k) s = fma(Ts[k + t * bw], d[k], s);  // (T^T d)_t
            w[t] = s;
        }
        __syncthreads();
        double sq = 0.0;
        for (int i = rlo + tid; i < rhi; i += kPT) {
            const double* vr = o.v + (i - o.off);
            double v0 = a[i], v1 = 0.0;
            int t = 0;
            for (; t + 1 < j; t += 2) {
                v0 = fma(-vr[(int64_t)t * o.ld], w[t], v0);
                v1 = fma(-vr[(int64_t)(t + 1) * o.ld], w[t + 1], v1);
            }
            if (t < j) v0 = fma(-vr[(int64_t)t * o.ld], w[t], v0);
            const double v = v0 + v1;
            a[i] = v;
            if (i > j) sq = fma(v, v, sq);
            if (i == j) scal[0] = v;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) red[tid >> 5] = sq;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int q = 0; q < kPT / 32; ++q) t += red[q];
            sc_.out()[0] = t;
        }
        sc_.sync();
        // ---- S3: Householder scalars (householder_vector, kernels.py:74-99) ----
        sc_.sums(1, red);
        __syncthreads();
        if (tid == 0) {
            const double sigma = red[0];
            const double alpha = scal[0];
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
            sc[0] = tau;
            sc[1] = beta;
            sc[2] = scale;
        }
        __syncthreads();
        const double tau = sc[0], beta = sc[1], scale = sc[2];
        double* vj = p.V + (int64_t)j * p.ldv;
        for (int i = rlo + tid; i < rhi; i += kPT) {
            double v;
            if (i < j) v = 0.0;
            else if (i == j) v = 1.0;
            else v = tau == 0.0 ? 0.0 : a[i] * scale;
            vj[i] = v;
            if (Vs) Vs[(i - rlo) + (size_t)j * nown] = v;
            if (i == j) a[i] = beta;
            else if (i > j) a[i] = 0.0;
        }
        __syncthreads();
        own_vdots(o, rlo, rhi, vj, j, qc.out(), qc.stride());
        // in-kernel Y extension: a mini-block ends at this column
        const bool ybnd = p.yin && ((j + 1 - ms) == p.m || j + 1 == jb);
        if (j + 1 < jb && !ybnd) s1_right(p, o, vrs, j + 1, ms, rlo, rhi, pc.out(), pc.stride());
        qc.sync();
        // ---- T column (kernels.py:156-160; every CTA, same order) ----
        qc.sums(j, d);
        __syncthreads();
        for (int r = tid; r < j; r += kPT) {
            double s = 0.0;
            for (int k = r; k < j; ++k) s = fma(Ts[r + k * bw], d[k], s);
            Ts[r + j * bw] = -tau * s;
        }
        if (tid == 0) Ts[j + j * bw] = tau;
        __syncthreads();
        if (ybnd) {
            yext_inline<CL>(p, o, ms, j + 1, rlo, rhi, vc, Ts, bw, vtv, avs);
            ms = j + 1;
            if (j + 1 < jb) {
                __syncthreads();
                s1_right(p, o, vrs, j + 1, ms, rlo, rhi, pc.out(), pc.stride());
                pc.sync();
            }
        }
    }
    if (cta == 0)
        for (int e = tid; e < bw * (jb - js); e += kPT) {
            const int r = e % bw, c = js + e / bw;
            p.T[r + (int64_t)c * p.ldt] = r <= c ? Ts[r + c * bw] : 0.0;
        }
    if constexpr (CL) cg::this_cluster().sync();  // no CTA leaves while its shared memory may be read
}

}  // namespace ssr
