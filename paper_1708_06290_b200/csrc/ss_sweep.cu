// Batched shifted solves on controller-Hessenberg data, sm_100a.
//
// Reference path (solvers.py:130-313): for every shift sigma_l the stacked
// matrix [top; Ahat - sigma_l I] is RQ-factorised bottom-up by a sliding
// window; only the m "active" transformed columns Z2 are kept per shift and
// the nb shift-independent panel columns Z1 of Ahat are shared by all
// shifts.  Per window step (solvers.py:165-200):
//     block  = [Z1 | Z2_l] rows r0..r0+nb  (lazy -sigma on Ahat's diagonal)
//     P_l    = first m columns of the block's scheduled Givens RQ factor
//     Z2_l[0:r0] <- Z2_l[0:r0] P_l[nb:] + Z1[0:r0] P_l[:nb] - sigma_l e P_l[:mnb]
// then the m x m head is reduced and back-substituted (solvers.py:204-231)
// and G_l = -Chat X (or x_l = Q X for the reduced solve).
//
// B200 mapping (per-shift window state in HBM/L2, updated in place):
//   k_seed      one pass writing Z2 for all shifts of a batch
//   two-level sweep (m in 4..8, 10, 20), per outer block of 128 columns:
//     k_block   one warp per shift: the four 32-row inner windows (Householder
//               chain, reverse accumulation, in-block row passes) -> the
//               composite W (ss_block.cuh)
//     k_far     persistent, warp-specialised (TMA bulk copies + mbarrier ring)
//               far-row update from W in two 64-column passes (ss_far.cuh)
//   one-level sweep (other m), per window of nb columns:
//     k_rq_house / k_rq   block RQ (row Householder; the reference's scheduled
//               Givens batch for m + 1 > 32) -> P_l
//     k_far (m = 1: ten shifts per unit; m = 20) / k_update_ws / k_update
//               the window update of rows [0, r0)
//   k_head      one CTA per shift: m x m head RQ fused with the triangular
//               solve and the -Chat X (or Q X) epilogue; only G / x leave
//               the device.
// ss_tf_eval_stream additionally streams Ahat from pinned host memory in the
// order the sweep consumes its columns (copy stream + one event per chunk).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ss_device.cuh"
#include "ss_internal.h"
#include "ss_rq_house.cuh"
#include "ss_update.cuh"
#include "ss_update_ws.cuh"
#include "ss_block.cuh"
#include "ss_rq_m1.cuh"
#include "ss_rq_big.cuh"
#include "ss_far4.cuh"
#include "ss_far.cuh"
#include "ss_fark.cuh"
#ifdef SS_FARK_DMMA
#include "ss_farkd.cuh"  // comparison builds only (see kFarkDmma)
#endif

using namespace ssd;

namespace {


struct Dims {
    int n, m, ptop;
    int ident_top;  // 1: identity top of height n (reduced solve)
    const double* A;
    int64_t lda;
    const double* T;  // dense top rows (Chat), ptop x n
    int64_t ldt;
    const double2* shifts;  // batch-local
    int sb;                 // shifts in this batch
    int64_t LDZ;            // leading dim of one Z2 column
};

__device__ __forceinline__ double panel_val(const Dims& d, int i, int col) {
    if (i < d.ptop) {
        if (d.ident_top) return i == col ? 1.0 : 0.0;
        return d.T[i + (int64_t)col * d.ldt];
    }
    return d.A[(i - d.ptop) + (int64_t)col * d.lda];
}

// ---------------------------------------------------------------------------
// ||A||_F^2 and trace(A), deterministic two-pass reduction (solvers.py:104-110)
// ---------------------------------------------------------------------------
__global__ void k_fro2_trace_part(int n, const double* __restrict__ A, int64_t lda,
                                  double* __restrict__ part) {
    __shared__ double sf[32], st[32];
    double f = 0.0, t = 0.0;
    for (int j = blockIdx.x; j < n; j += gridDim.x) {
        const double* col = A + (int64_t)j * lda;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            double v = col[i];
            f = fma(v, v, f);
        }
        if (threadIdx.x == 0) t += col[j];
    }
    for (int o = 16; o > 0; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
    if ((threadIdx.x & 31) == 0) sf[threadIdx.x >> 5] = f;
    if (threadIdx.x == 0) st[0] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double ff = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) ff += sf[w];
        part[2 * blockIdx.x] = ff;
        part[2 * blockIdx.x + 1] = st[0];
    }
}

__global__ void k_fro2_trace_final(int nparts, const double* __restrict__ part,
                                   double* __restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double f = 0.0, t = 0.0;
        for (int b = 0; b < nparts; ++b) {
            f += part[2 * b];
            t += part[2 * b + 1];
        }
        out[0] = f;
        out[1] = t;
    }
}

// ---------------------------------------------------------------------------
// seed (solvers.py:157-163): Z2_l = last m columns of [top; A], -sigma_l on
// A's diagonal.  The window state is updated in place afterwards.
// ---------------------------------------------------------------------------
__global__ void k_seed(Dims d, double2* __restrict__ Za) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int l = blockIdx.y;
    if (i >= d.LDZ) return;
    const double2 sig = d.shifts[l];
    for (int c = 0; c < d.m; ++c) {
        const int col = d.n - d.m + c;
        double2 v = cz();
        if (i < d.ptop + d.n) {
            v.x = panel_val(d, i, col);
            if (i == d.ptop + col) {
                v.x -= sig.x;
                v.y -= sig.y;
            }
        }
        const int64_t idx = ((int64_t)l * d.m + c) * d.LDZ + i;
        Za[idx] = v;
    }
}

// ---------------------------------------------------------------------------
// per-step block RQ: one CTA per shift (solvers.py:170-184, batched.py:64-122)
// ---------------------------------------------------------------------------
struct Step {
    int k, nb, mnb, r0, c0, nc;
    int lmp;  // log2 of the smallest power of two >= m
    int steps, rots;
    const uint32_t* rot;
    const int32_t* joff;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

__host__ __device__ inline size_t rq_smem_bytes(int nb, int m, int steps, int rots) {
    const int nc = nb + m;
    size_t b = 0;
    b += align16((size_t)rots * 4);           // rot
    b += align16((size_t)(steps + 1) * 4);    // joff
    const int zw = pk_size(nb, m) > nc * m ? pk_size(nb, m) : nc * m;
    b += (size_t)zw * 16;                     // Zb / W
    return b;
}

template <int SLOTS>
__global__ void k_rq(Dims d, Step st, const double2* __restrict__ Z2, double2* __restrict__ Pbuf) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int l = blockIdx.x;
    const int nb = st.nb, m = d.m, nc = st.nc;
    size_t off = 0;
    uint32_t* rot = (uint32_t*)(smem + off);
    off += align16((size_t)st.rots * 4);
    int* joff = (int*)(smem + off);
    off += align16((size_t)(st.steps + 1) * 4);
    double2* Zb = (double2*)(smem + off);

    for (int u = threadIdx.x; u < st.rots; u += blockDim.x) rot[u] = st.rot[u];
    for (int u = threadIdx.x; u <= st.steps; u += blockDim.x) joff[u] = st.joff[u];

    // pack the block (solvers.py:174-181); block row t is A-row k-nb+t
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const double2 sig = d.shifts[l];
    const int arow0 = st.k - nb;
    for (int col = warp; col < nc; col += nw) {
        double2* dst = Zb + pk_off(col, nb);
        const int hgt = pk_height(col, nb);
        if (col < nb) {
            const double* src = d.A + arow0 + (int64_t)(st.c0 + col) * d.lda;
            for (int t = lane; t < hgt; t += 32) {
                double2 v = make_double2(src[t], 0.0);
                if (t + m == col) {  // A's main diagonal inside the panel
                    v.x -= sig.x;
                    v.y -= sig.y;
                }
                dst[t] = v;
            }
        } else {
            const double2* src = Z2 + ((int64_t)l * m + (col - nb)) * d.LDZ + st.r0;
            for (int t = lane; t < hgt; t += 32) dst[t] = src[t];
        }
    }
    __syncthreads();
    block_rq_fused<SLOTS>(Zb, nb, nc, m, rot, joff, st.steps);  // W (j-major) over the block
    double2* dstP = Pbuf + (int64_t)l * nc * m;
    for (int u = threadIdx.x; u < nc * m; u += blockDim.x) dstP[u] = Zb[u];
}

// ---------------------------------------------------------------------------
// head (solvers.py:204-231 + :262-268 / :303-310): one CTA per shift.
// Warp 0 reduces the m x m head with the reference's rotation order,
// accumulating the rotations in Qh (m x m) instead of rotating every top
// row; the fused back-substitution gives X; then the epilogue applies
// top rows x (Qh X) with all warps.
// ---------------------------------------------------------------------------
struct HeadOut {
    int mode;          // 0 transfer function, 1 reduced solve
    const double* B;   // Bhat, read [0:m, 0:m]
    int64_t ldb;
    const double2* bd; // reduced: b_dirs (batch-local), m x sb
    int64_t ldbd;
    double rtol;
    const double* scal;  // [fro2, trace]
    double2* out;        // tf: G (batch-local, column l*m); reduced: X (batch-local)
    int64_t ldo;
    int32_t* fail;       // batch-local
    double2* ybuf;       // deferred reduced solve: y = Qh X (m per shift) for k_expand
    int l0;              // first batch-local shift of this launch
    double2* gscr;       // non-null: Hh / Qh / X in global scratch (3 m^2 per CTA; wide m)
};

__global__ void k_head(Dims d, HeadOut h, const double2* __restrict__ Z2) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int m = d.m, l = h.l0 + blockIdx.x;
    const int q = h.mode == 0 ? m : 1;
    double2* Hh = h.gscr ? h.gscr + (int64_t)blockIdx.x * 3 * m * m : (double2*)smem;  // m x m, col-major
    double2* Qh = Hh + m * m;      // m x m
    double2* X = Qh + m * m;       // m x q
    __shared__ int s_fail;
    const double2* zl = Z2 + (int64_t)l * m * d.LDZ;
    for (int u = threadIdx.x; u < m * m; u += blockDim.x) {
        const int c = u / m, r = u - c * m;
        Hh[u] = zl[(int64_t)c * d.LDZ + d.ptop + r];
        Qh[u] = make_double2(r == c ? 1.0 : 0.0, 0.0);
    }
    // right-hand side: Bhat[0:m,0:m] (tf) or Bhat[0:m,0:m] b_l (reduced)
    for (int u = threadIdx.x; u < m * q; u += blockDim.x) {
        const int c = u / m, r = u - c * m;
        double2 v;
        if (h.mode == 0) {
            v = make_double2(h.B[r + (int64_t)c * h.ldb], 0.0);
        } else {
            v = cz();
            for (int j = 0; j < m; ++j)
                v = rfma(h.B[r + (int64_t)j * h.ldb], h.bd[j + (int64_t)l * h.ldbd], v);
        }
        X[u] = v;  // holds rhs until row r is solved
    }
    if (threadIdx.x == 0) s_fail = -1;
    __syncthreads();

    const double2 sig = d.shifts[l];
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const double fro2 = h.scal[0], tr = h.scal[1];
        const double sc2 = fro2 - 2.0 * (sig.x * tr) + (sig.x * sig.x + sig.y * sig.y) * d.n;
        const double tol = h.rtol * sqrt(sc2 > 0.0 ? sc2 : 0.0);
        int fail = -1;
        for (int i = m - 1; i >= 0; --i) {
            for (int jj = 0; jj < i; ++jj) {
                const double2 a = Hh[i + i * m], b = Hh[i + jj * m];
                double c;
                double2 s, rho;
                givens_fast(a, b, c, s, rho);
                for (int r = lane; r < m; r += 32) {
                    if (r != i) {
                        double2 hh = Hh[r + i * m], tt = Hh[r + jj * m];
                        rot_apply(c, s, hh, tt);
                        Hh[r + i * m] = hh;
                        Hh[r + jj * m] = tt;
                    }
                    double2 qa = Qh[r + i * m], qb = Qh[r + jj * m];
                    rot_apply(c, s, qa, qb);
                    Qh[r + i * m] = qa;
                    Qh[r + jj * m] = qb;
                }
                __syncwarp();
                if (lane == 0) {
                    Hh[i + jj * m] = cz();
                    Hh[i + i * m] = rho;
                }
                __syncwarp();
            }
            const double2 piv = Hh[i + i * m];
            if (cabsd(piv) <= tol) {
                fail = i;
                break;
            }
            for (int c = lane; c < q; c += 32) {
                double2 acc = cz();
                for (int j = i + 1; j < m; ++j) acc = cfma(Hh[i + j * m], X[j + c * m], acc);
                X[i + c * m] = cdiv(csub(X[i + c * m], acc), piv);
            }
            __syncwarp();
        }
        if (lane == 0) s_fail = fail;
    }
    __syncthreads();
    const int fail = s_fail;
    if (fail >= 0) {
        const double qn = __longlong_as_double(0x7ff8000000000000ULL);
        if (h.mode == 0) {
            for (int u = threadIdx.x; u < d.ptop * m; u += blockDim.x) {
                const int c = u / d.ptop, i = u - c * d.ptop;
                h.out[i + ((int64_t)l * m + c) * h.ldo] = make_double2(qn, qn);
            }
        } else if (!h.ybuf) {
            for (int i = threadIdx.x; i < d.n; i += blockDim.x)
                h.out[i + (int64_t)l * h.ldo] = make_double2(qn, qn);
        }
        if (threadIdx.x == 0) h.fail[l] = fail;
        return;
    }
    // V = Qh X  (m x q), stored over Hh
    for (int u = threadIdx.x; u < m * q; u += blockDim.x) {
        const int c = u / m, r = u - c * m;
        double2 acc = cz();
        for (int j = 0; j < m; ++j) acc = cfma(Qh[r + j * m], X[j + c * m], acc);
        Hh[u] = acc;
    }
    __syncthreads();
    const double2* V = Hh;
    if (h.mode == 0) {
        // G_l = -(top rows) V   (p x m)
        for (int u = threadIdx.x; u < d.ptop * m; u += blockDim.x) {
            const int c = u / d.ptop, i = u - c * d.ptop;
            double2 acc = cz();
            for (int j = 0; j < m; ++j) acc = cfma(zl[(int64_t)j * d.LDZ + i], V[j + c * m], acc);
            h.out[i + ((int64_t)l * m + c) * h.ldo] = make_double2(-acc.x, -acc.y);
        }
    } else if (h.ybuf) {
        for (int r = threadIdx.x; r < m; r += blockDim.x) h.ybuf[(int64_t)l * m + r] = V[r];
    } else {
        for (int i = threadIdx.x; i < d.n; i += blockDim.x) {
            double2 acc = cz();
            for (int j = 0; j < m; ++j) acc = cfma(zl[(int64_t)j * d.LDZ + i], V[j], acc);
            h.out[i + (int64_t)l * h.ldo] = acc;
        }
    }
    if (threadIdx.x == 0) h.fail[l] = -1;
}

// ---------------------------------------------------------------------------
// Deferred identity top of the reduced solve (solvers.py:274-313).  The
// reference sweeps [I; Ahat - sigma I] and reads x = Z2[:n] y; the identity
// rows only ever receive  T <- T W22_c + E_c W12_c  (composite c over panel
// columns [c0_c, c0_c + K_c)), so with T_0 = the seed's identity columns
//   x = sum_c E_c W12_c (W22_{c+1} ... W22_C y) + E_seed (W22_1 ... W22_C y),
// one backward pass over the kept composites per shift (O(n m) instead of
// sweeping n identity rows through every far update).  One CTA per shift.
// ---------------------------------------------------------------------------
struct ExpandArgs {
    int n, m, group, ncomp;
    const double2* Xh;    // per shift: n x m (row = panel column), stride xh_stride
    int64_t xh_stride;
    const double2* W22h;  // per shift: ncomp x m x m (j-major), stride w22h_stride
    int64_t w22h_stride;
    const double2* Y;     // per shift: m
    const int32_t* fail;
    double2* X;           // n x sb, ldx
    int64_t ldx;
};

__global__ void __launch_bounds__(256) k_expand(ExpandArgs e) {
    extern __shared__ __align__(16) unsigned char smem[];
    double2* v = reinterpret_cast<double2*>(smem);  // [2][m]
    int* cs = reinterpret_cast<int*>(v + 2 * e.m);  // [ncomp][2]: (c0, K)
    const int l = blockIdx.x, m = e.m;
    double2* x = e.X + (int64_t)l * e.ldx;
    if (e.fail[l] >= 0) {
        const double qn = __longlong_as_double(0x7ff8000000000000ULL);
        for (int i = threadIdx.x; i < e.n; i += blockDim.x) x[i] = make_double2(qn, qn);
        return;
    }
    if (threadIdx.x == 0) {
        // the composites in sweep order, as enqueue_part's group loop forms them
        int c = 0;
        for (int ko = e.n; ko >= m + 1;) {
            const int NB1 = min(kBlkNB, ko - m);
            const int g = 1 + min(e.group - 1, (ko - NB1 - m) / kBlkNB);
            const int K = (g - 1) * kBlkNB + NB1;
            cs[2 * c] = ko - m - K;
            cs[2 * c + 1] = K;
            ++c;
            ko -= K;
        }
    }
    for (int t = threadIdx.x; t < m; t += blockDim.x) v[t] = e.Y[(int64_t)l * m + t];
    __syncthreads();
    const double2* xh = e.Xh + (int64_t)l * e.xh_stride;
    const double2* w22 = e.W22h + (int64_t)l * e.w22h_stride;
    int cur = 0;
    for (int c = e.ncomp - 1; c >= 0; --c) {
        const double2* vc = v + cur * m;
        const int c0 = cs[2 * c], K = cs[2 * c + 1];
        for (int j = threadIdx.x; j < K; j += blockDim.x) {
            const double2* wr = xh + (int64_t)(c0 + j) * m;
            double2 acc = cz();
            for (int t = 0; t < m; ++t) acc = cfma(wr[t], vc[t], acc);
            x[c0 + j] = acc;
        }
        // v <- W22_c v
        const double2* wc = w22 + (int64_t)c * m * m;
        double2* vn = v + (cur ^ 1) * m;
        for (int j = threadIdx.x; j < m; j += blockDim.x) {
            double2 acc = cz();
            for (int t = 0; t < m; ++t) acc = cfma(wc[(int64_t)j * m + t], vc[t], acc);
            vn[j] = acc;
        }
        cur ^= 1;
        __syncthreads();
    }
    for (int t = threadIdx.x; t < m; t += blockDim.x) x[e.n - m + t] = v[cur * m + t];
}

// ---------------------------------------------------------------------------
// host driver
// ---------------------------------------------------------------------------
// Opt in to the largest dynamic shared memory the kernel can take
// (the per-block opt-in limit minus its static shared memory).
template <typename F>
cudaError_t allow_max_smem(ss_handle* h, F* fn) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, fn);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(h->smem_optin - fa.sharedSizeBytes));
}

// Register tile of the update kernel: lane = (row group, column group q < G),
// R = 2G rows x C columns; a warp covers 64 rows x G*C columns.
struct UpdTile {
    int G = 1, C = 1;
    bool exact = true;
};

UpdTile pick_tile(int m) {
    UpdTile t;
    if (m % 10 == 0) { t.G = 2; t.C = 5; }
    else if (m % 8 == 0) { t.G = 2; t.C = 4; }
    else if (m <= 8) { t.G = 1; t.C = m; }
    else if (m % 5 == 0) { t.G = 1; t.C = 5; }
    else { t.G = 2; t.C = 5; t.exact = false; }
    return t;
}

template <int G, int C, bool EXACT>
int launch_update_t(ss_handle* h, dim3 grid, int threads, size_t smem, cudaStream_t st,
                    const UpdDims& u, const double2* zin, double2* zout, const double2* pbuf) {
    if (threads > 256 || smem > h->smem_optin) {
        // K-split with several column blocks per shift (m > 31): up to 10 warps
        static ss::DevMask configured_w;  // devices configured
        if (!configured_w.has(h)) {
            SS_CUDA_TRY(h, allow_max_smem(h, k_update<G, C, EXACT, 320>));
            SS_CUDA_TRY(h, allow_max_smem(h, k_update<G, C, EXACT, 320, true>));
            configured_w.set(h);
        }
        if (smem > h->smem_optin)  // staged P does not fit: read it from global memory
            k_update<G, C, EXACT, 320, true><<<grid, threads, upd_smem_bytes(u.nb, u.m, u.S, true), st>>>(
                u, zin, zout, pbuf);
        else
            k_update<G, C, EXACT, 320><<<grid, threads, smem, st>>>(u, zin, zout, pbuf);
        SS_LAUNCH_CHECK(h);
        return SS_OK;
    }
    static ss::DevMask configured;  // devices configured
    if (!configured.has(h)) {
        SS_CUDA_TRY(h, allow_max_smem(h, k_update<G, C, EXACT>));
        configured.set(h);
    }
    k_update<G, C, EXACT><<<grid, threads, smem, st>>>(u, zin, zout, pbuf);
    SS_LAUNCH_CHECK(h);
    return SS_OK;
}

template <int G, int C, bool ZID>
int launch_update_ws_z(ss_handle* h, dim3 grid, size_t smem, cudaStream_t st, const UpdDims& u,
                       const double2* zin, double2* zout, const double2* pbuf) {
    static ss::DevMask configured;  // devices configured
    if (!configured.has(h)) {
        SS_CUDA_TRY(h, allow_max_smem(h, k_update_ws<G, C, ZID>));
        configured.set(h);
    }
    k_update_ws<G, C, ZID><<<grid, kWsThreads, smem, st>>>(u, zin, zout, pbuf);
    SS_LAUNCH_CHECK(h);
    return SS_OK;
}

template <int G, int C>
int launch_update_ws_t(ss_handle* h, dim3 grid, size_t smem, cudaStream_t st, const UpdDims& u,
                       const double2* zin, double2* zout, const double2* pbuf) {
    if (u.zid) return launch_update_ws_z<G, C, true>(h, grid, smem, st, u, zin, zout, pbuf);
    return launch_update_ws_z<G, C, false>(h, grid, smem, st, u, zin, zout, pbuf);
}

template <int G, int C, int R, int NPAIR, int NST, bool ZID, int NCB, bool MSH = false>
int launch_far_z(ss_handle* h, int grid, size_t smem, cudaStream_t st, const UpdDims& u, double2* z,
                 const double2* pbuf) {
    static ss::DevMask configured;  // devices configured
    if (!configured.has(h)) {
        SS_CUDA_TRY(h, allow_max_smem(h, k_far<G, C, R, NPAIR, NST, ZID, NCB, MSH>));
        configured.set(h);
    }
    k_far<G, C, R, NPAIR, NST, ZID, NCB, MSH><<<grid, far_threads(NPAIR), smem, st>>>(u, z, pbuf);
    SS_LAUNCH_CHECK(h);
    return SS_OK;
}

// Far-row kernel shape: R rows x C columns per lane, 32/G row groups -> a
// tile of (32/G) R rows; NPAIR consumer pairs; NST ring stages.
struct FarShape {
    int G, C, R, NPAIR, NST, NCB;
    bool MSH = false;  // m = 1: the G C columns are G C different shifts
    int tile() const { return (32 / G) * R; }
    int m() const { return G * C * NCB; }
};

FarShape far_shape(const UpdTile& t) {
    // measured on B200 (config 2): R = 8 rows per lane (3 pairs, 255
    // registers, spills) and 3 pairs x 6 stages were slower than R = 2G with
    // 4 pairs / 8 stages
    return FarShape{t.G, t.C, 2 * t.G, 4, 8, 1};
}

// Persistent far-row update (ss_far.cuh): one CTA per SM over (tile, shift) units.
int launch_far(ss_handle* h, const FarShape& f, int grid, size_t smem, cudaStream_t st,
               const UpdDims& u, double2* z, const double2* pbuf) {
#define SS_FAR(GG, CC, RR, NP, NS, KB)                                                           \
    if (!f.MSH && f.G == GG && f.C == CC && f.R == RR && f.NPAIR == NP && f.NST == NS &&         \
        f.NCB == KB)                                                                             \
        return u.zid ? launch_far_z<GG, CC, RR, NP, NS, true, KB>(h, grid, smem, st, u, z, pbuf)  \
                     : launch_far_z<GG, CC, RR, NP, NS, false, KB>(h, grid, smem, st, u, z, pbuf);
    SS_FAR(2, 5, 4, 4, 8, 1) SS_FAR(2, 5, 4, 4, 4, 2)
    SS_FAR(2, 4, 4, 4, 8, 1)
    SS_FAR(1, 1, 2, 4, 8, 1) SS_FAR(1, 2, 2, 4, 8, 1) SS_FAR(1, 3, 2, 4, 8, 1) SS_FAR(1, 4, 2, 4, 8, 1)
    SS_FAR(1, 5, 2, 4, 8, 1) SS_FAR(1, 6, 2, 4, 8, 1) SS_FAR(1, 7, 2, 4, 8, 1) SS_FAR(1, 8, 2, 4, 8, 1)
#undef SS_FAR
    if (f.MSH && f.G == 2 && f.C == 5 && f.R == 4 && f.NPAIR == 4 && f.NST == 8 && f.NCB == 1)
        return u.zid ? launch_far_z<2, 5, 4, 4, 8, true, 1, true>(h, grid, smem, st, u, z, pbuf)
                     : launch_far_z<2, 5, 4, 4, 8, false, 1, true>(h, grid, smem, st, u, z, pbuf);
    return SS_EARG;
}

// 128-column far passes with the four-way K split (ss_far4.cuh), m = 10
template <bool ZID>
int launch_far4_z(ss_handle* h, int grid, size_t smem, cudaStream_t st, const UpdDims& u, double2* z,
                  const double2* pbuf) {
    static ss::DevMask configured;  // devices configured
    if (!configured.has(h)) {
        SS_CUDA_TRY(h, allow_max_smem(h, k_far4<2, 5, 4, ZID>));
        configured.set(h);
    }
    k_far4<2, 5, 4, ZID><<<grid, kFar4Threads, smem, st>>>(u, z, pbuf);
    SS_LAUNCH_CHECK(h);
    return SS_OK;
}

// Warp-specialised TMA/mbarrier update for tiles where one warp pair covers
// all m columns (G*C == m); returns SS_EARG when the tile is not covered.
int launch_update_ws(ss_handle* h, const UpdTile& t, dim3 grid, size_t smem, cudaStream_t st,
                     const UpdDims& u, const double2* zin, double2* zout, const double2* pbuf) {
    if (t.G == 2 && t.C == 5) return launch_update_ws_t<2, 5>(h, grid, smem, st, u, zin, zout, pbuf);
    if (t.G == 2 && t.C == 4) return launch_update_ws_t<2, 4>(h, grid, smem, st, u, zin, zout, pbuf);
    if (t.G == 1) {
        switch (t.C) {
#define SS_CASE(K) \
    case K: return launch_update_ws_t<1, K>(h, grid, smem, st, u, zin, zout, pbuf);
            SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8)
#undef SS_CASE
            default: break;
        }
    }
    return SS_EARG;
}

int launch_update(ss_handle* h, const UpdTile& t, dim3 grid, int threads, size_t smem,
                  cudaStream_t st, const UpdDims& u, const double2* zin, double2* zout,
                  const double2* pbuf) {
    if (t.G == 2 && t.C == 5 && t.exact) return launch_update_t<2, 5, true>(h, grid, threads, smem, st, u, zin, zout, pbuf);
    if (t.G == 2 && t.C == 5) return launch_update_t<2, 5, false>(h, grid, threads, smem, st, u, zin, zout, pbuf);
    if (t.G == 2 && t.C == 4) return launch_update_t<2, 4, true>(h, grid, threads, smem, st, u, zin, zout, pbuf);
    if (t.G == 1) {
        switch (t.C) {
#define SS_CASE(K) \
    case K: return launch_update_t<1, K, true>(h, grid, threads, smem, st, u, zin, zout, pbuf);
            SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8)
#undef SS_CASE
            default: break;
        }
    }
    return ss::set_err(h, SS_EARG, "unsupported update tile");
}

// Transposed sweep's rows-below update (ss_lq.cu) on the window-update
// kernel with the [A^T; -I] panel (k_update<..., TR = true>): the state has
// mp = m + 1 columns (the m active columns and w).
template <int G, int C, bool EXACT>
int launch_update_tr_t(ss_handle* h, dim3 grid, int threads, size_t smem, cudaStream_t st, const UpdDims& u,
                       double2* S, const double2* P) {
    static ss::DevMask configured;  // devices configured
    if (!configured.has(h)) {
        SS_CUDA_TRY(h, allow_max_smem(h, k_update<G, C, EXACT, 320, false, true>));
        SS_CUDA_TRY(h, allow_max_smem(h, k_update<G, C, EXACT, 320, true, true>));
        configured.set(h);
    }
    if (smem > h->smem_optin)
        k_update<G, C, EXACT, 320, true, true><<<grid, threads, upd_smem_bytes(u.nb, u.m, u.S, true), st>>>(u, S, S, P);
    else
        k_update<G, C, EXACT, 320, false, true><<<grid, threads, smem, st>>>(u, S, S, P);
    SS_LAUNCH_CHECK(h);
    return SS_OK;
}

}  // namespace

namespace ss {
int launch_update_tr(ss_handle* h, UpdDims u, int rows, double2* S, const double2* P, cudaStream_t st) {
    const UpdTile t = pick_tile(u.m);
    const int nws = (u.m + t.G * t.C - 1) / (t.G * t.C);
    u.nws = nws;
    u.ksplit = 1;
    u.jh = u.nb;
    u.S = std::max(1, std::min(8 / nws, 4));
    const size_t two_per_sm = h->smem_optin / 2 - 1024;
    while (u.S > 1 && upd_smem_bytes(u.nb, u.m, u.S) > two_per_sm) u.S--;
    u.SG = u.S * 4;
    u.pstride = (int64_t)u.nc * u.m;
    u.p12off = 0;
    u.p22off = (int64_t)u.nb * u.m;
    u.zid = 0;
    u.flags = 0;
    const dim3 grid((unsigned)((rows + kUpdRows - 1) / kUpdRows), (unsigned)((u.sb + u.SG - 1) / u.SG));
    const int threads = 32 * u.S * nws;
    const size_t smem = upd_smem_bytes(u.nb, u.m, u.S);
    if (t.G == 2 && t.C == 5 && t.exact) return launch_update_tr_t<2, 5, true>(h, grid, threads, smem, st, u, S, P);
    if (t.G == 2 && t.C == 5) return launch_update_tr_t<2, 5, false>(h, grid, threads, smem, st, u, S, P);
    if (t.G == 2 && t.C == 4) return launch_update_tr_t<2, 4, true>(h, grid, threads, smem, st, u, S, P);
    if (t.G == 1) {
        switch (t.C) {
#define SS_CASE(K) \
    case K: return launch_update_tr_t<1, K, true>(h, grid, threads, smem, st, u, S, P);
            SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8)
#undef SS_CASE
            default: break;
        }
    }
    return ss::set_err(h, SS_EARG, "unsupported update tile");
}
}  // namespace ss

namespace {

// widest window <= nb_req whose block RQ and update fit one SM's shared
// memory (the update may read P from global memory, k_update<..., PG>);
// 0 if none does (m too wide for this device)
int max_nb_for(ss_handle* h, int m, int nb_req) {
    for (int nb = nb_req; nb >= 1; nb = nb > 8 ? nb - 8 : nb - 1) {
        const size_t need = rq_smem_bytes(nb, m, nb * m, nb * m);
        const size_t upd = upd_smem_bytes(nb, m, 1, true);
        // m + 1 > 64 runs the scheduled Givens batch (k_rq): <= 16 warps keep
        // at most 8 x 32 rotations each in registers (~ nb m / 16 + nb + m)
        const bool rots_ok = m + 1 <= 64 || nb * m / 16 + nb + m <= 256;
        if (need <= h->smem_optin && upd <= h->smem_optin && nb + m <= 255 && rots_ok) return nb;
    }
    return 0;
}

struct SweepArgs {
    int mode;  // 0 tf, 1 reduced
    int n, m, p;
    const double* A;
    int64_t lda;
    const double* B;
    int64_t ldb;
    const double* C;
    int64_t ldc;
    const double2* shifts;
    int64_t s;
    const double2* bd;
    int64_t ldbd;
    int nb;
    int64_t batch;
    double rtol;
    double2* out;
    int64_t ldo;
    int32_t* fail;
    // streamed Ahat (ss_tf_eval_stream): host source; A above is the device
    // destination, filled chunk by chunk in sweep order on h->copy_stream
    const double* A_host = nullptr;
    int64_t lda_host = 0;
    // reduced solve with the identity top deferred (two-level sweep): the
    // sweep runs on Ahat alone (no top rows), each composite's W12 / W22 are
    // kept per shift and x = [I; 0]-part is expanded after the head (k_expand)
    bool defer = false;
    int group = 1;
};

// Streamed-Ahat bookkeeping for one call: chunk c's event is recorded on the
// copy stream after its columns landed; the compute stream waits on it right
// before the first kernel that reads those columns.
struct Feed {
    bool on = false;
    bool fro2_pending = false;  // ||A||_F / trace(A) after the last chunk
    int next = 0;               // next chunk to wait for
    int count = 0;
};

// Column chunks of Ahat in the order the sweep consumes them: the seed's last
// m columns, then each outer block's (two-level) or window's panel columns.
static void sweep_chunks(int n, int m, bool two_level, int nb0, std::vector<std::pair<int, int>>& out) {
    out.clear();
    out.push_back({n - m, n});
    for (int k = n; k >= m + 1;) {
        const int w = std::min(two_level ? kBlkNB : nb0, k - m);
        out.push_back({k - m - w, k - m});
        k -= w;
    }
}

static int feed_wait(ss_handle* h, Feed& f, cudaStream_t st) {
    if (!f.on || f.next >= f.count) return SS_OK;
    SS_CUDA_TRY(h, cudaStreamWaitEvent(st, h->chunk_ev[f.next], 0));
    ++f.next;
    return SS_OK;
}

// Per-part device buffers: Z2 ping-pong + P for the part's shifts.
struct PartBufs {
    double2* Z;  // window state, updated in place
    double2* P;
    double* pan = nullptr;  // packed panel of the K-streamed far kernel (k_fark)
    double2* W = nullptr;   // window composites: per shift (kWcWin nb0 + m) x m
    // deferred reduced solve: per shift W12 history (n x m, row = panel column,
    // j-major) and the composites' W22 (ncomp x m x m), plus the head's y (m)
    double2* Xh = nullptr;
    double2* W22h = nullptr;
    double2* Y = nullptr;
    int64_t xh_stride = 0, w22h_stride = 0;
};

// K-streamed far kernel (ss_fark.cuh): one pass per composite for m = 10, 20
// (transfer function); SS_FAR_PASSES=1 keeps the 64 / 128-column pass
// kernels (k_far / k_far4) for comparison.
constexpr int kFarkStages = 4;
// m = 20 unit shape: shifts per unit x ring stages (comparison builds vary them)
#ifndef SS_S20
#define SS_S20 4
#endif
#ifndef SS_N20
#define SS_N20 kFarkStages
#endif
static bool fark_supported(ss_handle* h, int m, int mode) {
    if (mode != 0 || getenv("SS_FAR_PASSES")) return false;
    if (m == 10) return fark_smem_bytes<1, 8, kFarkStages>() <= h->smem_optin;
    if (m == 20) return fark_smem_bytes<2, SS_S20, SS_N20>() <= h->smem_optin;
    return false;
}
static size_t fark_pan_bytes(int n, int ptop) {
    const size_t ntiles = (size_t)(ptop + n) / kFkTile + 2;
    return ntiles * ((4 * kBlkNB + kFkKC - 1) / kFkKC) * kFkKC * kFkTile * 8;  // K <= 4 outer blocks
}
// The far passes run on DFMA (k_fark / k_farkm).  north_star allows FP64
// tensor-core DMMA only in the reduction's trailing updates, so the DMMA
// consumers (ss_farkd.cuh: k_farkd / k_farkmd, measured +25% at config 4)
// are compiled only into comparison builds (-DSS_FARK_DMMA,
// tools/build_variant.sh), never into the product library.
#ifdef SS_FARK_DMMA
constexpr bool kFarkDmma = true;
// the packed panel in DMMA fragment order for k_farkd / k_farkmd
static void pack_panel(const FarKDims& fk, double* pan, cudaStream_t st) {
    k_pack_panel_d<<<fk.ntiles * fk.nk, 256, 0, st>>>(fk, pan);
}
static void pack_panel_tr(const FarKDims& fk, double* pan, cudaStream_t st) {
    k_pack_panel_tr_d<<<fk.ntiles * fk.nk, 256, 0, st>>>(fk, pan);
}
#else
constexpr bool kFarkDmma = false;
template <int NCB, int S>
__host__ __device__ constexpr int farkd_jz() { return fark_jz<NCB, S>(); }
static void pack_panel(const FarKDims& fk, double* pan, cudaStream_t st) {
    k_pack_panel<<<fk.ntiles * fk.nk, 256, 0, st>>>(fk, pan);
}
static void pack_panel_tr(const FarKDims& fk, double* pan, cudaStream_t st) {
    k_pack_panel_tr<<<fk.ntiles * fk.nk, 256, 0, st>>>(fk, pan);
}
#endif
#ifdef SS_FARK_DMMA
template <int NCB, int S, int NST, int WR, int WC>
int launch_farkd(ss_handle* h, int grid, cudaStream_t st, const FarKDims& fk, double2* Z, const double2* W) {
    static ss::DevMask configured;
    if (!configured.has(h)) {
        SS_CUDA_TRY(h, cudaFuncSetAttribute(k_farkd<NCB, S, NST, WR, WC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)fark_smem_bytes<NCB, S, NST>()));
        configured.set(h);
    }
    k_farkd<NCB, S, NST, WR, WC><<<grid, 32 * (1 + WR * WC * S), fark_smem_bytes<NCB, S, NST>(), st>>>(fk, Z, W);
    SS_LAUNCH_CHECK(h);
    return SS_OK;
}
#else
template <int NCB, int S, int NST, int WR, int WC>
int launch_farkd(ss_handle* h, int, cudaStream_t, const FarKDims&, double2*, const double2*) {
    return ss::set_err(h, SS_EARG, "DMMA far kernel not built (SS_FARK_DMMA)");
}
#endif
template <int NCB, int S, int NST = kFarkStages>
int launch_fark(ss_handle* h, int grid, cudaStream_t st, const FarKDims& fk, double2* Z, const double2* W) {
    static ss::DevMask configured;  // devices configured
    if (!configured.has(h)) {
        SS_CUDA_TRY(h, cudaFuncSetAttribute(k_fark<NCB, S, NST>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)fark_smem_bytes<NCB, S, NST>()));
        configured.set(h);
    }
    k_fark<NCB, S, NST><<<grid, 32 * (1 + NCB * S), fark_smem_bytes<NCB, S, NST>(), st>>>(fk, Z, W);
    SS_LAUNCH_CHECK(h);
    return SS_OK;
}

// ---------------------------------------------------------------------------
// Window composites for wide windows (m = 40, 50, 60 on the shared-memory
// RQ, k_rq_big): the windows of a composite (up to kWcWin windows of kWcNb
// columns, bottom-up) are factored one by one; each window's P updates only
// the composite's own rows above it ("near", the generic k_update) and is
// kept; the composite W = [W12 (K x m); W22 (m x m)] is then built from all
// of them at once (k_wsuffix, the suffix product of the windows' P22; the
// same algebra as folding window by window:
//     W12[window rows] <- P12,  W12[rows below] <- W12 P22,  W22 <- W22 P22)
// and the rows above the composite get ONE K-streamed update (k_farkd, one
// pass over the K columns).  The far rows' state x W22 share of
// the work drops from 2m / nb0 (104% at m = 50, nb0 = 96) to 2m / K.
// Same algebra as the two-level sweep's composites (ss_block.cuh).
// ---------------------------------------------------------------------------
// measured at config 5 (m = 50): (nb0, windows) = (96, 4) 315, (96, 6) 325,
// (64, 6) 336, (64, 8) 341, (48, 8) 326, (32, 12) 326 shifts/s -- narrower
// windows cut k_rq_big's chain (n nb / 2 row updates per shift), more
// windows per composite cut the far rows' 2m / K share, both add near updates
constexpr int kWcWin = 8;
constexpr int kWcNb = 64;
struct WcShape {
    int S, NST;
};
// Consumer warps per CTA = NCB S: a multiple of 4 keeps the four SM
// sub-partitions' FP64 pipes evenly loaded (m = 50: 10 warps, <5,2,3>, 344
// shifts/s at config 5; 15 warps, <5,3,2>, 364; 5 warps, <5,1,4>, 273)
static bool wc_shape(int m, WcShape& w) {
    if (m == 1) { w = {kFkmShifts, 4}; return true; }
    if (m == 40) { w = {2, 3}; return true; }
    if (m == 50) { w = kFarkDmma ? WcShape{1, 4} : WcShape{3, 2}; return true; }
    if (m == 60) { w = kFarkDmma ? WcShape{1, 4} : WcShape{2, 2}; return true; }
    return false;
}
static size_t wc_far_smem(int m) {
    switch (m) {
        case 1: return farkm_smem_bytes<4>();
        case 40: return fark_smem_bytes<4, 2, 3>();
        case 50: return kFarkDmma ? fark_smem_bytes<5, 1, 4>() : fark_smem_bytes<5, 3, 2>();
        case 60: return kFarkDmma ? fark_smem_bytes<6, 1, 4>() : fark_smem_bytes<6, 2, 2>();
        default: return ~(size_t)0;
    }
}
static int wc_jz(int m) {
    switch (m) {
        case 40: return kFarkDmma ? farkd_jz<4, 2>() : fark_jz<4, 2>();
        case 50: return kFarkDmma ? farkd_jz<5, 1>() : fark_jz<5, 3>();
        default: return kFarkDmma ? farkd_jz<6, 1>() : fark_jz<6, 2>();
    }
}
static int launch_farkm(ss_handle* h, int grid, cudaStream_t st, const FarKDims& fk, double2* Z,
                        const double2* W) {
    static ss::DevMask configured;  // devices configured
    if (!configured.has(h)) {
        SS_CUDA_TRY(h, cudaFuncSetAttribute(k_farkm<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)farkm_smem_bytes<4>()));
#ifdef SS_FARK_DMMA
        SS_CUDA_TRY(h, cudaFuncSetAttribute(k_farkmd<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)farkm_smem_bytes<4>()));
#endif
        configured.set(h);
    }
#ifdef SS_FARK_DMMA
    k_farkmd<4><<<grid, 32 * 9, farkm_smem_bytes<4>(), st>>>(fk, Z, W);
#else
    k_farkm<4><<<grid, 32 * 9, farkm_smem_bytes<4>(), st>>>(fk, Z, W);
#endif
    SS_LAUNCH_CHECK(h);
    return SS_OK;
}
static int launch_wc_far(ss_handle* h, int m, int grid, cudaStream_t st, const FarKDims& fk, double2* Z,
                         const double2* W) {
    // DMMA: four warps per shift (one m16 row tile each, every column tile)
    switch (m) {
        case 40: return kFarkDmma ? launch_farkd<4, 2, 3, 2, 2>(h, grid, st, fk, Z, W) : launch_fark<4, 2, 3>(h, grid, st, fk, Z, W);
        case 50: return kFarkDmma ? launch_farkd<5, 1, 4, 4, 2>(h, grid, st, fk, Z, W) : launch_fark<5, 3, 2>(h, grid, st, fk, Z, W);
        case 60: return kFarkDmma ? launch_farkd<6, 1, 4, 4, 2>(h, grid, st, fk, Z, W) : launch_fark<6, 2, 2>(h, grid, st, fk, Z, W);
        default: return ss::set_err(h, SS_EARG, "window composite: unsupported m");
    }
}

// Composite W layout: element (row, c) of shift l at
//   W + (l / G) gs + (l % G) ls + row rs + c
// (m > 1: G = 1, gs = per-shift stride, rs = m, j-major rows of one shift;
//  m = 1, k_farkm: G = 80, gs = (Kmax + 1) 80, ls = 1, rs = 80, the group's
//  shifts side by side in every row).
struct WcLayout {
    int G;
    int64_t gs, ls, rs;
    __host__ __device__ int64_t off(int l) const { return (int64_t)(l / G) * gs + (int64_t)(l % G) * ls; }
};

// The composite from ALL its windows' P at once (instead of folding window by
// window, which multiplies the earlier windows' W12 rows again for every
// later window: O(g^2) row products).  In processing order b = 0 .. g-1:
//     W12[x_b, x_b + nb_b) = P12_b S_b,  S_b = P22_{b+1} ... P22_{g-1},
//     W22 = P22_0 ... P22_{g-1}  (= S_{-1})
// built backward with S in shared memory; one CTA per shift.  Only the first
// mc <= M columns are carried (the padding of P / W is zero).
constexpr int kWsufMax = 64;  // windows per composite (the transposed G <= 64)
struct WsufArgs {
    int g, M, mc, K;
    int x[kWsufMax], nb[kWsufMax];
    const double2* P;   // window b, shift l: P + b * slab + l * (nb_b + M) M
    int64_t slab;
    double2* W;         // shift l: W + l * wstride, rows of M
    int64_t wstride;
};
// Both products of window b are ONE (nb + M) x M times M x M product:
// [W12_b; S_new] = P_b S.  Register-tiled: each thread owns 4 x 4 outputs
// (rows rt + nr i, columns ct + nc k: interleaved, so a warp's shared loads
// of one k are contiguous) with P_b and S staged in shared memory (row
// length LS = 4 ceil(M / 4) + 1: odd in 16-byte units, adjacent rows in
// different banks; zero padded).  Tiles are numbered S rows first, so a
// thread holds at most one S tile in registers across the barrier that
// precedes the in-place S update (M <= 64: ceil(M / 4)^2 <= kWsT).
constexpr int kWsT = 384;
__host__ __device__ inline int wsuf_nc(int M) { return (M + 3) >> 2; }
__host__ __device__ inline size_t wsuf_smem(int M, int nbmax) {
    const int Q = 4 * wsuf_nc(M), LS = Q + 1;
    return ((size_t)(nbmax + 3 + Q) * LS + (size_t)Q * LS) * 16;
}

__global__ void __launch_bounds__(kWsT) k_wsuffix(WsufArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int M = a.M, mc = a.mc, l = blockIdx.x, tid = threadIdx.x;
    const int nc = wsuf_nc(M), Q = 4 * nc, LS = Q + 1, nS = nc * nc;
    double2* S = reinterpret_cast<double2*>(smem);  // Q x LS (only mc x mc nonzero)
    double2* Ps = S + Q * LS;                       // (nb + Q) x LS
    double2* Wl = a.W + (int64_t)l * a.wstride;
    for (int e = tid; e < Q * LS; e += kWsT) {
        const int r = e / LS, c = e - r * LS;
        S[e] = make_double2(r == c && r < mc ? 1.0 : 0.0, 0.0);
    }
    for (int b = a.g - 1; b >= 0; --b) {
        const int nb = a.nb[b], R = nb + M, nrw = (nb + 3) >> 2;
        const double2* Pl = a.P + b * a.slab + (int64_t)l * R * M;
        // rows [0, 4 nrw) hold W12 (zero beyond nb), rows [4 nrw, 4 nrw + Q)
        // P22 (zero beyond M)
        const int W0 = 4 * nrw;
        for (int e = tid; e < (W0 + Q) * LS; e += kWsT) {
            const int r = e / LS, c = e - r * LS;
            const int pr = r < W0 ? (r < nb ? r : -1) : (r - W0 < M ? nb + r - W0 : -1);
            Ps[e] = (pr >= 0 && c < M) ? Pl[(int64_t)pr * M + c] : cz();
        }
        __syncthreads();
        const int ntiles = nS + nrw * nc;
        double2 keep[4][4];
        bool has_s = false;
        int ks_r = 0, ks_c = 0;
        for (int t = tid; t < ntiles; t += kWsT) {
            const bool st = t < nS;
            const int u = st ? t : t - nS;
            const int rt = u / nc, ct = u - rt * nc, nr = st ? nc : nrw;
            const double2* pr = Ps + (st ? W0 : 0) * LS + rt * LS;
            double2 acc[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int k = 0; k < 4; ++k) acc[i][k] = cz();
            for (int j = 0; j < mc; ++j) {
                double2 pa[4], sv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) pa[i] = pr[i * nr * LS + j];
#pragma unroll
                for (int k = 0; k < 4; ++k) sv[k] = S[j * LS + ct + nc * k];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int k = 0; k < 4; ++k) acc[i][k] = cfma(pa[i], sv[k], acc[i][k]);
            }
            if (st) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int k = 0; k < 4; ++k) keep[i][k] = acc[i][k];
                has_s = true;
                ks_r = rt;
                ks_c = ct;
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int r = rt + nrw * i;
                    if (r >= nb) continue;
                    double2* w = Wl + (int64_t)(a.x[b] + r) * M;
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (ct + nc * k < M) w[ct + nc * k] = acc[i][k];
                }
            }
        }
        __syncthreads();  // every read of S and Ps done
        if (has_s) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int k = 0; k < 4; ++k) S[(ks_r + nc * i) * LS + ks_c + nc * k] = keep[i][k];
        }
        // (the next window's staging barrier orders these writes)
    }
    __syncthreads();
    // W22 = S (the padding rows / columns of S are zero)
    for (int e = tid; e < M * M; e += kWsT) {
        const int r = e / M, c = e - r * M;
        Wl[(int64_t)(a.K + r) * M + c] = S[r * LS + c];
    }
}

// m = 1: the composite from all its windows' P at once (scalars: W12 rows of
// window b = P12_b times the suffix product of the later windows' P22, W22 =
// the product of all of them), in the group layout [group][row][80]
// (row-major across a group's shifts: coalesced), one thread per (row,
// shift).  Windows: rows [x_b, x_b + nb_b) of the composite, P of window b,
// shift l at P + b slab + l (nb_b + 1).
struct Wsuf1Args {
    int g, K, sb;
    int x[kWcWin], nb[kWcWin];
    const double2* P;
    int64_t slab, gstride;
    double2* W;
};
__global__ void __launch_bounds__(256) k_wsuffix1(Wsuf1Args a) {
    constexpr int S = kFkmShifts;
    const int ngroups = (a.sb + S - 1) / S;
    const int64_t per = (int64_t)(a.K + 1) * S;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < per * ngroups;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int grp = (int)(e / per);
        const int64_t rem = e - grp * per;
        const int row = (int)(rem / S), c = (int)(rem % S);
        const int l = min(grp * S + c, a.sb - 1);
        double2 v = make_double2(1.0, 0.0);
        int bw = -1;  // the window holding this row (W12), -1: the W22 row
        if (row < a.K)
            for (int b = 0; b < a.g; ++b)
                if (row >= a.x[b] && row < a.x[b] + a.nb[b]) bw = b;
        // suffix product of the P22 of the windows after bw (all of them for W22)
        for (int b = bw + 1; b < a.g; ++b)
            v = cmul(v, a.P[b * a.slab + (int64_t)l * (a.nb[b] + 1) + a.nb[b]]);
        if (bw >= 0) v = cmul(a.P[bw * a.slab + (int64_t)l * (a.nb[bw] + 1) + (row - a.x[bw])], v);
        a.W[grp * a.gstride + (int64_t)row * S + c] = v;
    }
}

// Enqueue the whole sweep (seed, window steps, head) for shifts
// [lo, lo + sb) of the call on stream `st`.
int launch_block(ss_handle* h, int m, int sb, size_t smem, cudaStream_t st, const BlkDims& bd,
                 double2* Z, double2* W) {
    switch (m) {
#define SS_CASE(K)                                                        \
    case K: {                                                             \
        static ss::DevMask configured;                                   \
        if (!configured.has(h)) {                                                \
            SS_CUDA_TRY(h, allow_max_smem(h, k_block<K, kBlkShiftsPerWarp>)); \
            configured.set(h);                                            \
        }                                                                 \
        k_block<K, kBlkShiftsPerWarp>                                     \
            <<<(sb + kBlkShiftsPerWarp - 1) / kBlkShiftsPerWarp, 32, smem, st>>>(bd, Z, W, sb); \
        break;                                                            \
    }
        SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) SS_CASE(10) SS_CASE(20)
#undef SS_CASE
        default: return ss::set_err(h, SS_EARG, "two-level sweep: unsupported m");
    }
    SS_LAUNCH_CHECK(h);
    return SS_OK;
}

// m + 1 > 32 (config 5): the shared-memory Householder RQ (ss_rq_big.cuh) on
// 96-column windows unless SS_BLOCK_RQ=givens asks for the reference's batch
static bool rq_big(int m) {
    const char* e = getenv("SS_BLOCK_RQ");
    return m + 1 > 32 && m + 1 <= 64 && !(e && strcmp(e, "givens") == 0);
}
constexpr int kRqBigNb = 96;

// m < 4: the per-window overhead 2m/nb is already < 13% at nb = 64 and the
// one-level sweep measured faster (config 3, m = 1: 13.7 vs 19.3 ms)
bool block_supported(int m) { return (m >= 4 && m <= 8) || m == 10 || m == 20; }

// Paired outer blocks (composite W over 256 columns for the far rows);
// SS_NO_PAIR=1 keeps one far update per 128-column block.
static int two_level_group(ss_handle* h, int m, int mode) {
    if (getenv("SS_NO_PAIR")) return 1;
    if (const char* e = getenv("SS_GROUP")) {
        const int g = atoi(e);
        if (g == 1 || g == 2 || g == 4) return g;
    }
    // one pass per composite (k_fark): 4 outer blocks per composite halve
    // the far rows' Z W22 share (2m / 512) and Z traffic; the pass kernels
    // keep pairs
    return fark_supported(h, m, mode) ? 4 : 2;
}
// Reference phase flops of the window sweep at block size nb0 (shape only:
// batched.py:58-61, solvers.py:186-199), independent of how the device
// schedules the work.
void account_ref_flops(ss_handle* h, int sb, int n, int m, int ptop, int nb0) {
    for (int k = n; k >= m + 1;) {
        const int nb = std::min(nb0, k - m), nc = nb + m, mnb = std::min(m, nb);
        const int r0 = ptop + k - nb;
        const ss::Sched* sc = ss::get_sched(h, nb, nc);
        double rq_fl = 0.0;
        if (sc)
            for (int qq = 0; qq < sc->rots; ++qq) rq_fl += 20.0 * ((sc->rot[qq] & 0xffu) + nc) + 16.0;
        h->flops[ss::PH_RQ] += rq_fl * sb;
        h->flops[ss::PH_BATCHED_GEMM] += (double)sb * (8.0 * r0 * m * m + 8.0 * mnb * m);
        h->flops[ss::PH_OUTER_GEMM] += 8.0 * r0 * ((double)sb * m) * nb;
        k -= nb;
    }
}

}  // namespace
namespace ss {
int wsuffix(ss_handle* h, cudaStream_t st, int sb, int g, const int* x, const int* nb, int M, int mc, int K,
            const double2* P, int64_t slab, double2* W, int64_t wstride);
}
namespace {

int enqueue_part(ss_handle* h, const SweepArgs& a, int64_t lo, int sb, PartBufs B, int nb0,
                 int64_t LDZ, double rtol, bool use_house, const UpdTile& tile, bool two_level,
                 bool wc, cudaStream_t st, Feed& feed) {
    const int n = a.n, m = a.m;
    const int ptop = a.mode == 0 ? a.p : (a.defer ? 0 : n);
    const int mode_far = a.defer ? 0 : a.mode;  // deferred reduced solve: far rows as tf with p = 0
    const int nws = (m + tile.G * tile.C - 1) / (tile.G * tile.C);  // warps per shift
    Dims d;
    d.n = n;
    d.m = m;
    d.ptop = ptop;
    d.ident_top = a.mode == 1 && !a.defer;
    d.A = a.A;
    d.lda = a.lda;
    d.T = a.C;
    d.ldt = a.ldc;
    d.shifts = a.shifts + lo;
    d.sb = sb;
    d.LDZ = LDZ;
    {
        int rc = feed_wait(h, feed, st);  // the seed's last m columns
        if (rc) return rc;
        dim3 g((unsigned)((LDZ + 255) / 256), (unsigned)sb);
        k_seed<<<g, 256, 0, st>>>(d, B.Z);
        SS_LAUNCH_CHECK(h);
    }
    int k = two_level ? 0 : n;
    if (two_level) {
        // ---- two-level sweep: k_block per outer block, far rows from W ----
        // Outer blocks are paired (A = the lower block, B the one above it):
        // after k_block(A) only B's own rows get A's update ("near"); k_block
        // (B) then folds A's W into the composite over both blocks, and the
        // rows above B get ONE update from it -- the Z2 W22 part on the far
        // rows is paid once per 256 columns instead of once per 128.
        account_ref_flops(h, sb, n, m, a.mode == 0 ? a.p : n, nb0);  // the reference's stack
        const int group = a.group;
        const int64_t wstride = (int64_t)(group * kBlkNB + m) * m;
        // far-row update of rows [rlo, r0) from the W rows [woff, woff + ncols
        // + m) of the buffer, panel columns [c0, c0 + ncols), in 64-column passes
        // m = 10: 128-column passes on the four-way-split far kernel (SS_FAR4=0: 64-column k_far)
        const bool far4 = m == 10 && tile.G == 2 && tile.C == 5 &&
                          !(getenv("SS_FAR4") && atoi(getenv("SS_FAR4")) == 0) &&
                          far4_smem_bytes<2, 5, 4>(128, m) + 1024 <= h->smem_optin;
        const int pw = far4 ? 128 : 64;
        const bool fark = B.pan != nullptr && fark_supported(h, m, mode_far);
        auto far_update = [&](int rlo, int r0, int c0, int ncols, int woff) -> int {
            const int rows = r0 - rlo;
            if (fark && rows > 0) {
                // one pass over the whole composite (ss_fark.cuh)
                FarKDims fk;
                fk.m = m;
                fk.ptop = ptop;
                fk.ident_top = d.ident_top;
                fk.A = a.A;
                fk.lda = a.lda;
                fk.T = a.C;
                fk.ldt = a.ldc;
                fk.shifts = d.shifts;
                fk.sb = sb;
                fk.LDZ = LDZ;
                fk.r0 = r0;
                fk.rlo = rlo;
                fk.c0 = c0;
                fk.K = ncols;
                fk.mnb = std::min(m, ncols);
                fk.wstride = wstride;
                fk.woff = woff;
                fk.nk = (ncols + kFkKC - 1) / kFkKC;
                // m = 20: 4 shifts x 2 column blocks per unit, 4 stages (measured
                // at config 4 against 3 x 4 / 5 x 3 / 6 x 2: 4.01k / 4.31k / 4.70k
                // vs 4.82k shifts/s)
                constexpr int S20 = SS_S20, N20 = SS_N20;
                const bool dmma = kFarkDmma;
                fk.jz = m == 10 ? (dmma ? farkd_jz<1, 4>() : fark_jz<1, 8>())
                                : (dmma ? farkd_jz<2, S20>() : fark_jz<2, S20>());
                fk.nz = (m + fk.jz - 1) / fk.jz;
                fk.ntiles = (rows + kFkTile - 1) / kFkTile;
                fk.pan = B.pan;
                cudaEvent_t ev = ss::timing_begin(h, st);
                pack_panel(fk, B.pan, st);
                SS_LAUNCH_CHECK(h);
                ss::timing_end(h, st, ev, ss::PH_OUTER_GEMM);
                const int S = m == 10 ? (dmma ? 4 : 8) : S20;
                const int64_t units = (int64_t)fk.ntiles * ((sb + S - 1) / S);
                // teams of 4 CTAs per shift group: the live W set drops from ~100 MB
                // (over L2) to ~25 MB, DRAM bytes per launch 8.5 -> 2.6 GB at config 4
                fk.spl = units >= 8 * (int64_t)h->num_sms ? 4 : 1;
                const int grid = (int)std::max<int64_t>(
                    fk.spl, std::min<int64_t>(units, h->num_sms) / fk.spl * fk.spl);
                double nnz = 0.0;  // algorithmic flops: structural nonzeros x m complex columns
                const int top_hi = std::min(r0, ptop);
                if (top_hi > rlo) nnz += (double)(top_hi - rlo) * ncols;
                if (r0 > std::max(rlo, ptop)) nnz += (double)(r0 - std::max(rlo, ptop)) * ncols;
                ev = ss::timing_begin(h, st);
                int rc = m == 10 ? (dmma ? launch_farkd<1, 4, kFarkStages, 2, 1>(h, grid, st, fk, B.Z, B.P)
                                         : launch_fark<1, 8>(h, grid, st, fk, B.Z, B.P))
                                 : (dmma ? launch_farkd<2, S20, N20, 2, 1>(h, grid, st, fk, B.Z, B.P)
                                         : launch_fark<2, S20, N20>(h, grid, st, fk, B.Z, B.P));
                if (rc) return rc;
                ss::timing_end(h, st, ev, ss::PH_UPDATE, 8.0 * rows * m * m * (double)sb,
                               8.0 * rows * (double)sb * m * ncols, 4.0 * m * nnz * sb);
                return SS_OK;
            }
            for (int jb = 0; rows > 0 && jb < ncols; jb += pw) {
                const int nbp = std::min(pw, ncols - jb);
                UpdDims u;
                u.n = n;
                u.m = m;
                u.ptop = ptop;
                u.ident_top = d.ident_top;
                u.A = a.A;
                u.lda = a.lda;
                u.T = a.C;
                u.ldt = a.ldc;
                u.shifts = d.shifts;
                u.sb = sb;
                u.LDZ = LDZ;
                u.nb = nbp;
                u.mnb = jb == 0 ? std::min(m, ncols) : 0;
                u.r0 = r0;
                u.c0 = c0 + jb;
                u.nc = nbp + m;
                u.rlo = rlo;
                u.nws = 1;
                u.ksplit = 2;
                u.pstride = wstride;
                u.p12off = (int64_t)(woff + jb) * m;
                u.p22off = (int64_t)(woff + ncols) * m;
                u.zid = jb == 0 ? 0 : 1;
                u.S = 1;
                u.SG = 32;
                // half 0 also carries the Z2 part (two panel columns' worth of
                // DFMA per column of m unless it is the identity) and the epilogue
                u.jh = u.zid ? nbp / 2 : std::max(0, std::min(nbp, (nbp - 2 * m) / 2 - 1));
                u.flags = 0;
                // algorithmic flops: structurally nonzero panel entries of the
                // far rows (Chat rows dense, identity rows one per column,
                // Ahat rows above the band dense) x m complex columns
                double nnz = 0.0;
                const int top_hi = std::min(r0, ptop);
                if (top_hi > rlo) {
                    if (a.mode == 0) {
                        nnz += (double)(top_hi - rlo) * nbp;
                    } else {
                        const int clo = std::max(rlo, u.c0), chi = std::min(top_hi, u.c0 + nbp);
                        nnz += (double)std::max(0, chi - clo);
                    }
                }
                if (r0 > std::max(rlo, ptop)) nnz += (double)(r0 - std::max(rlo, ptop)) * nbp;
                const double fl_alg = 4.0 * m * nnz * sb;
                cudaEvent_t ev = ss::timing_begin(h, st);
                int rc;
                if (far4) {
                    // role targets in panel-column equivalents: role 0 adds the
                    // Z2 W22 part (2m) or the Z2 read and the epilogue, role 3
                    // the read-add-write of the group buffer
                    const int extra0 = (u.zid ? 1 : 2 * m) + 4;
                    int T = (nbp + extra0 + 4 + 3) / 4;
                    int j1 = std::max(0, T - extra0);
                    const int rest = (nbp - j1);
                    const int q = (rest - 2) / 3;
                    u.jq[0] = std::min(nbp, j1);
                    u.jq[1] = std::min(nbp, u.jq[0] + q + 1);
                    u.jq[2] = std::min(nbp, u.jq[1] + q + 1);
                    const int64_t units = (int64_t)((rows + 63) / 64) * sb;
                    const int grid = (int)std::min<int64_t>(units, h->num_sms);
                    rc = u.zid ? launch_far4_z<true>(h, grid, far4_smem_bytes<2, 5, 4>(nbp, m), st, u, B.Z, B.P)
                               : launch_far4_z<false>(h, grid, far4_smem_bytes<2, 5, 4>(nbp, m), st, u, B.Z, B.P);
                } else {
                    const FarShape f = m == 20 ? FarShape{2, 5, 4, 4, 4, 2} : far_shape(tile);
                    const int64_t units = (int64_t)((rows + f.tile() - 1) / f.tile()) * sb;
                    const int grid = (int)std::min<int64_t>(units, h->num_sms);
                    rc = launch_far(h, f, grid, far_smem_bytes(nbp, m, f.tile(), f.NST), st, u, B.Z,
                                    B.P);
                }
                if (rc) return ss::set_err(h, rc, "two-level far update: unsupported tile");
                // reference-phase split of the measured time by the far update's shares
                ss::timing_end(h, st, ev, ss::PH_UPDATE, u.zid ? 0.0 : 8.0 * rows * m * m * (double)sb,
                               8.0 * rows * (double)sb * m * nbp, fl_alg);
            }
            return SS_OK;
        };
        auto block = [&](int ko, int NBo, int woff, int wprod) -> int {
            BlkDims bd;
            bd.m = m;
            bd.ptop = ptop;
            bd.k = ko;
            bd.NBo = NBo;
            bd.c0 = ko - m - NBo;
            bd.r0 = ptop + ko - NBo;
            bd.A = a.A;
            bd.lda = a.lda;
            bd.shifts = d.shifts;
            bd.LDZ = LDZ;
            bd.wstride = wstride;
            bd.woff = woff;
            bd.wprod = wprod;
            int rc = feed_wait(h, feed, st);  // this outer block's panel columns
            if (rc) return rc;
            cudaEvent_t ev = ss::timing_begin(h, st);
            rc = launch_block(h, m, sb, blk_smem_bytes(m), st, bd, B.Z, B.P);
            if (rc) return rc;
            ss::timing_end(h, st, ev, ss::PH_RQ);
            return SS_OK;
        };
        // Groups of g <= group outer blocks (1 = bottom, the first processed;
        // only block 1 of the whole sweep can be ragged).  Per shift the W
        // buffer holds [W_g | ... | W_2 | W_1 | W22]: block b writes its W12 at
        // rows (g - b) 128 and (b >= 2) folds the composite of blocks 1..b-1
        // below it by its W22 (ss_block.cuh, wprod), so rows [(g - b) 128, end)
        // are the composite of blocks 1..b.  Before block b + 1 its own rows
        // get that composite ("near", untouched since the group began); after
        // block g the rows above the group get ONE update over
        // (g - 1) 128 + NB1 columns.
        int ncomp = 0;  // composites so far (deferred reduced solve)
        for (int ko = n; ko >= m + 1;) {
            const int NB1 = std::min(kBlkNB, ko - m);
            const int avail = (ko - NB1 - m) / kBlkNB;  // full blocks above block 1
            const int g = 1 + std::min(group - 1, avail);
            int kb = ko, NBb = NB1;
            for (int b = 1; b <= g; ++b) {
                const int woff = (g - b) * kBlkNB;
                const int K = (b - 1) * kBlkNB + NB1;  // columns of the composite 1..b
                int rc = block(kb, NBb, woff, b == 1 ? 0 : (b - 2) * kBlkNB + NB1 + m);
                if (rc) return rc;
                const int c0 = kb - m - NBb, r0 = ptop + kb - NBb;
                if (b < g)
                    rc = far_update(r0 - kBlkNB, r0, c0, K, woff);  // near: block b + 1's rows
                else
                    rc = far_update(mode_far == 1 ? c0 : 0, r0, c0, K, 0);
                if (rc) return rc;
                if (b == g && a.defer) {
                    // keep the composite: W12 rows -> history rows [c0, c0 + K),
                    // W22 -> composite slot
                    SS_CUDA_TRY(h, cudaMemcpy2DAsync(B.Xh + (int64_t)c0 * m, (size_t)B.xh_stride * 16, B.P,
                                                     (size_t)wstride * 16, (size_t)K * m * 16, (size_t)sb,
                                                     cudaMemcpyDeviceToDevice, st));
                    SS_CUDA_TRY(h, cudaMemcpy2DAsync(B.W22h + (int64_t)ncomp * m * m, (size_t)B.w22h_stride * 16,
                                                     B.P + (int64_t)K * m, (size_t)wstride * 16,
                                                     (size_t)m * m * 16, (size_t)sb, cudaMemcpyDeviceToDevice,
                                                     st));
                    ++ncomp;
                }
                kb -= NBb;
                NBb = kBlkNB;
            }
            ko = kb;
        }
    }
    if (wc) {
        // ---- window composites (wide windows: k_rq_big + near k_update +
        // k_wsuffix per composite (m = 1: k_wsuffix1), one k_fark per
        // composite) ----
        account_ref_flops(h, sb, n, m, ptop, nb0);  // the reference's stack
        WcShape wsh;
        wc_shape(m, wsh);
        // composite W layout (k_fark: per shift j-major; m = 1, k_farkm:
        // groups of 80 shifts side by side)
        const int64_t wstride = m == 1 ? (int64_t)(kWcWin * nb0 + 1) * kFkmShifts : (int64_t)(kWcWin * nb0 + m) * m;
        static ss::DevMask configured;  // devices configured
        if (!configured.has(h)) {
            SS_CUDA_TRY(h, allow_max_smem(h, k_rq_big));
            configured.set(h);
        }
        while (k >= m + 1) {
            int kw[kWcWin], nbw[kWcWin], g = 0;
            // m = 1: 6 windows per composite (config 3: 8 / 6 / 4 / 2 windows
            // measured 1.36M / 1.42M / 1.40M / 1.29M shifts/s -- the near rows
            // grow with the square of the window count)
#ifndef SS_WC_M1
#define SS_WC_M1 6  // comparison builds vary it
#endif
            const int gmax = m == 1 ? SS_WC_M1 : kWcWin;
            for (int kk = k; kk >= m + 1 && g < gmax; ++g) {
                kw[g] = kk;
                nbw[g] = std::min(nb0, kk - m);
                kk -= nbw[g];
            }
            const int ktop = kw[g - 1], nbtop = nbw[g - 1];
            const int c0 = ktop - m - nbtop;          // first panel column of the composite
            const int K = (k - m) - c0;               // its columns
            const int r0G = ptop + ktop - nbtop;      // first row of its top window
            // m > 1: every window keeps its P (slab b), the composite is built
            // once at the end (k_wsuffix); m = 1 folds window by window
            const int64_t pslab = (int64_t)sb * (nb0 + m) * m;
            int xw[kWcWin];
            for (int b = 0; b < g; ++b) {
                const int nb = nbw[b], r0 = ptop + kw[b] - nb, cw = kw[b] - m - nb, nc = nb + m;
                double2* const Pw = B.P + b * pslab;
                xw[b] = cw - c0;
                int rc = feed_wait(h, feed, st);  // this window's panel columns
                if (rc) return rc;
                cudaEvent_t ev = ss::timing_begin(h, st);
                RqDims rd;
                rd.m = m;
                rd.ptop = ptop;
                rd.nb = nb;
                rd.k = kw[b];
                rd.c0 = cw;
                rd.r0 = r0;
                rd.nc = nc;
                rd.sb = sb;
                rd.A = a.A;
                rd.lda = a.lda;
                rd.shifts = d.shifts;
                rd.LDZ = LDZ;
                if (m == 1)
                    k_rq_m1<<<(sb + 4 * kM1Warps - 1) / (4 * kM1Warps), 32 * kM1Warps, 0, st>>>(rd, B.Z, Pw);
                else
                    k_rq_big<<<sb, kRqBigThreads, rq_big_smem_bytes(nb, m), st>>>(rd, B.Z, Pw);
                SS_LAUNCH_CHECK(h);
                ss::timing_end(h, st, ev, ss::PH_RQ);
                if (r0 > r0G && m == 1) {
                    // near (m = 1): the one-level far kernel with ten shifts per
                    // unit as its columns, rows [r0G, r0)
                    UpdDims u;
                    u.n = n;
                    u.m = m;
                    u.ptop = ptop;
                    u.ident_top = 0;
                    u.A = a.A;
                    u.lda = a.lda;
                    u.T = a.C;
                    u.ldt = a.ldc;
                    u.shifts = d.shifts;
                    u.sb = sb;
                    u.LDZ = LDZ;
                    u.nb = nb;
                    u.mnb = std::min(m, nb);
                    u.r0 = r0;
                    u.c0 = cw;
                    u.nc = nb + 1;
                    u.rlo = r0G;
                    u.nws = 1;
                    u.ksplit = 2;
                    u.S = 1;
                    u.SG = 32;
                    u.pstride = (int64_t)nc;
                    u.p12off = 0;
                    u.p22off = nb;
                    u.zid = 0;
                    u.flags = 0;
                    u.jh = std::max(0, std::min(nb, (nb - 2) / 2));
                    FarShape f{2, 5, 4, 4, 8, 1};
                    f.MSH = true;
                    const int rows = r0 - r0G;
                    const int64_t units = (int64_t)((rows + f.tile() - 1) / f.tile()) * ((sb + 9) / 10);
                    const int grid = (int)std::min<int64_t>(units, h->num_sms);
                    ev = ss::timing_begin(h, st);
                    rc = launch_far(h, f, grid, far_smem_bytes(nb, 10, f.tile(), f.NST), st, u, B.Z, Pw);
                    if (rc) return rc;
                    ss::timing_end(h, st, ev, ss::PH_UPDATE, 8.0 * rows * (double)sb,
                                   8.0 * rows * (double)sb * nb, 4.0 * (double)rows * nb * sb);
                } else if (r0 > r0G) {
                    // near: the composite's rows above this window (generic update)
                    UpdDims u;
                    u.n = n;
                    u.m = m;
                    u.ptop = ptop;
                    u.ident_top = 0;
                    u.A = a.A;
                    u.lda = a.lda;
                    u.T = a.C;
                    u.ldt = a.ldc;
                    u.shifts = d.shifts;
                    u.sb = sb;
                    u.LDZ = LDZ;
                    u.nb = nb;
                    u.mnb = std::min(m, nb);
                    u.r0 = r0;
                    u.c0 = cw;
                    u.nc = nc;
                    u.rlo = r0G;
                    u.pstride = (int64_t)nc * m;
                    u.p12off = 0;
                    u.p22off = (int64_t)nb * m;
                    u.zid = 0;
                    u.flags = 0;
                    u.nws = nws;
                    u.ksplit = (tile.exact && 64 * nws <= 320) ? 2 : 1;
                    u.jh = std::max(0, std::min(nb, (nb - 2 * m) / 2));
                    u.S = std::max(1, 8 / (nws * u.ksplit));
                    const size_t two_per_sm = h->smem_optin / 2 - 1024;
                    while (u.S > 1 && upd_smem_bytes(nb, m, u.S) > two_per_sm) u.S--;
                    u.SG = u.S * 4;
                    const int rows = r0 - r0G;
                    dim3 gu((unsigned)((rows + kUpdRows - 1) / kUpdRows), (unsigned)((sb + u.SG - 1) / u.SG));
                    ev = ss::timing_begin(h, st);
                    rc = launch_update(h, tile, gu, 32 * u.S * nws * u.ksplit, upd_smem_bytes(nb, m, u.S), st, u,
                                       B.Z, B.Z, Pw);
                    if (rc) return rc;
                    ss::timing_end(h, st, ev, ss::PH_UPDATE, 8.0 * rows * m * m * (double)sb,
                                   8.0 * rows * (double)sb * m * nb, 4.0 * m * (double)rows * nb * sb);
                }
            }
            if (m == 1) {
                cudaEvent_t ev = ss::timing_begin(h, st);
                Wsuf1Args wa;
                wa.g = g;
                wa.K = K;
                wa.sb = sb;
                for (int b = 0; b < g; ++b) {
                    wa.x[b] = xw[b];
                    wa.nb[b] = nbw[b];
                }
                wa.P = B.P;
                wa.slab = pslab;
                wa.gstride = wstride;
                wa.W = B.W;
                const int64_t tot = (int64_t)(K + 1) * kFkmShifts * ((sb + kFkmShifts - 1) / kFkmShifts);
                const int blocks = (int)std::min<int64_t>((tot + 255) / 256, 8 * (int64_t)h->num_sms);
                k_wsuffix1<<<blocks, 256, 0, st>>>(wa);
                SS_LAUNCH_CHECK(h);
                ss::timing_end(h, st, ev, ss::PH_BATCHED_GEMM);
            } else {
                cudaEvent_t ev = ss::timing_begin(h, st);
                int rc = ss::wsuffix(h, st, sb, g, xw, nbw, m, m, K, B.P, pslab, B.W, wstride);
                if (rc) return rc;
                ss::timing_end(h, st, ev, ss::PH_BATCHED_GEMM);
            }
            // far rows [0, r0G): one K-streamed pass over the composite
            const int rows = r0G;
            if (rows > 0) {
                FarKDims fk;
                fk.m = m;
                fk.ptop = ptop;
                fk.ident_top = 0;
                fk.A = a.A;
                fk.lda = a.lda;
                fk.T = a.C;
                fk.ldt = a.ldc;
                fk.shifts = d.shifts;
                fk.sb = sb;
                fk.LDZ = LDZ;
                fk.r0 = r0G;
                fk.rlo = 0;
                fk.c0 = c0;
                fk.K = K;
                fk.mnb = std::min(m, K);
                fk.wstride = wstride;
                fk.woff = 0;
                fk.nk = (K + kFkKC - 1) / kFkKC;
                fk.jz = wc_jz(m);
                fk.nz = (m + fk.jz - 1) / fk.jz;
                fk.ntiles = (rows + kFkTile - 1) / kFkTile;
                fk.pan = B.pan;
                cudaEvent_t ev = ss::timing_begin(h, st);
                pack_panel(fk, B.pan, st);
                SS_LAUNCH_CHECK(h);
                ss::timing_end(h, st, ev, ss::PH_OUTER_GEMM);
                const int64_t units = (int64_t)fk.ntiles * ((sb + wsh.S - 1) / wsh.S);
                fk.spl = units >= 8 * (int64_t)h->num_sms ? 4 : 1;
                const int grid = (int)std::max<int64_t>(
                    fk.spl, std::min<int64_t>(units, h->num_sms) / fk.spl * fk.spl);
                double nnz = (double)std::min(rows, ptop) * K;  // Chat rows dense
                if (rows > ptop) nnz += (double)(rows - ptop) * K;
                ev = ss::timing_begin(h, st);
                int rc = m == 1 ? launch_farkm(h, grid, st, fk, B.Z, B.W) : launch_wc_far(h, m, grid, st, fk, B.Z, B.W);
                if (rc) return rc;
                ss::timing_end(h, st, ev, ss::PH_UPDATE, 8.0 * rows * m * m * (double)sb,
                               8.0 * rows * (double)sb * m * K, 4.0 * m * nnz * sb);
            }
            k = ktop - nbtop;
        }
    }
    while (k >= m + 1) {
        Step s;
        s.k = k;
        s.nb = std::min(nb0, k - m);
        s.mnb = std::min(m, s.nb);
        s.r0 = ptop + k - s.nb;
        s.c0 = k - m - s.nb;
        s.nc = s.nb + m;
        s.lmp = 0;
        const ss::Sched* sc = ss::get_sched(h, s.nb, s.nc);
        if (!sc) return ss::set_err(h, SS_ENOMEM, "schedule allocation failed");
        s.steps = sc->steps;
        s.rots = sc->rots;
        s.rot = sc->d_rot;
        s.joff = sc->d_job_off;
        // ---- block RQ -> P (nc x m per shift, j-major) ----
        {
            int rc = feed_wait(h, feed, st);  // this window's panel columns
            if (rc) return rc;
        }
        cudaEvent_t ev = ss::timing_begin(h, st);
        if (use_house) {
            // one warp per shift: row-Householder block RQ (ss_rq_house.cuh)
            RqDims rd;
            rd.m = m;
            rd.ptop = ptop;
            rd.nb = s.nb;
            rd.k = s.k;
            rd.c0 = s.c0;
            rd.r0 = s.r0;
            rd.nc = s.nc;
            rd.sb = sb;
            rd.A = a.A;
            rd.lda = a.lda;
            rd.shifts = d.shifts;
            rd.LDZ = LDZ;
            const size_t sm = rqh_warp_smem(s.nb, m);
            if (m == 1 && s.nb <= 64 && !getenv("SS_RQ_M1_OFF"))
                k_rq_m1<<<(sb + 4 * kM1Warps - 1) / (4 * kM1Warps), 32 * kM1Warps, 0, st>>>(rd, B.Z, B.P);
            else if (m == 1) k_rq_house<2, 2><<<sb, 32, sm, st>>>(rd, B.Z, B.P);
            else if (m == 5) k_rq_house<6, 6><<<sb, 32, sm, st>>>(rd, B.Z, B.P);
            else if (m == 10) k_rq_house<11, 11><<<sb, 32, sm, st>>>(rd, B.Z, B.P);
            else if (m == 20) k_rq_house<21, 21><<<sb, 32, sm, st>>>(rd, B.Z, B.P);
            else if (m + 1 <= 2) k_rq_house<2><<<sb, 32, sm, st>>>(rd, B.Z, B.P);
            else if (m + 1 <= 4) k_rq_house<4><<<sb, 32, sm, st>>>(rd, B.Z, B.P);
            else if (m + 1 <= 8) k_rq_house<8><<<sb, 32, sm, st>>>(rd, B.Z, B.P);
            else if (m + 1 <= 16) k_rq_house<16><<<sb, 32, sm, st>>>(rd, B.Z, B.P);
            else k_rq_house<32><<<sb, 32, sm, st>>>(rd, B.Z, B.P);
        } else if (rq_big(m)) {
            // m + 1 > 32: Householder RQ with the windows in shared memory
            static ss::DevMask configured;  // devices configured
            if (!configured.has(h)) {
                SS_CUDA_TRY(h, allow_max_smem(h, k_rq_big));
                configured.set(h);
            }
            RqDims rd;
            rd.m = m;
            rd.ptop = ptop;
            rd.nb = s.nb;
            rd.k = s.k;
            rd.c0 = s.c0;
            rd.r0 = s.r0;
            rd.nc = s.nc;
            rd.sb = sb;
            rd.A = a.A;
            rd.lda = a.lda;
            rd.shifts = d.shifts;
            rd.LDZ = LDZ;
            k_rq_big<<<sb, kRqBigThreads, rq_big_smem_bytes(s.nb, m), st>>>(rd, B.Z, B.P);
        } else {
            // the reference's scheduled Givens batch: one warp per concurrent
            // rotation (<= 16 warps), rotation parameters in registers
            const size_t smem_rq = rq_smem_bytes(s.nb, m, s.steps, s.rots);
            const int nw = std::max(1, std::min(sc->max_job, 16));
            int per_warp = 0;
            for (int t = 0; t < sc->steps; ++t) {
                const int J = sc->job_off[t + 1] - sc->job_off[t];
                per_warp += (J + nw - 1) / nw;
            }
            const int slots = (per_warp + 31) / 32;
            if (slots <= 1) k_rq<1><<<sb, 32 * nw, smem_rq, st>>>(d, s, B.Z, B.P);
            else if (slots <= 2) k_rq<2><<<sb, 32 * nw, smem_rq, st>>>(d, s, B.Z, B.P);
            else if (slots <= 4) k_rq<4><<<sb, 32 * nw, smem_rq, st>>>(d, s, B.Z, B.P);
            else if (slots <= 8) k_rq<8><<<sb, 32 * nw, smem_rq, st>>>(d, s, B.Z, B.P);
            else return ss::set_err(h, SS_EARG, "window block too large for the register rotation store");
        }
        SS_LAUNCH_CHECK(h);
        ss::timing_end(h, st, ev, ss::PH_RQ);
        // ---- window update: S shifts per chunk, one warp per (shift, column
        // group); smem sized for two resident CTAs per SM when it fits ----
        UpdDims u;
        u.n = n;
        u.m = m;
        u.ptop = ptop;
        u.ident_top = d.ident_top;
        u.A = a.A;
        u.lda = a.lda;
        u.T = a.C;
        u.ldt = a.ldc;
        u.shifts = d.shifts;
        u.sb = sb;
        u.LDZ = LDZ;
        u.nb = s.nb;
        u.mnb = s.mnb;
        u.r0 = s.r0;
        u.c0 = s.c0;
        u.nc = s.nc;
        u.rlo = a.mode == 1 ? s.c0 : 0;
        u.pstride = (int64_t)s.nc * m;
        u.p12off = 0;
        u.p22off = (int64_t)s.nb * m;
        u.zid = 0;
        u.flags = 0;
        u.nws = nws;
        // a warp pair splits the panel K range of one (shift, column block) when
        // one block covers all m columns: twice the warps on the same staging
        // (also for several column blocks per shift when the block RQ is the
        // wide-window one: 2 nws warps per shift, SS_UPD_KSPLIT1=1 disables)
        u.ksplit = ((nws == 1 && tile.exact) || (nws > 1 && tile.exact && rq_big(m) && 64 * nws <= 320))
                       ? 2
                       : 1;  // scratch = the shift's m x 64 Z2 stage
        u.jh = std::max(0, std::min(s.nb, (s.nb - 2 * m) / 2));
        u.S = std::max(1, 8 / (nws * u.ksplit));
        const size_t two_per_sm = h->smem_optin / 2 - 1024;
        while (u.S > 1 && upd_smem_bytes(s.nb, m, u.S) > two_per_sm) u.S--;
        u.SG = u.S * 4;
        const int rows = s.r0 - u.rlo;
        dim3 g((unsigned)((rows + kUpdRows - 1) / kUpdRows), (unsigned)((sb + u.SG - 1) / u.SG));
        const size_t smem_u = upd_smem_bytes(s.nb, m, u.S);
        // reference flop accounting (batched.py:58-61, solvers.py:194-199)
        double rq_fl = 0.0;
        for (int qq = 0; qq < sc->rots; ++qq) rq_fl += 20.0 * ((sc->rot[qq] & 0xffu) + s.nc) + 16.0;
        h->flops[ss::PH_RQ] += rq_fl * sb;
        const double fl_b = (double)sb * (8.0 * s.r0 * m * m + 8.0 * s.mnb * m);
        const double fl_o = 8.0 * s.r0 * ((double)sb * m) * s.nb;
        h->flops[ss::PH_BATCHED_GEMM] += fl_b;
        h->flops[ss::PH_OUTER_GEMM] += fl_o;
        // algorithmic flops of this launch: every structural
        // nonzero of the panel rows it updates meets m complex columns once
        const double nnz =
            (a.mode == 0 ? (double)a.p * s.nb : (double)s.nb) + (double)(k - s.nb) * s.nb;
        const double fl_alg = 4.0 * m * nnz * sb;
        ev = ss::timing_begin(h, st);
        int rc;
        const bool ws = nws == 1 && tile.exact && tile.G * tile.C == m && m != 1 &&
                        ws_smem_bytes(s.nb, m) + 1024 <= h->smem_optin;
        if (ws) {
            // warp-specialised pipeline: 1 producer + 4 consumer pairs, SG shifts per CTA
            u.SG = 32;
            // half 0 also carries the Z2 x P22 part (2 panel columns' worth of
            // DFMA per column of m) and the epilogue: give it fewer panel columns
            u.jh = std::max(0, std::min(s.nb, (s.nb - 2 * m) / 2 - 1));
            dim3 gw((unsigned)((rows + kUpdRows - 1) / kUpdRows), (unsigned)((sb + u.SG - 1) / u.SG));
            rc = launch_update_ws(h, tile, gw, ws_smem_bytes(s.nb, m), st, u, B.Z, B.Z,
                                  B.P);
        } else if (m == 1 && far_smem_bytes(s.nb, 10, 64, 8) + 1024 <= h->smem_optin) {
            // m = 1: ten shifts per unit as the ten columns of the m = 10 tile
            FarShape f{2, 5, 4, 4, 8, 1};
            f.MSH = true;
            u.pstride = (int64_t)s.nc;  // nb + 1 complex per shift: P12 then the scalar P22
            u.p12off = 0;
            u.p22off = s.nb;
            u.zid = 0;
            u.flags = 0;
            u.jh = std::max(0, std::min(s.nb, (s.nb - 2) / 2));
            const int64_t units = (int64_t)((rows + f.tile() - 1) / f.tile()) * ((sb + 9) / 10);
            const int grid = (int)std::min<int64_t>(units, h->num_sms);
            // the kernel's stage holds 10 "columns" of nc = nb + 1 entries
            UpdDims um = u;
            um.nc = s.nb + 1;
            rc = launch_far(h, f, grid, far_smem_bytes(s.nb, 10, f.tile(), f.NST), st, um, B.Z, B.P);
        } else if (nws == 2 && tile.exact && tile.G == 2 && tile.C == 5 &&
                   far_smem_bytes(s.nb, m, 64, 4) + 1024 <= h->smem_optin) {
            // m = 20: persistent far kernel with two column blocks per unit
            // (one group of two pairs shares the unit's stage)
            const FarShape f{2, 5, 4, 4, 4, 2};
            u.pstride = (int64_t)s.nc * m;
            u.p12off = 0;
            u.p22off = (int64_t)s.nb * m;
            u.zid = 0;
            u.flags = 0;
            u.SG = 32;
            u.jh = std::max(0, std::min(s.nb, (s.nb - 2 * m) / 2 - 1));
            const int64_t units = (int64_t)((rows + f.tile() - 1) / f.tile()) * sb;
            const int grid = (int)std::min<int64_t>(units, h->num_sms);
            rc = launch_far(h, f, grid, far_smem_bytes(s.nb, m, f.tile(), f.NST), st, u, B.Z, B.P);
        } else {
            rc = launch_update(h, tile, g, 32 * u.S * nws * u.ksplit, smem_u, st, u, B.Z,
                               B.Z, B.P);
        }
        if (rc) return rc;
        ss::timing_end(h, st, ev, ss::PH_UPDATE, fl_b, fl_o, fl_alg);
        k -= s.nb;
    }
    HeadOut ho;
    ho.mode = a.mode;
    ho.B = a.B;
    ho.ldb = a.ldb;
    ho.bd = a.bd ? a.bd + lo * a.ldbd : nullptr;
    ho.ldbd = a.ldbd;
    ho.rtol = rtol;
    ho.scal = h->d_scal;
    ho.out = a.mode == 0 ? a.out + lo * m * a.ldo : a.out + lo * a.ldo;
    ho.ldo = a.ldo;
    ho.fail = a.fail + lo;
    ho.ybuf = a.defer ? B.Y : nullptr;
    if (feed.on && feed.fro2_pending) {
        // streamed Ahat: all chunks are in (the last wait came with the last
        // window); the pivot tolerances need ||A||_F and trace(A)
        int rc = ss::fro2_trace(h, n, a.A, a.lda, st);
        if (rc) return rc;
        feed.fro2_pending = false;
    }
    cudaEvent_t evh = ss::timing_begin(h, st);
    const size_t smem_h = (size_t)(2 * m * m + m * (a.mode == 0 ? m : 1)) * 16;
    if (smem_h <= h->smem_optin) {
        ho.l0 = 0;
        ho.gscr = nullptr;
        k_head<<<sb, 128, smem_h, st>>>(d, ho, B.Z);
        SS_LAUNCH_CHECK(h);
    } else {
        // wide m (3 m^2 complex > shared memory): the head matrices of up to
        // `chunk` shifts at a time in global scratch (L2-resident for one wave)
        const size_t per = (size_t)3 * m * m * 16;
        const int chunk = (int)std::max<size_t>(1, std::min<size_t>((size_t)sb, ((size_t)256 << 20) / per));
        int rc = ss::ensure_ws(h, per * chunk, 1);
        if (rc) return rc;
        ho.gscr = (double2*)h->ws2;
        for (int l0 = 0; l0 < sb; l0 += chunk) {
            ho.l0 = l0;
            k_head<<<std::min(chunk, sb - l0), 128, 0, st>>>(d, ho, B.Z);
            SS_LAUNCH_CHECK(h);
        }
    }
    if (a.defer) {
        ExpandArgs e;
        e.n = n;
        e.m = m;
        e.group = a.group;
        e.ncomp = 0;
        for (int ko = n; ko >= m + 1;) {  // composite count (the group loop's)
            const int NB1 = std::min(kBlkNB, ko - m);
            const int g = 1 + std::min(a.group - 1, (ko - NB1 - m) / kBlkNB);
            ko -= (g - 1) * kBlkNB + NB1;
            ++e.ncomp;
        }
        e.Xh = B.Xh;
        e.xh_stride = B.xh_stride;
        e.W22h = B.W22h;
        e.w22h_stride = B.w22h_stride;
        e.Y = B.Y;
        e.fail = ho.fail;
        e.X = ho.out;
        e.ldx = ho.ldo;
        k_expand<<<sb, 256, (size_t)2 * m * 16 + (size_t)e.ncomp * 8, st>>>(e);
        SS_LAUNCH_CHECK(h);
    }
    ss::timing_end(h, st, evh, ss::PH_TAIL);
    h->flops[ss::PH_TAIL] += a.mode == 0 ? (double)sb * 8.0 * a.p * m * m : (double)sb * 8.0 * n * m;
    return SS_OK;
}


// ---------------------------------------------------------------------------
// Pseudospectrum epilogue (solvers.py:501-530 structured_pseudospectrum_grid
// with two_norm_small): ||G_l||_2 of every p x m block on the device.  One
// 128-thread CTA per shift (persistent over shifts) forms the k x k Gram
// matrix H (k = min(p, m)) and runs parallel two-sided Hermitian Jacobi to
// convergence: per round the k/2 disjoint pairs of a round-robin ordering
// (Brent-Luk) get their rotations from the 2x2 blocks of H, then all
// column updates (disjoint columns), then all row updates (disjoint rows),
// each spread over the CTA; ||G||_2 = sqrt(lambda_max).  H lives in shared
// memory for k <= kPnSmem, else in a per-CTA slot of global scratch (L2).
// Failed shifts give +inf.
// ---------------------------------------------------------------------------
constexpr int kPnThreads = 128;
constexpr int kPnSmem = 96;  // 96 x 97 x 16 B = 149 KB

__host__ __device__ inline int pn_ld(int k) { return k + 1; }
// per-pair arrays (k/2 + 1 pairs) + reduction slots, rounded up so H
// (double2) is 16-byte aligned
__host__ __device__ inline int pn_pairs(int k) { return k / 2 + 1; }
__host__ __device__ inline size_t pnorm_hdr_bytes(int k) {
    return (((size_t)pn_pairs(k) * (16 + 8 + 8 + 4 + 4) + (kPnThreads / 32 + 2) * 8) + 15) & ~(size_t)15;
}

template <bool GLOBAL_H>
__global__ void __launch_bounds__(kPnThreads) k_pnorm(int p, int m, int64_t s, const double2* __restrict__ G,
                                                      int64_t ldg, const int32_t* __restrict__ fail,
                                                      double* __restrict__ norms, double2* __restrict__ scratch) {
    extern __shared__ __align__(16) unsigned char smem[];
    const bool gram_cols = p >= m;  // H = G^H G (m x m) or G G^H (p x p)
    const int k = gram_cols ? m : p, r = gram_cols ? p : m;
    const int kp = k + (k & 1);  // padded with a dummy index when k is odd
    const int np = kp / 2, ld = pn_ld(k);
    const int tid = threadIdx.x;
    // per-pair rotation: e (phase of H[a][b]), cs, sn, the pair (a, b)
    const int npk = pn_pairs(k);
    double2* e_ = reinterpret_cast<double2*>(smem);
    double* cs_ = reinterpret_cast<double*>(e_ + npk);
    double* sn_ = cs_ + npk;
    double* red = sn_ + npk;  // [kPnThreads / 32 + 2]
    int* pa = reinterpret_cast<int*>(red + kPnThreads / 32 + 2);
    int* pb = pa + npk;
    double2* H = GLOBAL_H ? scratch + (int64_t)blockIdx.x * k * ld
                          : reinterpret_cast<double2*>(smem + pnorm_hdr_bytes(k));
    for (int64_t l = blockIdx.x; l < s; l += gridDim.x) {
        __syncthreads();  // H of the previous shift is dead
        if (fail[l] >= 0) {
            if (tid == 0) norms[l] = __longlong_as_double(0x7ff0000000000000ULL);
            continue;
        }
        const double2* Gl = G + l * m * ldg;  // G_l(i, j) = Gl[i + j * ldg]
        double f2 = 0.0;
        for (int u = tid; u < k * k; u += blockDim.x) {
            const int i = u % k, j = u / k;
            double2 acc = cz();
            for (int t = 0; t < r; ++t) {
                const double2 a = gram_cols ? Gl[t + (int64_t)i * ldg] : Gl[i + (int64_t)t * ldg];
                const double2 b = gram_cols ? Gl[t + (int64_t)j * ldg] : Gl[j + (int64_t)t * ldg];
                // gram_cols: conj(G_ti) G_tj ; else G_it conj(G_jt)
                const double2 x = gram_cols ? make_double2(a.x, -a.y) : a;
                const double2 y = gram_cols ? b : make_double2(b.x, -b.y);
                acc = cfma(x, y, acc);
            }
            H[i * ld + j] = acc;
            f2 = fma(acc.x, acc.x, fma(acc.y, acc.y, f2));
        }
        // block sum helper (deterministic order)
        auto bsum = [&](double v) -> double {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            __syncthreads();
            if ((tid & 31) == 0) red[tid >> 5] = v;
            __syncthreads();
            double t = 0.0;
            for (int w = 0; w < kPnThreads / 32; ++w) t += red[w];
            return t;
        };
        const double fro2 = bsum(f2);
        for (int sweep = 0; sweep < 40 && k > 1; ++sweep) {
            double o = 0.0;
            for (int u = tid; u < k * k; u += blockDim.x) {
                const int i = u % k, j = u / k;
                if (i < j) o = fma(H[i * ld + j].x, H[i * ld + j].x, fma(H[i * ld + j].y, H[i * ld + j].y, o));
            }
            const double off = bsum(o);
            if (off <= 1e-32 * fro2 || off == 0.0) break;
            for (int rd = 0; rd < kp - 1; ++rd) {
                // round-robin pairs: (rd, kp - 1) and ((rd + i), (rd - i)) mod (kp - 1)
                for (int i = tid; i < np; i += blockDim.x) {
                    int a = i == 0 ? rd : (rd + i) % (kp - 1);
                    int b = i == 0 ? kp - 1 : (rd - i + kp - 1) % (kp - 1);
                    if (a > b) { const int t = a; a = b; b = t; }
                    double cs = 1.0, sn = 0.0;
                    double2 e = make_double2(1.0, 0.0);
                    if (b < k) {
                        const double2 c = H[a * ld + b];
                        const double ac = hypot(c.x, c.y);
                        if (ac != 0.0) {
                            e = make_double2(c.x / ac, c.y / ac);
                            const double ha = H[a * ld + a].x, hb = H[b * ld + b].x;
                            const double tau = (hb - ha) / (2.0 * ac);
                            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                            cs = 1.0 / sqrt(1.0 + t * t);
                            sn = t * cs;
                        }
                    }
                    cs_[i] = cs;
                    sn_[i] = sn;
                    e_[i] = e;
                    pa[i] = a;
                    pb[i] = (b < k && sn != 0.0) ? b : -1;  // -1: no rotation
                }
                __syncthreads();
                // columns: H V with V_aa = cs, V_ab = sn, V_ba = -sn conj(e), V_bb = cs conj(e)
                for (int u = tid; u < np * k; u += blockDim.x) {
                    const int i = u / k, row = u - i * k;
                    const int b = pb[i];
                    if (b < 0) continue;
                    const int a = pa[i];
                    const double cs = cs_[i], sn = sn_[i];
                    const double2 ce = make_double2(e_[i].x, -e_[i].y);
                    const double2 x = H[row * ld + a], y = cmul(H[row * ld + b], ce);
                    H[row * ld + a] = make_double2(cs * x.x - sn * y.x, cs * x.y - sn * y.y);
                    H[row * ld + b] = make_double2(sn * x.x + cs * y.x, sn * x.y + cs * y.y);
                }
                __syncthreads();
                // rows: V^H (H V)
                for (int u = tid; u < np * k; u += blockDim.x) {
                    const int i = u / k, col = u - i * k;
                    const int b = pb[i];
                    if (b < 0) continue;
                    const int a = pa[i];
                    const double cs = cs_[i], sn = sn_[i];
                    const double2 e = e_[i];
                    const double2 x = H[a * ld + col], y = cmul(H[b * ld + col], e);
                    H[a * ld + col] = make_double2(cs * x.x - sn * y.x, cs * x.y - sn * y.y);
                    H[b * ld + col] = make_double2(sn * x.x + cs * y.x, sn * x.y + cs * y.y);
                }
                __syncthreads();
                // the 2x2 blocks are diagonal now: exact zeros, real diagonals
                for (int i = tid; i < np; i += blockDim.x) {
                    const int b = pb[i];
                    if (b < 0) continue;
                    const int a = pa[i];
                    H[a * ld + b] = H[b * ld + a] = cz();
                    H[a * ld + a].y = 0.0;
                    H[b * ld + b].y = 0.0;
                }
                __syncthreads();
            }
        }
        __syncthreads();
        if (tid == 0) {
            double lmax = 0.0;
            for (int i = 0; i < k; ++i) lmax = fmax(lmax, H[i * ld + i].x);
            norms[l] = sqrt(lmax);
        }
    }
}

__host__ inline size_t pnorm_smem(int k, bool global_h) {
    size_t b = pnorm_hdr_bytes(k);
    if (!global_h) b += (size_t)k * pn_ld(k) * 16;
    return b;
}

}  // namespace

namespace ss {
// ||A||_F^2 and trace(A) into h->d_scal[0:2] (the per-shift singularity
// thresholds, solvers.py:104-110), deterministic two-pass reduction.
int fro2_trace(ss_handle* h, int n, const double* A, int64_t lda, cudaStream_t st) {
    const int parts = std::min(4 * h->num_sms, std::max(n, 1));
    int rc = ss::ensure_ws(h, 1 << 20, 1);
    if (rc) return rc;
    double* part = (double*)h->ws2;
    if (parts * 2 * sizeof(double) > h->ws2_bytes) return ss::set_err(h, SS_EARG, "scratch");
    k_fro2_trace_part<<<parts, 256, 0, st>>>(n, A, lda, part);
    SS_LAUNCH_CHECK(h);
    k_fro2_trace_final<<<1, 32, 0, st>>>(parts, part, h->d_scal);
    SS_LAUNCH_CHECK(h);
    return SS_OK;
}
}  // namespace ss

namespace {

int run_sweep(ss_handle* h, const SweepArgs& a_in, cudaStream_t st) {
    SweepArgs a = a_in;
    const int n = a.n, m = a.m;
    if (a.s == 0) return SS_OK;
    ss::DevGuard dg(h->device);
    SS_CUDA_TRY(h, dg.err);
    // NaN selects the reference default 1e3 n eps (solvers.py:95-97); any other
    // value is used as given (0: only exactly-zero pivots fail, solvers.py:227)
    const double rtol = std::isnan(a.rtol) ? 1e3 * n * 2.220446049250313e-16 : a.rtol;
    const int nb0_req = max_nb_for(h, m, std::max(1, std::min(a.nb, std::max(n - m, 1))));
    if (nb0_req < 1) return ss::set_err(h, SS_EARG, "m too large: the window does not fit shared memory");

    static ss::DevMask attrs;  // devices configured
    if (!attrs.has(h)) {
        SS_CUDA_TRY(h, allow_max_smem(h, k_rq<1>));
        SS_CUDA_TRY(h, allow_max_smem(h, k_rq<2>));
        SS_CUDA_TRY(h, allow_max_smem(h, k_rq<4>));
        SS_CUDA_TRY(h, allow_max_smem(h, k_rq<8>));
        SS_CUDA_TRY(h, allow_max_smem(h, k_rq_house<2>));
        SS_CUDA_TRY(h, allow_max_smem(h, k_rq_house<4>));
        SS_CUDA_TRY(h, allow_max_smem(h, k_rq_house<8>));
        SS_CUDA_TRY(h, allow_max_smem(h, k_rq_house<16>));
        SS_CUDA_TRY(h, allow_max_smem(h, k_rq_house<32>));
        SS_CUDA_TRY(h, allow_max_smem(h, k_rq_house<2, 2>));
        SS_CUDA_TRY(h, allow_max_smem(h, k_rq_house<6, 6>));
        SS_CUDA_TRY(h, allow_max_smem(h, k_rq_house<11, 11>));
        SS_CUDA_TRY(h, allow_max_smem(h, k_rq_house<21, 21>));
        SS_CUDA_TRY(h, allow_max_smem(h, k_head));
        attrs.set(h);
    }
    // block RQ flavour: row Householder (one warp per shift) unless m+1 > 32
    // or SS_BLOCK_RQ=givens selects the reference's scheduled Givens batch
    const char* rqenv = getenv("SS_BLOCK_RQ");
    const bool use_house = (m + 1 <= 32) && !(rqenv && strcmp(rqenv, "givens") == 0);
    const UpdTile tile = pick_tile(m);
    // the Householder block RQ maps one block row to one thread of two warps
    int nb_big = kRqBigNb;
    // the generic update stages the whole (nb + m) x m P per shift: the
    // widest window whose update and RQ fit one SM's shared memory
    while (nb_big > 8 && (upd_smem_bytes(nb_big, m, 1) + 1024 > h->smem_optin ||
                          rq_big_smem_bytes(nb_big, m) + 1024 > h->smem_optin))
        nb_big -= 8;
    int nb0 = use_house ? std::min(nb0_req, 64) : (rq_big(m) ? nb_big : nb0_req);

    // two-level sweep (ss_block.cuh) when the fused block kernel and the
    // warp-specialised far update cover m; SS_ONE_LEVEL=1 forces the
    // per-window sweep
    // (m = 20: the far passes run k_far with two column blocks per unit)
    const bool two_level = use_house && block_supported(m) && tile.exact &&
                           (tile.G * tile.C == m || (m == 20 && tile.G == 2 && tile.C == 5)) &&
                           !getenv("SS_ONE_LEVEL") &&
                           far_smem_bytes(64, m, 64, m == 20 ? 4 : 8) + 1024 <= h->smem_optin;
    // reduced solve on the two-level sweep: identity top deferred (k_expand);
    // SS_NO_DEFER=1 sweeps the identity rows as the reference does
    // wide windows (m = 40 / 50 / 60, transfer function): window composites
    // with one K-streamed far pass per kWcWin windows (SS_ONE_LEVEL=1: per window)
    WcShape wsh;
    const bool wc = !two_level && a.mode == 0 && (rq_big(m) || (m == 1 && use_house)) && wc_shape(m, wsh) &&
                    !getenv("SS_ONE_LEVEL") && !(m == 1 && getenv("SS_RQ_M1_OFF")) &&
                    wc_far_smem(m) <= h->smem_optin && wsuf_smem(m, kWcNb) <= h->smem_optin &&
                    kWcWin * kWcNb <= 4 * kBlkNB;
    if (wc) nb0 = std::min(nb0, kWcNb);
    a.defer = a.mode == 1 && two_level && !getenv("SS_NO_DEFER");
    const int mode_far = a.defer ? 0 : a.mode;
    a.group = two_level ? two_level_group(h, m, mode_far) : 1;
    const int ptop = a.mode == 0 ? a.p : (a.defer ? 0 : n);
    const int64_t LDZ = ((int64_t)(ptop + n) + 7) & ~(int64_t)7;
    int ncomp = 0;
    for (int ko = n; a.defer && ko >= m + 1; ++ncomp) {
        const int NB1 = std::min(kBlkNB, ko - m);
        ko -= (1 + std::min(a.group - 1, (ko - NB1 - m) / kBlkNB) - 1) * kBlkNB + NB1;
    }
    const int64_t xh_stride = a.defer ? (int64_t)n * m : 0;
    const int64_t w22h_stride = a.defer ? (int64_t)ncomp * m * m : 0;
    const int64_t y_stride = a.defer ? m : 0;  // the head's y for k_expand
    // fro2 / trace for the per-shift singularity thresholds (streamed Ahat:
    // after the last chunk, just before the first head)
    Feed feed;
    if (a.A_host) {
        std::vector<std::pair<int, int>> chunks;
        sweep_chunks(n, m, two_level, nb0, chunks);
        if (!h->copy_stream)
            SS_CUDA_TRY(h, cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
        while (h->chunk_ev.size() < chunks.size()) {
            cudaEvent_t e;
            SS_CUDA_TRY(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            h->chunk_ev.push_back(e);
        }
        // the destination may still be read by earlier work on st
        SS_CUDA_TRY(h, cudaEventRecord(h->ev_a, st));
        SS_CUDA_TRY(h, cudaStreamWaitEvent(h->copy_stream, h->ev_a, 0));
        for (size_t c = 0; c < chunks.size(); ++c) {
            const int c0 = chunks[c].first, c1 = chunks[c].second;
            if (c1 > c0)
                SS_CUDA_TRY(h, cudaMemcpy2DAsync(const_cast<double*>(a.A) + (int64_t)c0 * a.lda,
                                                 (size_t)a.lda * 8, a.A_host + (int64_t)c0 * a.lda_host,
                                                 (size_t)a.lda_host * 8, (size_t)n * 8, (size_t)(c1 - c0),
                                                 cudaMemcpyHostToDevice, h->copy_stream));
            SS_CUDA_TRY(h, cudaEventRecord(h->chunk_ev[c], h->copy_stream));
        }
        feed.on = true;
        feed.fro2_pending = true;
        feed.count = (int)chunks.size();
    } else {
        int rc = ss::fro2_trace(h, n, a.A, a.lda, st);
        if (rc) return rc;
    }

    // batch size from memory: the window state + P (or W) per shift
    const int ncmax = nb0 + m;
    const int64_t wc_stride = wc ? (int64_t)(kWcWin * nb0 + m) * m : 0;  // composite W per shift
    const size_t wc_slack = m == 1 ? (size_t)kFkmShifts * wc_stride * 16 : 0;  // last group of 80 shifts
    const int wc_slabs = wc ? kWcWin : 1;  // window P kept per composite (k_wsuffix / k_wsuffix1)
    const int64_t pst = two_level ? (int64_t)(a.group * kBlkNB + m) * m : (int64_t)wc_slabs * ncmax * m + wc_stride;
    const size_t per_shift = (size_t)LDZ * m * 16 + (size_t)pst * 16 + 64 +
                             (size_t)(xh_stride + w22h_stride + y_stride) * 16;
    int64_t sb_max = std::min<int64_t>(a.batch > 0 ? a.batch : a.s, a.s);
    if (per_shift * (size_t)sb_max + 256 > h->ws_bytes) {
        // only when the workspace has to grow: cudaMemGetInfo is a driver
        // query measured at 1-80 ms of host time on a busy box, which stalls
        // the enqueue (and the GPU behind it)
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        const size_t cap = std::max<size_t>(fr / 2 + h->ws_bytes / 2, per_shift);
        sb_max = std::min<int64_t>(sb_max, (int64_t)(cap / per_shift));
        sb_max = std::max<int64_t>(sb_max, 1);
    }
    sb_max = std::min<int64_t>(sb_max, a.s);
    {
        int rc = ss::ensure_ws(h, per_shift * (size_t)sb_max + 256 + wc_slack, 0);
        if (rc) return rc;
    }
    double2* Z0 = (double2*)h->ws;
    double2* P0 = Z0 + (size_t)sb_max * m * LDZ;
    double2* Xh0 = P0 + (size_t)sb_max * pst;
    double2* W22h0 = Xh0 + (size_t)sb_max * xh_stride;
    double2* Y0 = W22h0 + (size_t)sb_max * w22h_stride;
    double* pan = nullptr;  // k_fark's packed panel, after the 1 MB scratch of fro2_trace
    // (wide-window composites run two halves of a batch on two streams: one
    // packed panel per half)
    const size_t pan_elems = fark_pan_bytes(n, ptop) / 8;
    if ((two_level && fark_supported(h, m, mode_far)) || wc) {
        int rc = ss::ensure_ws(h, (1u << 20) + (wc ? 2 : 1) * pan_elems * 8, 1);
        if (rc) return rc;
        pan = reinterpret_cast<double*>(static_cast<char*>(h->ws2) + (1u << 20));
    }

    // Independent halves of a batch on two streams: the latency-bound block
    // RQ of one half overlaps the FP64-bound window update of the other.
    // (the persistent far-row kernel -- two-level sweep, and the one-level
    // m = 20 update -- owns every SM, so it runs on one stream; otherwise
    // two halves overlap)
    const bool far_m20 = !two_level && tile.exact && tile.G == 2 && tile.C == 5 &&
                         (m + tile.G * tile.C - 1) / (tile.G * tile.C) == 2;
    const bool far_m1 = !two_level && m == 1;
    int NS = (two_level || far_m20 || far_m1) ? 1 : 2;
    if (sb_max < 64 || feed.on) NS = 1;
    cudaStream_t streams[2] = {st, st};
    if (NS == 2) {
        if (!h->aux_stream) SS_CUDA_TRY(h, cudaStreamCreateWithFlags(&h->aux_stream, cudaStreamNonBlocking));
        streams[1] = h->aux_stream;
        SS_CUDA_TRY(h, cudaEventRecord(h->ev_a, st));
        SS_CUDA_TRY(h, cudaStreamWaitEvent(streams[1], h->ev_a, 0));
    }
    for (int64_t lo = 0; lo < a.s; lo += sb_max) {
        const int sb = (int)std::min<int64_t>(sb_max, a.s - lo);
        const int parts = (NS == 2 && sb >= 64) ? 2 : 1;
        int off = 0;
        for (int p = 0; p < parts; ++p) {
            const int cnt = sb / parts + (p < sb % parts ? 1 : 0);
            PartBufs B;
            B.Z = Z0 + (size_t)off * m * LDZ;
            B.P = P0 + (size_t)off * pst;
            B.pan = pan && wc ? pan + (size_t)p * pan_elems : pan;
            if (wc) B.W = B.P + (size_t)wc_slabs * cnt * ncmax * m;  // after the parts' window P
            if (a.defer) {
                B.Xh = Xh0 + (size_t)off * xh_stride;
                B.W22h = W22h0 + (size_t)off * w22h_stride;
                B.Y = Y0 + (size_t)off * m;
                B.xh_stride = xh_stride;
                B.w22h_stride = w22h_stride;
            }
            int rc = enqueue_part(h, a, lo + off, cnt, B, nb0, LDZ, rtol, use_house, tile,
                                  two_level, wc, streams[p], feed);
            if (rc) return rc;
            off += cnt;
        }
        if (NS == 2 && lo + sb_max < a.s) {
            // the next batch reuses both parts' buffers: join before reuse
            SS_CUDA_TRY(h, cudaEventRecord(h->ev_b, streams[1]));
            SS_CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_b, 0));
            SS_CUDA_TRY(h, cudaEventRecord(h->ev_a, st));
            SS_CUDA_TRY(h, cudaStreamWaitEvent(streams[1], h->ev_a, 0));
        }
    }
    if (NS == 2) {
        SS_CUDA_TRY(h, cudaEventRecord(h->ev_b, streams[1]));
        SS_CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_b, 0));
    }
    return SS_OK;
}

}  // namespace

namespace ss {
// ---- transposed-sweep composites (ss_lq.cu): far pass ----------
// The far pass's -I rows [rlo, r0) (rlo >= n): their panel row has at most
// one entry (-1 in column i - n), so instead of the dense K-streamed pass:
//   z_i <- z_i W22 - [0 <= i - dlo < K] W12[i - dlo]        (dlo = n + c0)
// One CTA per (row tile, shift): the rows' mc state columns and W22 in
// shared memory; a thread owns 4 rows x 4 columns in registers (rows rg +
// RG r, columns cg + CG c, CG = ceil(mc / 4) column groups, RG = 256 / CG
// row groups: the tile is 4 RG rows, so no thread slot is spent on columns
// past mc): 8 shared loads per 16 complex FMAs.
__host__ __device__ inline int tl_cg(int mc) { return (mc + 3) / 4; }
__host__ __device__ inline int tl_rows(int mc) { return 4 * (256 / tl_cg(mc)); }
__host__ __device__ inline size_t tl_smem(int M, int mc) { return (size_t)(M * M + mc * tl_rows(mc)) * 16; }
__global__ void __launch_bounds__(256) k_tr_lower(int M, int mc, int64_t LDS, double2* __restrict__ S, int rlo,
                                                  int r0, int dlo, int K, const double2* __restrict__ W,
                                                  int64_t wstride) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int CG = tl_cg(mc), RG = 256 / CG, TR = 4 * RG;
    double2* W22 = reinterpret_cast<double2*>(smem);  // M x M
    double2* Zs = W22 + M * M;                         // [mc][TR]
    const int l = blockIdx.y, t = threadIdx.x;
    const int i0 = rlo + blockIdx.x * TR;
    const double2* Wl = W + (int64_t)l * wstride;
    double2* Sl = S + (int64_t)l * M * LDS;
    for (int e = t; e < M * M; e += 256) W22[e] = Wl[(int64_t)K * M + e];
    for (int e = t; e < mc * TR; e += 256) {
        const int j = e / TR, r = e - j * TR;
        Zs[e] = i0 + r < r0 ? Sl[(int64_t)j * LDS + i0 + r] : cz();
    }
    __syncthreads();
    if (t >= RG * CG) return;
    const int rg = t % RG, cg = t / RG;
    double2 acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = cz();
    for (int j = 0; j < mc; ++j) {  // padding columns (>= mc) are zero
        double2 z[4], w[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) z[r] = Zs[j * TR + rg + RG * r];
#pragma unroll
        for (int c = 0; c < 4; ++c) w[c] = cg + CG * c < mc ? W22[j * M + cg + CG * c] : cz();
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[r][c] = cfma(z[r], w[c], acc[r][c]);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int i = i0 + rg + RG * r;
        if (i >= r0) continue;
        const int dd = i - dlo;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int col = cg + CG * c;
            if (col >= mc) continue;
            double2 v = acc[r][c];
            if (dd >= 0 && dd < K) v = csub(v, Wl[(int64_t)dd * M + col]);
            Sl[(int64_t)col * LDS + i] = v;
        }
    }
}

// Split far pass of the transposed composites (m a multiple of 10): the z2
// columns run the K-streamed k_fark at exactly M = m columns, the w column
// (which never feeds z2: W22's w row is e_m) runs k_farkm with 80 shifts per
// unit as its columns; w first takes the old z2's contribution z2 W22[:m, m]
// (k_tr_wprep) and the composite is split into W_z ((K + m) x m per shift)
// and the group-major w column (k_tr_wsplit).
__global__ void __launch_bounds__(256) k_tr_wprep(int m, int64_t LDS, double2* __restrict__ S, int rlo, int r0,
                                                  int K, const double2* __restrict__ W, int64_t wstride) {
    __shared__ double2 wz[64];
    const int l = blockIdx.y, mp = m + 1;
    const double2* Wl = W + (int64_t)l * wstride;
    for (int j = threadIdx.x; j < m; j += blockDim.x) wz[j] = Wl[(int64_t)(K + j) * mp + m];
    __syncthreads();
    const int i = rlo + blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= r0) return;
    double2* Sl = S + (int64_t)l * mp * LDS;
    double2 a0 = Sl[(int64_t)m * LDS + i], a1 = cz();
    int j = 0;
    for (; j + 1 < m; j += 2) {
        a0 = cfma(Sl[(int64_t)j * LDS + i], wz[j], a0);
        a1 = cfma(Sl[(int64_t)(j + 1) * LDS + i], wz[j + 1], a1);
    }
    if (j < m) a0 = cfma(Sl[(int64_t)j * LDS + i], wz[j], a0);
    Sl[(int64_t)m * LDS + i] = cadd(a0, a1);
}

__global__ void __launch_bounds__(256) k_tr_wsplit(int m, int K, int sb, const double2* __restrict__ W,
                                                   int64_t wstride, double2* __restrict__ Wz, int64_t wzstride,
                                                   double2* __restrict__ Ww, int64_t gstride) {
    const int l = blockIdx.y, mp = m + 1;
    const double2* Wl = W + (int64_t)l * wstride;
    double2* Wzl = Wz + (int64_t)l * wzstride;
    const int grp = l / kFkmShifts, q = l - grp * kFkmShifts;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < (K + mp) * mp; e += gridDim.x * blockDim.x) {
        const int r = e / mp, c = e - r * mp;
        if (c < m && r < K + m) Wzl[(int64_t)r * m + c] = Wl[e];                              // W12 / W22 of z2
        else if (c == m && r < K) Ww[grp * gstride + (int64_t)r * kFkmShifts + q] = Wl[e];   // W12 of w
        else if (c == m && r == K + m) Ww[grp * gstride + (int64_t)K * kFkmShifts + q] = Wl[e];  // W22[m][m]
    }
    (void)sb;
}

// the composite W of g windows from their P slabs (k_wsuffix)
int wsuffix(ss_handle* h, cudaStream_t st, int sb, int g, const int* x, const int* nb, int M, int mc, int K,
            const double2* P, int64_t slab, double2* W, int64_t wstride) {
    static ss::DevMask configured;
    if (!configured.has(h)) {
        SS_CUDA_TRY(h, allow_max_smem(h, k_wsuffix));
        configured.set(h);
    }
    if (g > kWsufMax) return ss::set_err(h, SS_EARG, "composite: too many windows");
    WsufArgs a;
    a.g = g;
    a.M = M;
    a.mc = mc;
    a.K = K;
    for (int b = 0; b < g; ++b) {
        a.x[b] = x[b];
        a.nb[b] = nb[b];
    }
    a.P = P;
    a.slab = slab;
    a.W = W;
    a.wstride = wstride;
    int nbmax = 0;
    for (int b = 0; b < g; ++b) nbmax = std::max(nbmax, nb[b]);
    const size_t smem = wsuf_smem(M, nbmax);
    if (M > 64 || smem > h->smem_optin) return ss::set_err(h, SS_EARG, "composite: state too wide");
    k_wsuffix<<<sb, kWsT, smem, st>>>(a);
    SS_LAUNCH_CHECK(h);
    return SS_OK;
}

// state widths the composite far pass supports (M = 10 NCB)
// The transposed sweep's K-streamed passes over M state columns (M = 10 ..
// 60): (shifts per unit, Z-chunk width) and the launch, on k_farkd (DMMA;
// -DSS_FARK_DFMA: k_fark)
static int tr_shape(int M, int& jz) {
    if (kFarkDmma) {
        switch (M) {
            case 10: jz = farkd_jz<1, 4>(); return 4;
            case 20: jz = farkd_jz<2, 4>(); return 4;
            case 30: jz = farkd_jz<3, 2>(); return 2;
            case 40: jz = farkd_jz<4, 2>(); return 2;
            case 50: jz = farkd_jz<5, 1>(); return 1;
            case 60: jz = farkd_jz<6, 1>(); return 1;
            default: return 0;
        }
    }
    switch (M) {
        case 10: jz = fark_jz<1, 8>(); return 8;
        case 20: jz = fark_jz<2, 4>(); return 4;
        case 30: jz = fark_jz<3, 4>(); return 4;
        case 40: jz = fark_jz<4, 2>(); return 2;
        case 50: jz = fark_jz<5, 3>(); return 3;
        case 60: jz = fark_jz<6, 2>(); return 2;
        default: return 0;
    }
}
static int tr_launch(ss_handle* h, int M, int grid, cudaStream_t st, const FarKDims& fk, double2* S,
                     const double2* W) {
    if (kFarkDmma) {
        switch (M) {
            case 10: return launch_farkd<1, 4, kFarkStages, 2, 1>(h, grid, st, fk, S, W);
            case 20: return launch_farkd<2, 4, kFarkStages, 2, 1>(h, grid, st, fk, S, W);
            case 30: return launch_farkd<3, 2, kFarkStages, 4, 1>(h, grid, st, fk, S, W);
            case 40: return launch_farkd<4, 2, 3, 2, 2>(h, grid, st, fk, S, W);
            case 50: return launch_farkd<5, 1, 4, 4, 2>(h, grid, st, fk, S, W);
            default: return launch_farkd<6, 1, 4, 4, 2>(h, grid, st, fk, S, W);
        }
    }
    switch (M) {
        case 10: return launch_fark<1, 8>(h, grid, st, fk, S, W);
        case 20: return launch_fark<2, 4>(h, grid, st, fk, S, W);
        case 30: return launch_fark<3, 4, 2>(h, grid, st, fk, S, W);
        case 40: return launch_fark<4, 2, 3>(h, grid, st, fk, S, W);
        case 50: return launch_fark<5, 3, 2>(h, grid, st, fk, S, W);
        default: return launch_fark<6, 2, 2>(h, grid, st, fk, S, W);
    }
}

bool tr_far_supported(ss_handle* h, int M) {
    switch (M) {
        case 10: return fark_smem_bytes<1, 8, kFarkStages>() <= h->smem_optin;
        case 20: return fark_smem_bytes<2, 4, kFarkStages>() <= h->smem_optin;
        case 30: return (kFarkDmma ? fark_smem_bytes<3, 2, kFarkStages>() : fark_smem_bytes<3, 4, 2>()) <= h->smem_optin;
        case 40: case 50: case 60: return wc_far_smem(M) <= h->smem_optin;
        default: return false;
    }
}

// Far rows [rlo, r0) of the transposed sweep from the composite over panel
// columns [c0, c0 + K) of [A^T; -I]: one K-streamed k_fark pass (packed panel
// from k_pack_panel_tr); the lazy -sigma rows are the first min(m, K) far
// rows (the composite's last columns' diagonal).
int tr_far(ss_handle* h, cudaStream_t st, int n, int m, int M, const double* A, int64_t lda,
           const double2* shifts, int sb, double2* S, int64_t LDS, int rlo, int r0_all, int c0, int K,
           const double2* W, int64_t wstride) {
    // the -I rows first (k_tr_lower), then the dense A^T rows (k_fark)
    if (r0_all > std::max(rlo, n)) {
        static ss::DevMask configured;
        if (!configured.has(h)) {
            SS_CUDA_TRY(h, allow_max_smem(h, k_tr_lower));
            configured.set(h);
        }
        const int lo = std::max(rlo, n), nr = r0_all - lo;
        cudaEvent_t ev = ss::timing_begin(h, st);
        k_tr_lower<<<dim3((unsigned)((nr + tl_rows(m + 1) - 1) / tl_rows(m + 1)), (unsigned)sb), 256,
                     tl_smem(M, m + 1), st>>>(M, m + 1, LDS, S, lo, r0_all, n + c0, K, W, wstride);
        SS_LAUNCH_CHECK(h);
        ss::timing_end(h, st, ev, ss::PH_BATCHED_GEMM);
    }
    const int r0 = std::min(r0_all, n);
    const int rows = r0 - rlo;
    if (rows <= 0) return SS_OK;
    {
        int rc = ss::ensure_ws(h, (1u << 20) + fark_pan_bytes(2 * n, 0), 1);
        if (rc) return rc;
    }
    double* pan = reinterpret_cast<double*>(static_cast<char*>(h->ws2) + (1u << 20));
    FarKDims fk;
    fk.m = M;
    fk.ptop = 0;
    fk.ident_top = 0;
    fk.A = A;
    fk.lda = lda;
    fk.T = nullptr;
    fk.ldt = 0;
    fk.shifts = shifts;
    fk.sb = sb;
    fk.LDZ = LDS;
    fk.r0 = r0;
    fk.rlo = rlo;
    fk.c0 = c0;
    fk.K = K;
    // diagonal entries (c, c) of the composite's columns that fall in the far rows
    fk.lz0 = std::max(rlo, c0);
    fk.lzp = fk.lz0 - c0;
    fk.mnb = std::max(0, c0 + K - fk.lz0);
    fk.lzset = 1;
    fk.n = n;
    fk.wstride = wstride;
    fk.woff = 0;
    fk.nk = (K + kFkKC - 1) / kFkKC;
    fk.ntiles = (rows + kFkTile - 1) / kFkTile;
    fk.pan = pan;
    const int S_ = tr_shape(M, fk.jz);
    if (!S_) return ss::set_err(h, SS_EARG, "transposed composite: unsupported width");
    fk.nz = (M + fk.jz - 1) / fk.jz;
    cudaEvent_t ev = ss::timing_begin(h, st);
    pack_panel_tr(fk, pan, st);
    SS_LAUNCH_CHECK(h);
    ss::timing_end(h, st, ev, ss::PH_OUTER_GEMM);
    const int64_t units = (int64_t)fk.ntiles * ((sb + S_ - 1) / S_);
    fk.spl = units >= 8 * (int64_t)h->num_sms ? 4 : 1;
    const int grid = (int)std::max<int64_t>(fk.spl, std::min<int64_t>(units, h->num_sms) / fk.spl * fk.spl);
    // algorithmic flops: the A^T rows are dense in the panel columns, the -I
    // rows have one entry per column (m + 1 real state columns)
    const int arows = std::max(0, std::min(r0, n) - rlo);
    const double nnz = (double)arows * K + (double)std::min(K, std::max(0, r0 - std::max(rlo, n)));
    ev = ss::timing_begin(h, st);
    int rc = tr_launch(h, M, grid, st, fk, S, W);
    if (rc) return rc;
    ss::timing_end(h, st, ev, ss::PH_UPDATE, 8.0 * rows * M * M * (double)sb, 8.0 * rows * (double)sb * M * K,
                   4.0 * (m + 1) * nnz * sb);
    return SS_OK;
}


int tr_far_split(ss_handle* h, cudaStream_t st, int n, int m, const double* A, int64_t lda,
                 const double2* shifts, int sb, double2* S, int64_t LDS, int rlo, int r0_all, int c0, int K,
                 const double2* W, int64_t wstride, double2* Wz, int64_t wzstride, double2* Ww, int64_t gstride) {
    const int mp = m + 1;
    // the -I rows (state z2 and w, mp columns)
    if (r0_all > std::max(rlo, n)) {
        static ss::DevMask configured;
        if (!configured.has(h)) {
            SS_CUDA_TRY(h, allow_max_smem(h, k_tr_lower));
            configured.set(h);
        }
        const int lo = std::max(rlo, n), nr = r0_all - lo;
        cudaEvent_t ev = ss::timing_begin(h, st);
        k_tr_lower<<<dim3((unsigned)((nr + tl_rows(mp) - 1) / tl_rows(mp)), (unsigned)sb), 256,
                     tl_smem(mp, mp), st>>>(mp, mp, LDS, S, lo, r0_all, n + c0, K, W, wstride);
        SS_LAUNCH_CHECK(h);
        ss::timing_end(h, st, ev, ss::PH_BATCHED_GEMM);
    }
    const int r0 = std::min(r0_all, n), rows = r0 - rlo;
    if (rows <= 0) return SS_OK;
    {
        int rc = ss::ensure_ws(h, (1u << 20) + fark_pan_bytes(2 * n, 0), 1);
        if (rc) return rc;
    }
    double* pan = reinterpret_cast<double*>(static_cast<char*>(h->ws2) + (1u << 20));
    FarKDims fk;
    fk.m = m;
    fk.ptop = 0;
    fk.ident_top = 0;
    fk.A = A;
    fk.lda = lda;
    fk.T = nullptr;
    fk.ldt = 0;
    fk.shifts = shifts;
    fk.sb = sb;
    fk.LDZ = LDS;
    fk.r0 = r0;
    fk.rlo = rlo;
    fk.c0 = c0;
    fk.K = K;
    fk.lz0 = std::max(rlo, c0);
    fk.lzp = fk.lz0 - c0;
    fk.mnb = std::max(0, c0 + K - fk.lz0);
    fk.lzset = 1;
    fk.n = n;
    fk.woff = 0;
    fk.nk = (K + kFkKC - 1) / kFkKC;
    fk.ntiles = (rows + kFkTile - 1) / kFkTile;
    fk.pan = pan;
    fk.zstride = (int64_t)mp * LDS;
    cudaEvent_t ev = ss::timing_begin(h, st);
    // one packed panel for both passes (k_farkmd and k_farkd read the
    // fragment order; -DSS_FARK_DFMA: k_farkm / k_fark the lane-interleaved one)
    pack_panel_tr(fk, pan, st);
    SS_LAUNCH_CHECK(h);
    k_tr_wprep<<<dim3((unsigned)((rows + 255) / 256), (unsigned)sb), 256, 0, st>>>(m, LDS, S, rlo, r0, K, W,
                                                                                   wstride);
    SS_LAUNCH_CHECK(h);
    k_tr_wsplit<<<dim3(8, (unsigned)sb), 256, 0, st>>>(m, K, sb, W, wstride, Wz, wzstride, Ww, gstride);
    SS_LAUNCH_CHECK(h);
    ss::timing_end(h, st, ev, ss::PH_OUTER_GEMM);
    const int arows = rows;
    const double nnz = (double)arows * K;
    // w: 80 shifts per unit as columns
    {
        FarKDims fw = fk;
        fw.wstride = gstride;
        fw.zoff = (int64_t)m * LDS;
        const int64_t units = (int64_t)fw.ntiles * ((sb + kFkmShifts - 1) / kFkmShifts);
        fw.spl = units >= 8 * (int64_t)h->num_sms ? 4 : 1;
        const int grid = (int)std::max<int64_t>(fw.spl, std::min<int64_t>(units, h->num_sms) / fw.spl * fw.spl);
        ev = ss::timing_begin(h, st);
        int rc = launch_farkm(h, grid, st, fw, S, Ww);
        if (rc) return rc;
        ss::timing_end(h, st, ev, ss::PH_UPDATE, 0.0, 8.0 * rows * (double)sb * K, 4.0 * nnz * sb);
    }
    // z2: exact m = 10 NCB columns
    const int S_ = tr_shape(m, fk.jz);
    if (!S_) return ss::set_err(h, SS_EARG, "transposed split far pass: unsupported m");
    fk.nz = (m + fk.jz - 1) / fk.jz;
    fk.wstride = wzstride;
    const int64_t units = (int64_t)fk.ntiles * ((sb + S_ - 1) / S_);
    fk.spl = units >= 8 * (int64_t)h->num_sms ? 4 : 1;
    const int grid = (int)std::max<int64_t>(fk.spl, std::min<int64_t>(units, h->num_sms) / fk.spl * fk.spl);
    ev = ss::timing_begin(h, st);
    int rc = tr_launch(h, m, grid, st, fk, S, Wz);
    if (rc) return rc;
    ss::timing_end(h, st, ev, ss::PH_UPDATE, 8.0 * rows * m * m * (double)sb, 8.0 * rows * (double)sb * m * K,
                   4.0 * m * nnz * sb);
    return SS_OK;
}

bool tr_split_supported(ss_handle* h, int m) {
    return m % 10 == 0 && m <= 60 && tr_far_supported(h, m) && farkm_smem_bytes<4>() <= h->smem_optin;
}
}  // namespace ss

extern "C" {

int ss_tf_eval(ss_handle* h, int n, int m, int p, const double* Ahat, int64_t lda,
               const double* Bhat, int64_t ldb, const double* Chat, int64_t ldc,
               const double* shifts, int64_t s, int nb, int64_t batch, double rtol, double* G,
               int64_t ldg, int32_t* fail_row, void* stream) {
    if (!h) return SS_EARG;
    if (n < 1 || m < 1 || m > n || p < 0 || s < 0)
        return ss::set_err(h, SS_EDIM, "inconsistent controller-Hessenberg form");
    if (lda < n || ldb < m || (p > 0 && ldc < p) || (p > 0 && ldg < p))
        return ss::set_err(h, SS_EDIM, "leading dimension too small");
    if (nb < 1) return ss::set_err(h, SS_EARG, "window block size must be >= 1");
    if (s > 0 && (!Ahat || !Bhat || !shifts || !fail_row || (p > 0 && (!Chat || !G))))
        return ss::set_err(h, SS_EARG, "null pointer");
    SweepArgs a{};
    a.mode = 0;
    a.n = n;
    a.m = m;
    a.p = p;
    a.A = Ahat;
    a.lda = lda;
    a.B = Bhat;
    a.ldb = ldb;
    a.C = Chat;
    a.ldc = ldc > 0 ? ldc : 1;
    a.shifts = (const double2*)shifts;
    a.s = s;
    a.bd = nullptr;
    a.ldbd = 0;
    a.nb = nb;
    a.batch = batch;
    a.rtol = rtol;
    a.out = (double2*)G;
    a.ldo = ldg > 0 ? ldg : 1;
    a.fail = fail_row;
    return run_sweep(h, a, (cudaStream_t)stream);
}

int ss_tf_eval_stream(ss_handle* h, int n, int m, int p, const double* Ahat_host,
                      int64_t lda_host, double* Ahat_dev, int64_t lda_dev, const double* Bhat,
                      int64_t ldb, const double* Chat, int64_t ldc, const double* shifts, int64_t s,
                      int nb, int64_t batch, double rtol, double* G, int64_t ldg, int32_t* fail_row,
                      void* stream) {
    if (!h) return SS_EARG;
    if (n < 1 || m < 1 || m > n || p < 0 || s < 0)
        return ss::set_err(h, SS_EDIM, "inconsistent controller-Hessenberg form");
    if (lda_host < n || lda_dev < n || ldb < m || (p > 0 && ldc < p) || (p > 0 && ldg < p))
        return ss::set_err(h, SS_EDIM, "leading dimension too small");
    if (nb < 1) return ss::set_err(h, SS_EARG, "window block size must be >= 1");
    if (s > 0 && (!Ahat_host || !Ahat_dev || !Bhat || !shifts || !fail_row || (p > 0 && (!Chat || !G))))
        return ss::set_err(h, SS_EARG, "null pointer");
    SweepArgs a{};
    a.mode = 0;
    a.n = n;
    a.m = m;
    a.p = p;
    a.A = Ahat_dev;
    a.lda = lda_dev;
    a.A_host = Ahat_host;
    a.lda_host = lda_host;
    a.B = Bhat;
    a.ldb = ldb;
    a.C = Chat;
    a.ldc = ldc > 0 ? ldc : 1;
    a.shifts = (const double2*)shifts;
    a.s = s;
    a.nb = nb;
    a.batch = batch;
    a.rtol = rtol;
    a.out = (double2*)G;
    a.ldo = ldg > 0 ? ldg : 1;
    a.fail = fail_row;
    return run_sweep(h, a, (cudaStream_t)stream);
}

int ss_pspec_eval(ss_handle* h, int n, int m, int p, const double* Ahat, int64_t lda,
                  const double* Bhat, int64_t ldb, const double* Chat, int64_t ldc,
                  const double* shifts, int64_t s, int nb, int64_t batch, double rtol, double* G,
                  int64_t ldg, double* norms, int32_t* fail_row, void* stream) {
    if (!h) return SS_EARG;
    if (p < 1) return ss::set_err(h, SS_EARG, "pseudospectrum: p must be >= 1");
    if (s > 0 && !norms) return ss::set_err(h, SS_EARG, "null pointer");
    int rc = ss_tf_eval(h, n, m, p, Ahat, lda, Bhat, ldb, Chat, ldc, shifts, s, nb, batch, rtol, G,
                        ldg, fail_row, stream);
    if (rc || s == 0) return rc;
    ss::DevGuard dg(h->device);
    SS_CUDA_TRY(h, dg.err);
    cudaStream_t st = (cudaStream_t)stream;
    const int k = std::min(p, m);
    const bool gh = k > kPnSmem;
    const unsigned grid = (unsigned)std::min<int64_t>(s, (int64_t)h->num_sms * 4);
    double2* scratch = nullptr;
    if (gh) {  // one k x (k + 1) slot per CTA (the sweep's workspace is free again)
        rc = ss::ensure_ws(h, (size_t)grid * k * pn_ld(k) * 16, 0);
        if (rc) return rc;
        scratch = (double2*)h->ws;
    }
    static ss::DevMask attrs;
    if (!attrs.has(h)) {
        SS_CUDA_TRY(h, cudaFuncSetAttribute(k_pnorm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)pnorm_smem(kPnSmem, false)));
        attrs.set(h);
    }
    cudaEvent_t ev = ss::timing_begin(h, st);
    if (gh)
        k_pnorm<true><<<grid, kPnThreads, pnorm_smem(k, true), st>>>(p, m, s, (const double2*)G, ldg,
                                                                     fail_row, norms, scratch);
    else
        k_pnorm<false><<<grid, kPnThreads, pnorm_smem(k, false), st>>>(p, m, s, (const double2*)G, ldg,
                                                                       fail_row, norms, nullptr);
    SS_LAUNCH_CHECK(h);
    ss::timing_end(h, st, ev, ss::PH_TAIL);
    return SS_OK;
}

int ss_solve_reduced(ss_handle* h, int n, int m, const double* Ahat, int64_t lda,
                     const double* Bhat, int64_t ldb, const double* shifts, int64_t s,
                     const double* bdirs, int64_t ldbd, int nb, int64_t batch, double rtol,
                     double* X, int64_t ldx, int32_t* fail_row, void* stream) {
    if (!h) return SS_EARG;
    if (n < 1 || m < 1 || m > n || s < 0)
        return ss::set_err(h, SS_EDIM, "inconsistent controller-Hessenberg form");
    if (lda < n || ldb < m || ldbd < m || ldx < n)
        return ss::set_err(h, SS_EDIM, "leading dimension too small");
    if (nb < 1) return ss::set_err(h, SS_EARG, "window block size must be >= 1");
    if (s > 0 && (!Ahat || !Bhat || !shifts || !bdirs || !X || !fail_row))
        return ss::set_err(h, SS_EARG, "null pointer");
    SweepArgs a{};
    a.mode = 1;
    a.n = n;
    a.m = m;
    a.p = 0;
    a.A = Ahat;
    a.lda = lda;
    a.B = Bhat;
    a.ldb = ldb;
    a.C = nullptr;
    a.ldc = 1;
    a.shifts = (const double2*)shifts;
    a.s = s;
    a.bd = (const double2*)bdirs;
    a.ldbd = ldbd;
    a.nb = nb;
    a.batch = batch;
    a.rtol = rtol;
    a.out = (double2*)X;
    a.ldo = ldx;
    a.fail = fail_row;
    return run_sweep(h, a, (cudaStream_t)stream);
}

}  // extern "C"
