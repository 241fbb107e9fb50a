/*
 * shiftsolve_oracle.c -- CPU restatement of the reference shifted-solve path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle and the CPU
 * baseline ("kind": "port") for the B200 library in paper_1708_06290_b200/.
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) may load it; the product path never does.
 *
 * It restates, in plain C99, the algorithm of the reference package
 * `shiftsolve` (pure Python/numpy, /root/reference/pkg/src/shiftsolve):
 *
 *   givens / rotate_columns        kernels.py:118-153
 *   householder_vector             kernels.py:74-99
 *   greedy_schedule                schedule.py:88-159
 *   _factor_block / batched_rq     batched.py:64-122
 *   _shift_scales                  solvers.py:104-110
 *   _sweep_rq                      solvers.py:130-201
 *   _head_solve_rq                 solvers.py:204-231
 *   eval_transfer_function         solvers.py:234-271
 *   solve_shifted_reduced          solvers.py:274-313
 *   reduce_controller_hessenberg   hessenberg.py:260-328 (unblocked form, the
 *                                  same reflectors as oracles.py:75-106)
 *
 * Parity pin: tests/golden/ holds vectors produced by the Python reference
 * itself (tests/golden/make_golden.py); tests/test_oracle_golden.py checks
 * this restatement against them before the GPU path is checked against it.
 *
 * Per-shift work is independent (solvers.py:25-28), so the sweep runs one
 * shift at a time and OpenMP spreads shifts over host threads.  The panel
 * Z1 is real; multiplying a real by a complex with the naive formula is
 * bitwise equal to the reference's complex(x,0) * z, so the panel is kept
 * real here.  All matrices are column-major (kernels.py:1-11).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double _Complex zc;

#define ORC_EPS 2.220446049250313e-16

/* ------------------------------------------------------------------ */
/* kernels.py:118-136  givens(a, b) -> (c, s, r)                        */
/* ------------------------------------------------------------------ */
static void orc_givens(zc a, zc b, double* c, zc* s, zc* r) {
    if (b == 0) { *c = 1.0; *s = 0.0; *r = a; return; }
    if (a == 0) {
        double babs = cabs(b);
        *c = 0.0; *s = conj(b) / babs; *r = babs; return;
    }
    double aabs = cabs(a);
    double d = hypot(aabs, cabs(b));
    zc phase = a / aabs;
    *c = aabs / d;
    *s = phase * conj(b) / d;
    *r = phase * d;
}

/* kernels.py:139-153: helper <- c*h + s*t ; target <- c*t - conj(s)*h */
static void orc_rotate_columns(zc* M, long ld, int helper, int target, double c, zc s,
                               int lo, int hi) {
    zc* h = M + (long)helper * ld;
    zc* t = M + (long)target * ld;
    zc cs = conj(s);
    for (int i = lo; i < hi; ++i) {
        zc xh = h[i], xt = t[i];
        h[i] = c * xh + s * xt;
        t[i] = c * xt - cs * xh;
    }
}

/* ------------------------------------------------------------------ */
/* schedule.py:88-159  greedy_schedule(n_rows, n_cols)                 */
/* job_size: capacity n_rows*delta+1; rot_info: capacity 3*n_rows*delta */
/* returns num_steps (or -1 on bad shape); *num_rots set.               */
/* ------------------------------------------------------------------ */
int orc_greedy_schedule(int n_rows, int n_cols, int64_t* job_size, int64_t* rot_info,
                        int* num_rots) {
    if (n_rows < 1 || n_cols < n_rows) return -1;
    const int delta = n_cols - n_rows, w = delta + 1;
    /* position (r, c), 1-based, c in [r, r+delta] -> index (r-1)*w + (c-r) */
    char* ready = (char*)malloc((size_t)n_rows * w);
    char* avail = (char*)malloc((size_t)n_rows * w);
    int* busy = (int*)malloc(sizeof(int) * ((size_t)n_rows * w + 1));
    int* prom = (int*)malloc(sizeof(int) * ((size_t)n_rows * w + 1));
    for (int r = 1; r <= n_rows; ++r)
        for (int c = r; c <= r + delta; ++c) {
            ready[(r - 1) * w + (c - r)] = 1;
            avail[(r - 1) * w + (c - r)] = (r == n_rows) || (c == r);
        }
    int nbusy = 0, nprom = 0, steps = 0, rots = 0;
    for (;;) {
        for (int i = 0; i < nbusy; ++i) ready[busy[i]] = 1;
        nbusy = 0;
        for (int i = 0; i < nprom; ++i) avail[prom[i]] = 1;
        nprom = 0;
        int count = 0;
        for (int r = n_rows; r >= 1; --r) {
            for (int c1 = r; c1 <= r + delta; ++c1) {
                int p1 = (r - 1) * w + (c1 - r);
                if (!(ready[p1] && avail[p1])) continue;
                for (int c2 = r + delta; c2 > c1; --c2) {
                    int p2 = (r - 1) * w + (c2 - r);
                    if (ready[p2] && avail[p2]) {
                        rot_info[3 * rots + 0] = r;
                        rot_info[3 * rots + 1] = c1;
                        rot_info[3 * rots + 2] = c2;
                        ++rots; ++count;
                        ready[p1] = 0; ready[p2] = 0;
                        busy[nbusy++] = p2;
                        if (r > 1) {
                            int pu = (r - 2) * w + (c1 - (r - 1));
                            avail[pu] = 0;
                            prom[nprom++] = pu;
                        }
                        break;
                    }
                }
            }
        }
        if (count == 0) break;
        job_size[steps++] = count;
    }
    free(ready); free(avail); free(busy); free(prom);
    *num_rots = rots;
    return steps;
}

/* ------------------------------------------------------------------ */
/* batched.py:64-90  _factor_block (upper variant) on one block         */
/* Z: nr x nc (ld nr), Pfull: nc x nc (ld nc), starts as identity.      */
/* ------------------------------------------------------------------ */
static void orc_factor_block(zc* Z, int nr, zc* Pfull, int nc, int steps,
                             const int64_t* job, const int64_t* info) {
    int off = 0;
    for (int t = 0; t < steps; ++t) {
        for (int k = off; k < off + job[t]; ++k) {
            int r = (int)info[3 * k], c1 = (int)info[3 * k + 1], c2 = (int)info[3 * k + 2];
            double c; zc s, rr;
            orc_givens(Z[(r - 1) + (long)(c2 - 1) * nr], Z[(r - 1) + (long)(c1 - 1) * nr], &c, &s, &rr);
            orc_rotate_columns(Z, nr, c2 - 1, c1 - 1, c, s, 0, r);
            Z[(r - 1) + (long)(c1 - 1) * nr] = 0.0;
            Z[(r - 1) + (long)(c2 - 1) * nr] = rr;
            orc_rotate_columns(Pfull, nc, c2 - 1, c1 - 1, c, s, 0, nc);
        }
        off += (int)job[t];
    }
}

typedef struct { int nr, nc, steps, rots; int64_t* job; int64_t* info; } orc_sched;

static int orc_sched_make(orc_sched* sc, int nr, int nc) {
    int delta = nc - nr;
    sc->nr = nr; sc->nc = nc;
    sc->job = (int64_t*)malloc(sizeof(int64_t) * ((size_t)nr * delta + 1));
    sc->info = (int64_t*)malloc(sizeof(int64_t) * (3 * (size_t)nr * delta + 3));
    sc->steps = orc_greedy_schedule(nr, nc, sc->job, sc->info, &sc->rots);
    return sc->steps;
}
static void orc_sched_free(orc_sched* sc) { free(sc->job); free(sc->info); }

/* batched.py:93-122  batched_rq: s blocks side by side in Z (nr x s*nc). */
int orc_batched_rq(int nr, int nc, int s, zc* Z, int m_keep, zc* P) {
    if (nr < 1 || nc < nr || s < 0 || m_keep < 1 || m_keep > nc) return -1;
    orc_sched sc;
    orc_sched_make(&sc, nr, nc);
    zc* Pfull = (zc*)malloc(sizeof(zc) * (size_t)nc * nc);
    for (int l = 0; l < s; ++l) {
        memset(Pfull, 0, sizeof(zc) * (size_t)nc * nc);
        for (int i = 0; i < nc; ++i) Pfull[i + (long)i * nc] = 1.0;
        orc_factor_block(Z + (long)l * nc * nr, nr, Pfull, nc, sc.steps, sc.job, sc.info);
        memcpy(P + (long)l * m_keep * nc, Pfull, sizeof(zc) * (size_t)nc * m_keep);
    }
    free(Pfull);
    orc_sched_free(&sc);
    return 0;
}

/* solvers.py:104-110: ||A - sigma I||_F in closed form */
static void orc_fro2_trace(int n, const double* A, long lda, double* fro2, double* tr) {
    double f = 0.0, t = 0.0;
    for (int j = 0; j < n; ++j) {
        for (int i = 0; i < n; ++i) f += A[i + j * lda] * A[i + j * lda];
        t += A[j + j * lda];
    }
    *fro2 = f; *tr = t;
}
static double orc_shift_scale(double fro2, double tr, int n, zc sig) {
    double v = fro2 - 2.0 * creal(conj(sig) * tr) + (cabs(sig) * cabs(sig)) * n;
    return sqrt(v > 0.0 ? v : 0.0);
}

/* ------------------------------------------------------------------ */
/* solvers.py:130-201  _sweep_rq for ONE shift.                          */
/* top == NULL -> identity top of height n (ptop = n).                   */
/* z2: (ptop+n) x m, ld = ptop+n.                                        */
/* ------------------------------------------------------------------ */
typedef struct {
    zc *blk, *Pfull, *tmp, *prod;
    int nb0, m, ncap, rows;
    orc_sched sfull, slast;
    int last_nb;
} orc_ws;

/* panel value [top; A](i, col) */
static inline double orc_panel(int i, int col, int ptop, const double* A, long lda,
                               const double* top, long ldt) {
    if (i < ptop) return top ? top[i + (long)col * ldt] : (i == col ? 1.0 : 0.0);
    return A[(i - ptop) + (long)col * lda];
}

/* rdiag (nullable): rdiag[0] = min |R_ii|, rdiag[1] = sum log|R_ii| over the
   window blocks' R diagonals (after the RQ a block is [0 | R] with R nb x nb
   upper triangular in its last nb columns); the head pivots are added by
   orc_head_solve.  These give the condition estimate of SURVEY 8(d)
   (||Ahat - sigma I||_F / min |R_ii|) and a determinant check. */
static void orc_sweep_one(int n, int m, int ptop, const double* A, long lda,
                          const double* top, long ldt, zc sigma, int nb0, zc* z2,
                          orc_ws* ws, double* rdiag) {
    const long ld = ptop + n;
    /* seed: last m columns of the stack with the shift on A's diagonal */
    for (int c = 0; c < m; ++c) {
        zc* col = z2 + c * ld;
        for (int i = 0; i < ptop; ++i)
            col[i] = top ? top[i + (long)(n - m + c) * ldt] : ((i == n - m + c) ? 1.0 : 0.0);
        for (int i = 0; i < n; ++i) col[ptop + i] = A[i + (long)(n - m + c) * lda];
        col[ptop + n - m + c] -= sigma;
    }
    int k = n;
    while (k >= m + 1) {
        int nb = nb0 < (k - m) ? nb0 : (k - m);
        int mnb = m < nb ? m : nb;
        int r0 = ptop + k - nb;
        int c0 = k - m - nb;
        int nc = nb + m;
        orc_sched* sc = (nb == nb0) ? &ws->sfull : &ws->slast;
        if (nb != nb0 && ws->last_nb != nb) {
            if (ws->last_nb > 0) orc_sched_free(&ws->slast);
            orc_sched_make(&ws->slast, nb, nc);
            ws->last_nb = nb;
        }
        /* pack block (solvers.py:174-181) */
        zc* Zb = ws->blk;
        for (int j = 0; j < nb; ++j)
            for (int t = 0; t < nb; ++t)
                Zb[t + (long)j * nb] = orc_panel(r0 + t, c0 + j, ptop, A, lda, top, ldt);
        for (int j = 0; j < m; ++j)
            for (int t = 0; t < nb; ++t) Zb[t + (long)(nb + j) * nb] = z2[r0 + t + j * ld];
        if (nb > m)
            for (int t = 0; t < nb - m; ++t) Zb[t + (long)(t + m) * nb] -= sigma;
        /* RQ (batched.py:93-122), P* kept in full, first m columns used */
        zc* P = ws->Pfull;
        memset(P, 0, sizeof(zc) * (size_t)nc * nc);
        for (int i = 0; i < nc; ++i) P[i + (long)i * nc] = 1.0;
        orc_factor_block(Zb, nb, P, nc, sc->steps, sc->job, sc->info);
        if (rdiag)
            for (int t = 0; t < nb; ++t) {
                double a = cabs(Zb[t + (long)(m + t) * nb]);
                if (a < rdiag[0]) rdiag[0] = a;
                rdiag[1] += log(a);
            }
        /* update_shift (solvers.py:187-191): z2[:r0] = z2[:r0] @ P[nb:nb+m] */
        zc* tmp = ws->tmp;
        for (int c = 0; c < m; ++c) {
            zc* tc = tmp + (long)c * r0;
            for (int i = 0; i < r0; ++i) tc[i] = 0.0;
            for (int j = 0; j < m; ++j) {
                zc pj = P[(nb + j) + (long)c * nc];
                const zc* zj = z2 + j * ld;
                for (int i = 0; i < r0; ++i) tc[i] += zj[i] * pj;
            }
        }
        for (int c = 0; c < m; ++c) memcpy(z2 + c * ld, tmp + (long)c * r0, sizeof(zc) * r0);
        /* lazy shift correction: z2[r0-m : r0-m+mnb] -= sigma * P[:mnb] */
        for (int c = 0; c < m; ++c)
            for (int t = 0; t < mnb; ++t) z2[(r0 - m + t) + c * ld] -= sigma * P[t + (long)c * nc];
        /* outer gemm (solvers.py:197-199 -> kernels.py:212-243): z2 += Z1 @ P[:nb] */
        zc* prod = ws->prod;
        for (int c = 0; c < m; ++c) {
            zc* pc = prod + (long)c * r0;
            for (int i = 0; i < r0; ++i) pc[i] = 0.0;
            for (int j = 0; j < nb; ++j) {
                zc pj = P[j + (long)c * nc];
                int col = c0 + j;
                int i = 0;
                if (top) {
                    const double* tcol = top + (long)col * ldt;
                    for (; i < ptop; ++i) pc[i] += tcol[i] * pj;
                } else {
                    pc[col] += pj; /* identity top: one nonzero per panel column */
                    i = ptop;
                }
                const double* acol = A + (long)col * lda - ptop;
                for (; i < r0; ++i) pc[i] += acol[i] * pj;
            }
            zc* zc_ = z2 + c * ld;
            for (int i = 0; i < r0; ++i) zc_[i] += pc[i];
        }
        k -= nb;
    }
}

/* solvers.py:204-231  _head_solve_rq for one shift; returns -1 or pivot i */
static int orc_head_solve(zc* z2, long ld, int ptop, int m, const zc* rhs, int q, double tol,
                          zc* X /* m x q, ld m */, double* rdiag, double* pmin) {
    for (int i = 0; i < m * q; ++i) X[i] = 0.0;
    for (int i = m - 1; i >= 0; --i) {
        int row = ptop + i;
        for (int jj = 0; jj < i; ++jj) {
            double c; zc s, rr;
            orc_givens(z2[row + i * ld], z2[row + jj * ld], &c, &s, &rr);
            orc_rotate_columns(z2, ld, i, jj, c, s, 0, ptop + m);
            z2[row + jj * ld] = 0.0;
            z2[row + i * ld] = rr;
        }
        zc piv = z2[row + i * ld];
        if (rdiag) {
            double a = cabs(piv);
            if (a < rdiag[0]) rdiag[0] = a;
            rdiag[1] += log(a);
        }
        if (pmin && cabs(piv) < *pmin) *pmin = cabs(piv);
        if (cabs(piv) <= tol) return i;
        for (int c = 0; c < q; ++c) {
            zc acc = 0.0;
            for (int j = i + 1; j < m; ++j) acc += z2[row + j * ld] * X[j + c * m];
            X[i + c * m] = (rhs[i + c * m] - acc) / piv;
        }
    }
    return -1;
}

static int orc_ws_init(orc_ws* ws, int n, int m, int ptop, int nb0) {
    memset(ws, 0, sizeof(*ws));
    int nbc = nb0 < (n - m) ? nb0 : (n - m);
    if (nbc < 1) nbc = 1;
    int nc = nbc + m;
    ws->nb0 = nbc; ws->m = m;
    ws->blk = (zc*)malloc(sizeof(zc) * (size_t)nbc * nc);
    ws->Pfull = (zc*)malloc(sizeof(zc) * (size_t)nc * nc);
    ws->tmp = (zc*)malloc(sizeof(zc) * (size_t)(ptop + n) * m);
    ws->prod = (zc*)malloc(sizeof(zc) * (size_t)(ptop + n) * m);
    if (n - m >= 1) orc_sched_make(&ws->sfull, nbc, nc);
    ws->last_nb = 0;
    return 0;
}
static void orc_ws_free(orc_ws* ws) {
    free(ws->blk); free(ws->Pfull); free(ws->tmp); free(ws->prod);
    if (ws->sfull.job) orc_sched_free(&ws->sfull);
    if (ws->last_nb > 0) orc_sched_free(&ws->slast);
}

static void orc_set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

/* ------------------------------------------------------------------ */
/* solvers.py:234-271  eval_transfer_function                           */
/* G: p x (s*m) complex, ld ldg; fail[l] = -1 or the failing head index. */
/* Failed slices are NaN (solvers.py:256).                               */
/* ------------------------------------------------------------------ */
/* diag (nullable): per shift 3 doubles -- kappa = ||Ahat - sigma I||_F /
   min |R_ii| (SURVEY 8(d) condition estimate), the smallest computed head
   pivot relative to ||Ahat - sigma I||_F (the quantity the singular test
   compares with rtol, solvers.py:226-228), and sum log |R_ii| (=
   log |det(Ahat - sigma I)| when no pivot failed).  Test infrastructure. */
int orc_tf_eval_diag(int n, int m, int p, const double* A, long lda, const double* B, long ldb,
                     const double* C, long ldc, const zc* shifts, int s, int nb, double rtol,
                     zc* G, long ldg, int* fail, int nthreads, double* diag);
int orc_solve_reduced_diag(int n, int m, const double* A, long lda, const double* B, long ldb,
                           const zc* shifts, int s, const zc* bdirs, long ldbd, int nb,
                           double rtol, zc* Xo, long ldx, int* fail, int nthreads, double* diag);

int orc_tf_eval(int n, int m, int p, const double* A, long lda, const double* B, long ldb,
                const double* C, long ldc, const zc* shifts, int s, int nb, double rtol,
                zc* G, long ldg, int* fail, int nthreads) {
    return orc_tf_eval_diag(n, m, p, A, lda, B, ldb, C, ldc, shifts, s, nb, rtol, G, ldg, fail,
                            nthreads, NULL);
}

int orc_tf_eval_diag(int n, int m, int p, const double* A, long lda, const double* B, long ldb,
                     const double* C, long ldc, const zc* shifts, int s, int nb, double rtol,
                     zc* G, long ldg, int* fail, int nthreads, double* diag) {
    if (n < 1 || m < 1 || m > n || p < 0 || nb < 1 || s < 0) return -1;
    if (isnan(rtol)) rtol = 1e3 * n * ORC_EPS; /* NaN: reference default */
    double fro2, tr;
    orc_fro2_trace(n, A, lda, &fro2, &tr);
    zc* Bh = (zc*)malloc(sizeof(zc) * (size_t)m * m);
    for (int j = 0; j < m; ++j)
        for (int i = 0; i < m; ++i) Bh[i + j * m] = B[i + (long)j * ldb];
    orc_set_threads(nthreads);
    const double qnan = nan("");
#pragma omp parallel
    {
        orc_ws ws;
        orc_ws_init(&ws, n, m, p, nb);
        zc* z2 = (zc*)malloc(sizeof(zc) * (size_t)(p + n) * m);
        zc* X = (zc*)malloc(sizeof(zc) * (size_t)m * m);
#pragma omp for schedule(dynamic, 1)
        for (int l = 0; l < s; ++l) {
            double rd[2] = {INFINITY, 0.0}, pm = INFINITY;
            orc_sweep_one(n, m, p, A, lda, C, ldc, shifts[l], nb, z2, &ws, diag ? rd : NULL);
            double scale = orc_shift_scale(fro2, tr, n, shifts[l]);
            double tol = rtol * scale;
            int bad = orc_head_solve(z2, p + n, p, m, Bh, m, tol, X, diag ? rd : NULL, &pm);
            fail[l] = bad;
            if (diag) {
                diag[3 * l] = scale / rd[0];
                diag[3 * l + 1] = pm / scale;
                diag[3 * l + 2] = rd[1];
            }
            for (int c = 0; c < m; ++c) {
                zc* g = G + (long)(l * m + c) * ldg;
                for (int i = 0; i < p; ++i) {
                    if (bad >= 0) { g[i] = CMPLX(qnan, qnan); continue; }
                    zc acc = 0.0;
                    for (int j = 0; j < m; ++j) acc += z2[i + (long)j * (p + n)] * X[j + c * m];
                    g[i] = -acc;
                }
            }
        }
        free(z2); free(X);
        orc_ws_free(&ws);
    }
    free(Bh);
    return 0;
}

/* solvers.py:274-313  solve_shifted_reduced: X n x s (ld ldx) */
int orc_solve_reduced(int n, int m, const double* A, long lda, const double* B, long ldb,
                      const zc* shifts, int s, const zc* bdirs, long ldbd, int nb,
                      double rtol, zc* Xo, long ldx, int* fail, int nthreads) {
    return orc_solve_reduced_diag(n, m, A, lda, B, ldb, shifts, s, bdirs, ldbd, nb, rtol, Xo, ldx,
                                  fail, nthreads, NULL);
}

int orc_solve_reduced_diag(int n, int m, const double* A, long lda, const double* B, long ldb,
                           const zc* shifts, int s, const zc* bdirs, long ldbd, int nb,
                           double rtol, zc* Xo, long ldx, int* fail, int nthreads, double* diag) {
    if (n < 1 || m < 1 || m > n || nb < 1 || s < 0) return -1;
    if (isnan(rtol)) rtol = 1e3 * n * ORC_EPS; /* NaN: reference default */
    double fro2, tr;
    orc_fro2_trace(n, A, lda, &fro2, &tr);
    orc_set_threads(nthreads);
    const double qnan = nan("");
#pragma omp parallel
    {
        orc_ws ws;
        orc_ws_init(&ws, n, m, n, nb);
        zc* z2 = (zc*)malloc(sizeof(zc) * (size_t)(2 * n) * m);
        zc* Y = (zc*)malloc(sizeof(zc) * (size_t)m);
        zc* rhs = (zc*)malloc(sizeof(zc) * (size_t)m);
#pragma omp for schedule(dynamic, 1)
        for (int l = 0; l < s; ++l) {
            /* rhs = Bh @ b_dirs[:, l]  (solvers.py:304) */
            for (int i = 0; i < m; ++i) {
                zc acc = 0.0;
                for (int j = 0; j < m; ++j) acc += B[i + (long)j * ldb] * bdirs[j + (long)l * ldbd];
                rhs[i] = acc;
            }
            double rd[2] = {INFINITY, 0.0}, pm = INFINITY;
            orc_sweep_one(n, m, n, A, lda, NULL, 0, shifts[l], nb, z2, &ws, diag ? rd : NULL);
            double scale = orc_shift_scale(fro2, tr, n, shifts[l]);
            double tol = rtol * scale;
            int bad = orc_head_solve(z2, 2 * n, n, m, rhs, 1, tol, Y, diag ? rd : NULL, &pm);
            fail[l] = bad;
            if (diag) {
                diag[3 * l] = scale / rd[0];
                diag[3 * l + 1] = pm / scale;
                diag[3 * l + 2] = rd[1];
            }
            zc* x = Xo + (long)l * ldx;
            for (int i = 0; i < n; ++i) {
                if (bad >= 0) { x[i] = CMPLX(qnan, qnan); continue; }
                zc acc = 0.0;
                for (int j = 0; j < m; ++j) acc += z2[i + (long)j * 2 * n] * Y[j];
                x[i] = acc;
            }
        }
        free(z2); free(Y); free(rhs);
        orc_ws_free(&ws);
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* kernels.py:74-99 householder_vector, real case.  x has len entries.   */
/* v[0] = 1; returns tau, *beta.                                         */
/* ------------------------------------------------------------------ */
static double orc_householder(const double* x, int len, double* v, double* beta) {
    double alpha = x[0], sigma = 0.0;
    for (int i = 1; i < len; ++i) sigma += x[i] * x[i];
    v[0] = 1.0;
    for (int i = 1; i < len; ++i) v[i] = 0.0;
    if (sigma == 0.0) { *beta = alpha; return 0.0; }
    double anorm = sqrt(alpha * alpha + sigma);
    double b = (alpha >= 0) ? -anorm : anorm;
    double tau = (b - alpha) / b;
    double den = alpha - b;
    for (int i = 1; i < len; ++i) v[i] = x[i] / den;
    *beta = b;
    return tau;
}

/* M[r0:r0+len, c0:c1] -= tau v (v^T M[r0:r0+len, c0:c1]) */
static void orc_left(double* M, long ld, int r0, int len, int c0, int c1, const double* v,
                     double tau) {
    for (int j = c0; j < c1; ++j) {
        double* col = M + (long)j * ld + r0;
        double w = 0.0;
        for (int i = 0; i < len; ++i) w += v[i] * col[i];
        w *= tau;
        for (int i = 0; i < len; ++i) col[i] -= v[i] * w;
    }
}
/* M[0:rows, c0:c0+len] -= (M[0:rows, c0:c0+len] v) (tau v)^T */
static void orc_right(double* M, long ld, int rows, int c0, int len, const double* v,
                      double tau, double* w) {
    for (int i = 0; i < rows; ++i) w[i] = 0.0;
    for (int j = 0; j < len; ++j) {
        const double* col = M + (long)(c0 + j) * ld;
        for (int i = 0; i < rows; ++i) w[i] += col[i] * v[j];
    }
    for (int j = 0; j < len; ++j) {
        double* col = M + (long)(c0 + j) * ld;
        double tv = tau * v[j];
        for (int i = 0; i < rows; ++i) col[i] -= w[i] * tv;
    }
}

/* hessenberg.py:260-328 reduce_controller_hessenberg, unblocked.
 * In place: A (n x n) -> Ahat, B (n x m) -> Bhat, C (p x n) -> Chat,
 * Q (n x n, nullable) accumulates the orthogonal factor. */
int orc_reduce_chf(int n, int m, int p, double* A, long lda, double* B, long ldb, double* C,
                   long ldc, double* Q, long ldq) {
    if (n < 1 || m < 1 || m >= n || p < 0) return -1;
    double* v = (double*)malloc(sizeof(double) * n);
    double* w = (double*)malloc(sizeof(double) * (n > p ? n : p) + 8);
    if (Q)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) Q[i + (long)j * ldq] = (i == j) ? 1.0 : 0.0;
    /* QR of B with the similarity applied immediately (hessenberg.py:297-315) */
    int jmax = m < (n - 1) ? m : (n - 1);
    for (int j = 0; j < jmax; ++j) {
        double beta;
        double tau = orc_householder(B + j + (long)j * ldb, n - j, v, &beta);
        B[j + (long)j * ldb] = beta;
        for (int i = j + 1; i < n; ++i) B[i + (long)j * ldb] = 0.0;
        if (tau != 0.0) {
            orc_left(B, ldb, j, n - j, j + 1, m, v, tau);
            orc_left(A, lda, j, n - j, 0, n, v, tau);
            orc_right(A, lda, n, j, n - j, v, tau, w);
            orc_right(C, ldc, p, j, n - j, v, tau, w);
            if (Q) orc_right(Q, ldq, n, j, n - j, v, tau, w);
        }
    }
    for (int j = 0; j < m; ++j)
        for (int i = m; i < n; ++i) B[i + (long)j * ldb] = 0.0;
    /* band reduction, one column at a time (oracles.py:75-106 form) */
    for (int j = 0; j < n - m - 1; ++j) {
        int len = n - j - m;
        double beta;
        double* x = A + (j + m) + (long)j * lda;
        double tau = orc_householder(x, len, v, &beta);
        x[0] = beta;
        for (int i = 1; i < len; ++i) x[i] = 0.0;
        if (tau == 0.0) continue;
        orc_left(A, lda, j + m, len, j + 1, n, v, tau);
        orc_right(A, lda, n, j + m, len, v, tau, w);
        orc_right(C, ldc, p, j + m, len, v, tau, w);
        if (Q) orc_right(Q, ldq, n, j + m, len, v, tau, w);
    }
    free(v); free(w);
    return 0;
}
