/*
 * shiftsolve_b200.h -- C ABI of the B200-native batched shifted solver.
 *
 * The reference (`shiftsolve`, pure Python) has no native boundary: its
 * operator surface is the Python functions cited below.  This header is the
 * drop-in C boundary a maintainer of the reference would bind (ctypes stub in
 * INTEGRATION.md); paper_1708_06290_b200/_lib.py binds it the same way.
 *
 * Conventions (all entry points):
 *   - every matrix is column-major with an explicit leading dimension
 *     (reference kernels.py:1-11);
 *   - complex data is interleaved complex128 (re, im), i.e. numpy / torch /
 *     cuDoubleComplex layout, passed as double*;
 *   - array pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors)
 *     on the handle's device; `stream` is a cudaStream_t (NULL = legacy
 *     default stream); all work is stream-ordered and the call returns
 *     without synchronising unless stated;
 *   - return value: SS_OK or an SS_E* code; ss_last_error() explains it.
 *     Singular shifts are NOT errors: they are reported per shift in
 *     fail_row (reference solvers.py:226-228, 263-266).
 */
#ifndef SHIFTSOLVE_B200_H
#define SHIFTSOLVE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_OK 0
#define SS_EDIM 1    /* inconsistent dimensions (reference DimensionMismatchError) */
#define SS_EARG 2    /* bad scalar argument, e.g. nb < 1 (reference ValueError)      */
#define SS_ECUDA 3   /* CUDA runtime error                                          */
#define SS_ENOMEM 4  /* device workspace allocation failed                          */

typedef struct ss_handle ss_handle;

/* Library version (major*10000 + minor*100 + patch). */
int ss_version(void);

/* Create / destroy a handle bound to `device`.  The handle owns the device
 * workspace (window arrays, rotation tables, cached schedules); use one
 * handle per host thread or stream.  Nothing is allocated in the hot loop. */
int ss_create(ss_handle** h, int device);
void ss_destroy(ss_handle* h);
const char* ss_last_error(const ss_handle* h);

/* Greedy step-parallel Givens annihilation plan for an n_rows x n_cols upper
 * trapezoid (host function).  Replaces schedule.py:88-159 greedy_schedule.
 * job_size[num_steps], rot_info[3*num_rots] (1-based (r, c1, c2) triplets,
 * same order as the reference).  Capacities: job_cap >= n_rows*(n_cols-n_rows)+1,
 * info_cap >= 3*n_rows*(n_cols-n_rows). */
int ss_greedy_schedule(int n_rows, int n_cols, int64_t* job_size, int64_t job_cap,
                       int64_t* rot_info, int64_t info_cap, int* num_steps, int* num_rots);

/* Transfer function on controller-Hessenberg data.
 * Replaces solvers.py:234-271 eval_transfer_function (and the sweep
 * solvers.py:130-231 beneath it):
 *   G(:, l*m:(l+1)*m) = C (sigma_l I - A)^{-1} B = -Chat (Ahat - sigma_l I)^{-1} Bhat
 * Ahat n x n (m-Hessenberg, zeros below the m-th subdiagonal), Bhat: only
 * Bhat[0:m, 0:m] is read, Chat p x n.  shifts: s complex128.  nb: window
 * block (>= 1; clamped to what one SM's shared memory holds for this m).
 * batch: shifts per device pass (<= 0: sized from free memory).  rtol: the
 * relative pivot threshold, used as given (0: only exactly-zero pivots fail,
 * solvers.py:227); NaN selects the reference default 1e3*n*eps
 * (solvers.py:95-97).  G: p x (s*m) complex128, leading dim ldg.
 * fail_row[l]: -1, or the 0-based head pivot index that fell below
 * rtol*||Ahat - sigma_l I||_F (G slice is then NaN). */
int ss_tf_eval(ss_handle* h, int n, int m, int p, const double* Ahat, int64_t lda,
               const double* Bhat, int64_t ldb, const double* Chat, int64_t ldc,
               const double* shifts, int64_t s, int nb, int64_t batch, double rtol,
               double* G, int64_t ldg, int32_t* fail_row, void* stream);

/* ss_tf_eval with Ahat in (pinned) host memory: Ahat is copied to the
 * caller's device buffer Ahat_dev (n x n, lda_dev) on an internal copy
 * stream in the order the sweep consumes its columns (the seed's last m
 * columns, then one outer block / window at a time, right to left); each
 * step waits only for its own columns, so the 8 n^2-byte transfer overlaps
 * the sweep.  Everything else as ss_tf_eval (device B, C, shifts, G). */
int ss_tf_eval_stream(ss_handle* h, int n, int m, int p, const double* Ahat_host,
                      int64_t lda_host, double* Ahat_dev, int64_t lda_dev, const double* Bhat,
                      int64_t ldb, const double* Chat, int64_t ldc, const double* shifts, int64_t s,
                      int nb, int64_t batch, double rtol, double* G, int64_t ldg, int32_t* fail_row,
                      void* stream);

/* Structured pseudospectrum: ss_tf_eval (G into the caller's scratch G)
 * followed by a device epilogue norms[l] = ||G_l||_2 (p x m block; +inf for
 * a singular shift).  Replaces solvers.py:501-530 (two_norm_small's numpy
 * SVD): Gram matrix + parallel Hermitian Jacobi per shift, any p >= 1, m. */
int ss_pspec_eval(ss_handle* h, int n, int m, int p, const double* Ahat, int64_t lda,
                  const double* Bhat, int64_t ldb, const double* Chat, int64_t ldc,
                  const double* shifts, int64_t s, int nb, int64_t batch, double rtol, double* G,
                  int64_t ldg, double* norms, int32_t* fail_row, void* stream);

/* Reduced shifted solves (Ahat - sigma_l I) x_l = Bhat b_l.
 * Replaces solvers.py:274-313 solve_shifted_reduced.  bdirs: m x s
 * complex128 (ldbd); X: n x s complex128 (ldx), NaN column on failure. */
int ss_solve_reduced(ss_handle* h, int n, int m, const double* Ahat, int64_t lda,
                     const double* Bhat, int64_t ldb, const double* shifts, int64_t s,
                     const double* bdirs, int64_t ldbd, int nb, int64_t batch, double rtol,
                     double* X, int64_t ldx, int32_t* fail_row, void* stream);

/* Transposed shifted solves (Ahat - sigma_l I)^T x_l = c_l, general
 * right-hand sides.  Replaces solvers.py:320-486 solve_shifted_transposed
 * (top-down LQ sweep with fused forward substitution, batched.py:125-182).
 * rhs: n x s complex128 (ldr); X: n x s complex128 (ldx), NaN column on
 * failure; fail_row[l]: -1 or the 0-based row of the first pivot that fell
 * below rtol*||Ahat - sigma_l I||_F.  Requires m + 1 <= 256; nb is clamped
 * to 32 (one warp per window), and for m + 1 > 32 to what the shared-memory
 * window of k_lq_big holds. */
int ss_solve_transposed(ss_handle* h, int n, int m, const double* Ahat, int64_t lda,
                        const double* shifts, int64_t s, const double* rhs, int64_t ldr,
                        int nb, int64_t batch, double rtol, double* X, int64_t ldx,
                        int32_t* fail_row, void* stream);

/* In-place orthogonal reduction of (A, B, C) to controller-Hessenberg form.
 * Replaces hessenberg.py:260-328 reduce_controller_hessenberg.
 * A n x n -> Ahat (exact zeros below the m-th subdiagonal), B n x m -> Bhat
 * (upper triangular, rows m.. exactly zero), C p x n -> Chat.  Q (nullable)
 * n x n receives the accumulated orthogonal factor (Q^T A Q = Ahat).
 * block_size: panel width (>= 1).  1 <= m < n required. */
int ss_reduce_chf(ss_handle* h, int n, int m, int p, double* A, int64_t lda, double* B,
                  int64_t ldb, double* C, int64_t ldc, double* Q, int64_t ldq,
                  int block_size, void* stream);

/* Per-phase accounting under the reference phase names (counters.py:17-23):
 * index 0 contr_hess_reduction, 1 small_batched_rq, 2 batched_gemm,
 * 3 outer_gemm, 4 tail_solves.  flops follow the reference's shape-only
 * formulas; seconds are CUDA-event times recorded around every kernel while
 * timing is enabled.  Recording never synchronises; ss_phase_stats and
 * ss_update_kernel_stats wait for the recorded events and fold them in. */
int ss_set_timing(ss_handle* h, int enabled);
int ss_phase_stats(ss_handle* h, double* seconds5, double* flops5);
void ss_reset_stats(ss_handle* h);

/* Live statistics of the dominant kernel (the window update, k_update):
 * launches, summed CUDA-event seconds and summed algorithmic flops
 * (4 m x structurally-nonzero panel entries per shift) since
 * the last ss_reset_stats, for roofline accounting. */
int ss_update_kernel_stats(ss_handle* h, int64_t* launches, double* seconds, double* alg_flops);

/* Diagnostic: measured FP64 FMA throughput of this device (TFLOP/s) from a
 * DFMA-chain kernel over all SMs -- the denominator of the FP64 roofline. */
int ss_probe_dfma_peak(ss_handle* h, double* tflops);

/* Diagnostics: measured FP64 tensor-core (DMMA m16n8k8) peak in TFLOP/s. */
int ss_probe_dmma_peak(ss_handle* h, double* tflops);

/* Diagnostics / tests: the reduction's FP64 tensor-core GEMM (ss_gemm.cuh),
 * C = alpha op(A) op(B) + beta C, column-major device pointers, op(X) = X^T
 * when ta / tb is nonzero.  Deterministic (split-K partials summed in order). */
int ss_dgemm(ss_handle* h, int ta, int tb, int M, int N, int K, double alpha, const double* A,
             int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
             void* stream);

/* Number of device kernels this handle has launched since creation. */
int64_t ss_launch_count(const ss_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* SHIFTSOLVE_B200_H */
