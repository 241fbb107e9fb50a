"""CPU parity oracle for the B200 shifted-solve library.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py (the cpu_baseline leg and ``--impl reference``) as the checker and
the CPU baseline; the product package ``paper_1708_06290_b200`` never
imports it.

Two layers:

* ``shiftsolve_oracle.c`` (built to ``oracle/build/libshiftsolve_oracle.so``)
  -- a C restatement of the reference's window sweep, batched Givens RQ,
  greedy schedule, head solve and controller-Hessenberg reduction; each C
  function cites the reference file:line it follows.
* ``lu_solve_shifted`` / ``oracle_transfer_function`` below -- a restatement
  of the reference's independent dense LU oracle (oracles.py:28-72), used to
  cross-check both the C restatement and the GPU path on small systems.

The C restatement is pinned to the reference by tests/golden/*.npz, which
tests/golden/make_golden.py produced by importing the Python reference.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "build", "libshiftsolve_oracle.so")
_lib = None

EPS = float(np.finfo(np.float64).eps)


def build() -> str:
    """Compile the C restatement (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(
                os.path.join(_HERE, "shiftsolve_oracle.c")):
            build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        I = ctypes.c_int
        Lg = ctypes.c_long
        D = ctypes.c_double
        L.orc_greedy_schedule.argtypes = [I, I, P, P, P]
        L.orc_greedy_schedule.restype = I
        L.orc_batched_rq.argtypes = [I, I, I, P, I, P]
        L.orc_batched_rq.restype = I
        L.orc_tf_eval.argtypes = [I, I, I, P, Lg, P, Lg, P, Lg, P, I, I, D, P, Lg, P, I]
        L.orc_tf_eval.restype = I
        L.orc_solve_reduced.argtypes = [I, I, P, Lg, P, Lg, P, I, P, Lg, I, D, P, Lg, P, I]
        L.orc_solve_reduced.restype = I
        L.orc_tf_eval_diag.argtypes = L.orc_tf_eval.argtypes + [P]
        L.orc_tf_eval_diag.restype = I
        L.orc_solve_reduced_diag.argtypes = L.orc_solve_reduced.argtypes + [P]
        L.orc_solve_reduced_diag.restype = I
        L.orc_reduce_chf.argtypes = [I, I, I, P, Lg, P, Lg, P, Lg, P, Lg]
        L.orc_reduce_chf.restype = I
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def greedy_schedule(n_rows: int, n_cols: int):
    """schedule.py:88-159 -> (job_size int64[steps], rot_info int64[3*rots])."""
    delta = n_cols - n_rows
    job = np.zeros(n_rows * max(delta, 0) + 1, dtype=np.int64)
    info = np.zeros(3 * n_rows * max(delta, 0) + 3, dtype=np.int64)
    nrots = ctypes.c_int(0)
    steps = lib().orc_greedy_schedule(n_rows, n_cols, _ptr(job), _ptr(info), ctypes.byref(nrots))
    if steps < 0:
        raise ValueError("bad schedule shape")
    return job[:steps].copy(), info[:3 * nrots.value].copy()


def batched_rq(Z: np.ndarray, n_rows: int, n_cols: int, m_keep: int | None = None):
    """batched.py:93-122 on packed blocks Z (n_rows x s*n_cols) -> (R, P)."""
    Z = np.array(Z, dtype=np.complex128, order="F")
    s = Z.shape[1] // n_cols
    m_keep = n_cols if m_keep is None else m_keep
    P = np.zeros((n_cols, s * m_keep), dtype=np.complex128, order="F")
    rc = lib().orc_batched_rq(n_rows, n_cols, s, _ptr(Z), m_keep, _ptr(P))
    if rc:
        raise ValueError("bad batched_rq arguments")
    return Z, P


def _f64(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def tf_eval(Ahat, Bhat, Chat, shifts, nb: int = 32, rtol: float | None = None,
            threads: int = 0, diag: bool = False):
    """solvers.py:234-271 -> (G p x s*m, fail int32[s] (-1 ok / head index)).

    ``diag=True`` also returns an (s, 3) array per shift: kappa =
    ||Ahat - sigma I||_F / min |R_ii| (SURVEY 8(d) condition estimate), the
    smallest computed head pivot / ||Ahat - sigma I||_F (what the singular
    test compares with rtol) and sum log |R_ii| (log |det(Ahat - sigma I)|)."""
    A, B, C = _f64(Ahat), _f64(Bhat), _f64(Chat)
    n, m, p = A.shape[0], B.shape[1], C.shape[0]
    sh = np.ascontiguousarray(np.asarray(shifts, dtype=np.complex128).ravel())
    s = len(sh)
    G = np.zeros((p, s * m), dtype=np.complex128, order="F")
    fail = np.zeros(s, dtype=np.int32)
    dg = np.zeros((s, 3)) if diag else None
    rc = lib().orc_tf_eval_diag(n, m, p, _ptr(A), A.shape[0], _ptr(B), B.shape[0], _ptr(C),
                                max(C.shape[0], 1), _ptr(sh), s, nb,
                                float("nan") if rtol is None else rtol, _ptr(G), max(p, 1),
                                _ptr(fail), threads, _ptr(dg) if diag else None)
    if rc:
        raise ValueError("bad tf_eval arguments")
    return (G, fail, dg) if diag else (G, fail)


def solve_reduced(Ahat, Bhat, shifts, b_dirs, nb: int = 32, rtol: float | None = None,
                  threads: int = 0, diag: bool = False):
    """solvers.py:274-313 -> (X n x s, fail int32[s]) (+ diag as in tf_eval)."""
    A, B = _f64(Ahat), _f64(Bhat)
    n, m = A.shape[0], B.shape[1]
    sh = np.ascontiguousarray(np.asarray(shifts, dtype=np.complex128).ravel())
    s = len(sh)
    bd = np.asfortranarray(np.asarray(b_dirs, dtype=np.complex128).reshape(m, s))
    X = np.zeros((n, s), dtype=np.complex128, order="F")
    fail = np.zeros(s, dtype=np.int32)
    dg = np.zeros((s, 3)) if diag else None
    rc = lib().orc_solve_reduced_diag(n, m, _ptr(A), n, _ptr(B), B.shape[0], _ptr(sh), s,
                                      _ptr(bd), m, nb, float("nan") if rtol is None else rtol,
                                      _ptr(X), n, _ptr(fail), threads,
                                      _ptr(dg) if diag else None)
    if rc:
        raise ValueError("bad solve_reduced arguments")
    return (X, fail, dg) if diag else (X, fail)


def reduce_chf(A, B, C, accumulate: bool = False):
    """hessenberg.py:260-328 (unblocked) -> (Ahat, Bhat, Chat, Q|None)."""
    Ah = np.array(A, dtype=np.float64, order="F")
    Bh = np.array(B, dtype=np.float64, order="F")
    Ch = np.array(C, dtype=np.float64, order="F")
    n, m, p = Ah.shape[0], Bh.shape[1], Ch.shape[0]
    Q = np.zeros((n, n), order="F") if accumulate else None
    rc = lib().orc_reduce_chf(n, m, p, _ptr(Ah), n, _ptr(Bh), n, _ptr(Ch), max(p, 1),
                              _ptr(Q) if Q is not None else None, n)
    if rc:
        raise ValueError("bad reduce arguments")
    return Ah, Bh, Ch, Q


# ---------------------------------------------------------------------------
# independent dense LU oracle: restatement of oracles.py:28-72
# ---------------------------------------------------------------------------

def lu_solve_shifted(A, sigma, rhs, transpose: bool = False):
    """Row-pivoted LU solve of (A - sigma I) x = rhs (oracles.py:28-66)."""
    n = A.shape[0]
    M = np.asarray(A, dtype=np.complex128) - sigma * np.eye(n)
    if transpose:
        M = M.T.copy()
    M = np.array(M)
    piv = np.arange(n)
    for k in range(n):
        q = k + int(np.argmax(np.abs(M[k:, k])))
        if M[q, k] == 0:
            raise ZeroDivisionError(f"singular at column {k}")
        if q != k:
            M[[k, q], :] = M[[q, k], :]
            piv[[k, q]] = piv[[q, k]]
        M[k + 1:, k] /= M[k, k]
        M[k + 1:, k + 1:] -= np.outer(M[k + 1:, k], M[k, k + 1:])
    b = np.array(rhs, dtype=np.complex128)
    vec = b.ndim == 1
    b = b.reshape(n, -1)[piv, :]
    for k in range(n):
        b[k + 1:, :] -= np.outer(M[k + 1:, k], b[k, :])
    for k in range(n - 1, -1, -1):
        b[k, :] = (b[k, :] - M[k, k + 1:] @ b[k + 1:, :]) / M[k, k]
    return b[:, 0] if vec else b


def oracle_transfer_function(A, B, C, sigma):
    """G(sigma) = C (sigma I - A)^{-1} B via one LU solve (oracles.py:69-72)."""
    X = lu_solve_shifted(A, sigma, np.asarray(B, dtype=np.complex128))
    return -np.asarray(C, dtype=np.complex128) @ X


def random_stable_system(n: int, m: int, p: int, seed: int = 0, margin: float = 0.05):
    """Seeded stable triple, restating systems.py:71-86 (same rng call order)."""
    rng = np.random.default_rng(seed)
    A = np.asfortranarray(rng.standard_normal((n, n)))
    abscissa = float(np.max(np.real(np.linalg.eigvals(A))))
    A -= (abscissa + margin * np.sqrt(n)) * np.eye(n)
    B = np.asfortranarray(rng.standard_normal((n, m)))
    C = np.asfortranarray(rng.standard_normal((p, n)))
    return A, B, C
