"""Drop-in batched shifted solvers on controller-Hessenberg data (B200).

Same names, signatures, result types, error behaviour and phase counters as
the reference's solvers.py (``eval_transfer_function`` :234-271,
``solve_shifted_reduced`` :274-313, ``solve_shifted_transposed`` :320-486,
``structured_pseudospectrum_grid`` :508-530); the window sweep, the batched Givens RQ and the head solve run
inside libshiftsolve_b200.so (csrc/ss_sweep.cu) on the GPU.

Behaviour kept from the reference:
  * ``G = -Chat (Ahat - sigma I)^{-1} Bhat`` (solvers.py:267), slice l of G
    is the p x m value at ``shifts[l]``;
  * a shift whose head pivot is <= ``rtol * ||Ahat - sigma I||_F`` with
    ``rtol = 1e3 n eps`` (solvers.py:95-97) is recorded in ``failures``
    (shift index -> 0-based pivot index) with a NaN slice; the other shifts
    are unaffected (bitwise: each shift is computed in isolation);
  * ``on_singular="raise"`` raises ``SingularShiftError`` after ALL shifts;
  * ``nb < 1`` raises ``ValueError``; shape problems raise
    ``DimensionMismatchError``.
Differences: ``pool`` is accepted and ignored (the GPU replaces the worker
pools); ``batch_size`` only bounds device memory (results do not depend on
it); ``nb`` is clamped to what one SM's shared memory holds for the given m.

Inputs may be numpy arrays (results come back as numpy) or torch tensors
(results stay on the tensors' device).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as D
from . import _lib
from .counters import PhaseCounters
from .errors import DimensionMismatchError, SingularShiftError
from .hessenberg import ControllerHessForm

EPS = float(np.finfo(np.float64).eps)


@dataclass
class TransferFunctionResult:
    """Slice l of ``G`` is the p x m value at ``shifts[l]``; ``failures`` maps
    shift index to the pivot row that flagged it singular (reference
    solvers.py:71-83)."""

    G: object
    shifts: object
    failures: dict[int, int] = field(default_factory=dict)

    def value(self, l: int):
        m = self.G.shape[1] // len(self.shifts)
        return self.G[:, l * m:(l + 1) * m]


@dataclass
class ShiftedSolveResult:
    """Solutions of a batch of shifted systems, one column per shift
    (reference solvers.py:86-92)."""

    x: object
    shifts: object
    failures: dict[int, int] = field(default_factory=dict)


def default_singular_rtol(n: int) -> float:
    """Relative pivot threshold below which a shift is singular (solvers.py:95-97)."""
    return 1e3 * n * EPS


def _check_chf(chf: ControllerHessForm) -> None:
    """solvers.py:113-115."""
    if tuple(chf.Ahat.shape) != (chf.n, chf.n) or chf.Bhat.shape[0] != chf.n:
        raise DimensionMismatchError("inconsistent controller-Hessenberg form")
    if chf.m < 1 or chf.m > chf.n or chf.Bhat.shape[1] < chf.m:
        raise DimensionMismatchError("inconsistent controller-Hessenberg form")
    if chf.Chat.shape[1] != chf.n or chf.Chat.shape[0] != chf.p:
        raise DimensionMismatchError("inconsistent controller-Hessenberg form")


def _batch(batch_size) -> int:
    return 0 if batch_size is None else max(1, int(batch_size))


def _shifts_in(shifts):
    if isinstance(shifts, torch.Tensor):
        return shifts.reshape(-1).to(torch.complex128)
    return np.asarray(shifts, dtype=np.complex128).ravel()


def _failures(fail: torch.Tensor) -> dict[int, int]:
    f = fail.cpu().numpy()
    bad = np.nonzero(f >= 0)[0]
    return {int(l): int(f[l]) for l in bad}


def eval_transfer_function(chf: ControllerHessForm, shifts, nb: int = 32,
                           batch_size: int | None = None, *, pool=None,
                           counter: PhaseCounters | None = None,
                           on_singular: str = "raise",
                           singular_rtol: float | None = None) -> TransferFunctionResult:
    """Values of C (sigma I - A)^{-1} B for every shift (solvers.py:234-271)."""
    del pool  # the GPU replaces the reference's worker pools
    _check_chf(chf)
    shifts = _shifts_in(shifts)
    n, m, p = chf.n, chf.m, chf.p
    if nb < 1:
        raise ValueError("window block size must be >= 1")
    rtol = default_singular_rtol(n) if singular_rtol is None else float(singular_rtol)
    s = len(shifts)
    host = all(D.is_host(a) for a in (chf.Ahat, chf.Bhat, chf.Chat, shifts))
    dev = D.device_of(chf.Ahat, chf.Bhat, chf.Chat, shifts)
    # A column-major, pinned host Ahat is streamed to the device in the order
    # the sweep consumes its columns (right to left, one outer block at a
    # time) on a copy stream, overlapped with the sweep (ss_tf_eval_stream)
    Ah = chf.Ahat
    stream_a = (isinstance(Ah, torch.Tensor) and Ah.device.type == "cpu" and Ah.is_pinned()
                and Ah.dtype == torch.float64 and Ah.stride(0) == 1 and Ah.stride(1) >= n)
    with torch.cuda.device(dev):
        if stream_a:
            A = torch.empty((n, n), dtype=torch.float64, device=dev).t()
        else:
            A = D.fmat(Ah, torch.float64, dev)
        B = D.fmat(chf.Bhat, torch.float64, dev)
        C = D.fmat(chf.Chat, torch.float64, dev)
        sh = D.fvec(shifts, torch.complex128, dev)
        G = torch.empty((s * m, max(p, 1)), dtype=torch.complex128, device=dev).t()[:p, :]
        fail = torch.empty(s, dtype=torch.int32, device=dev)
        h = _lib.handle(dev.index)
        L = _lib.load()
        with D.timed_call(h, counter):
            if stream_a:
                rc = L.ss_tf_eval_stream(h.ptr, n, m, p, Ah.data_ptr(), Ah.stride(1), D.ptr(A), n,
                                         D.ptr(B), D.ld(B), D.ptr(C), D.ld(C), D.ptr(sh), s,
                                         int(nb), _batch(batch_size), rtol, D.ptr(G), max(p, 1),
                                         D.ptr(fail), D.stream_ptr(dev))
            else:
                rc = L.ss_tf_eval(h.ptr, n, m, p, D.ptr(A), D.ld(A), D.ptr(B), D.ld(B), D.ptr(C),
                                  D.ld(C), D.ptr(sh), s, int(nb), _batch(batch_size), rtol,
                                  D.ptr(G), max(p, 1), D.ptr(fail), D.stream_ptr(dev))
        D.check(h, rc)
        failures = _failures(fail)
    Gout = G.cpu().numpy() if host else G
    if failures and on_singular == "raise":
        raise SingularShiftError(sorted((l, i) for l, i in failures.items()))
    return TransferFunctionResult(G=Gout, shifts=shifts, failures=failures)


def solve_shifted_reduced(chf: ControllerHessForm, shifts, b_dirs, nb: int = 32,
                          batch_size: int | None = None, *, pool=None,
                          counter: PhaseCounters | None = None,
                          on_singular: str = "raise",
                          singular_rtol: float | None = None) -> ShiftedSolveResult:
    """Solve (A - sigma_l I) x_l = B bhat_l for every shift (solvers.py:274-313)."""
    del pool
    _check_chf(chf)
    shifts = _shifts_in(shifts)
    n, m = chf.n, chf.m
    s = len(shifts)
    if tuple(b_dirs.shape) != (m, s):
        raise DimensionMismatchError("b_dirs must be m x s")
    if nb < 1:
        raise ValueError("window block size must be >= 1")
    rtol = default_singular_rtol(n) if singular_rtol is None else float(singular_rtol)
    host = all(D.is_host(a) for a in (chf.Ahat, chf.Bhat, shifts, b_dirs))
    dev = D.device_of(chf.Ahat, chf.Bhat, shifts, b_dirs)
    with torch.cuda.device(dev):
        A = D.fmat(chf.Ahat, torch.float64, dev)
        B = D.fmat(chf.Bhat, torch.float64, dev)
        bd = D.fmat(b_dirs, torch.complex128, dev)
        sh = D.fvec(shifts, torch.complex128, dev)
        X = torch.empty((s, n), dtype=torch.complex128, device=dev).t()
        fail = torch.empty(s, dtype=torch.int32, device=dev)
        h = _lib.handle(dev.index)
        L = _lib.load()
        with D.timed_call(h, counter):
            rc = L.ss_solve_reduced(h.ptr, n, m, D.ptr(A), D.ld(A), D.ptr(B), D.ld(B), D.ptr(sh),
                                    s, D.ptr(bd), D.ld(bd), int(nb), _batch(batch_size), rtol,
                                    D.ptr(X), n, D.ptr(fail), D.stream_ptr(dev))
        D.check(h, rc)
        failures = _failures(fail)
    Xout = X.cpu().numpy() if host else X
    if failures and on_singular == "raise":
        raise SingularShiftError(sorted((l, i) for l, i in failures.items()))
    return ShiftedSolveResult(x=Xout, shifts=shifts, failures=failures)


def solve_shifted_transposed(chf: ControllerHessForm, shifts, rhs, nb: int = 32,
                             batch_size: int | None = None, *, pool=None,
                             counter: PhaseCounters | None = None,
                             on_singular: str = "raise",
                             singular_rtol: float | None = None) -> ShiftedSolveResult:
    """Solve (A - sigma_l I)^T x_l = c_l for general right-hand sides
    (solvers.py:320-355): top-down windowed LQ of [A^T - sigma I; -I] with the
    forward substitution fused into the sweep (csrc/ss_lq.cu).  Every pivot
    of the LQ factor is checked against ``rtol * ||Ahat - sigma I||_F``; a
    failing shift gets a NaN column and its first failing row in
    ``failures``.  ``nb`` is clamped to 32 (and, for m + 1 > 32, to what the
    shared-memory window of csrc/ss_lq.cu:k_lq_big holds); m + 1 <= 256."""
    del pool
    _check_chf(chf)
    shifts = _shifts_in(shifts)
    n, m = chf.n, chf.m
    s = len(shifts)
    if tuple(rhs.shape) != (n, s):
        raise DimensionMismatchError("rhs must be n x s")
    if nb < 1:
        raise ValueError("window block size must be >= 1")
    rtol = default_singular_rtol(n) if singular_rtol is None else float(singular_rtol)
    host = all(D.is_host(a) for a in (chf.Ahat, shifts, rhs))
    dev = D.device_of(chf.Ahat, shifts, rhs)
    with torch.cuda.device(dev):
        A = D.fmat(chf.Ahat, torch.float64, dev)
        c = D.fmat(rhs, torch.complex128, dev)
        sh = D.fvec(shifts, torch.complex128, dev)
        X = torch.empty((s, n), dtype=torch.complex128, device=dev).t()
        fail = torch.empty(s, dtype=torch.int32, device=dev)
        h = _lib.handle(dev.index)
        L = _lib.load()
        with D.timed_call(h, counter):
            rc = L.ss_solve_transposed(h.ptr, n, m, D.ptr(A), D.ld(A), D.ptr(sh), s, D.ptr(c),
                                       D.ld(c), int(nb), _batch(batch_size), rtol, D.ptr(X), n,
                                       D.ptr(fail), D.stream_ptr(dev))
        D.check(h, rc)
        failures = _failures(fail)
    Xout = X.cpu().numpy() if host else X
    if failures and on_singular == "raise":
        raise SingularShiftError(sorted((l, i) for l, i in failures.items()))
    return ShiftedSolveResult(x=Xout, shifts=shifts, failures=failures)


def two_norm_small(M) -> float:
    """Spectral norm of a small dense matrix (solvers.py:501-505)."""
    M = np.asarray(M)
    if M.size == 0:
        return 0.0
    return float(np.linalg.svd(M, compute_uv=False)[0])


def structured_pseudospectrum_grid(chf: ControllerHessForm, grid, nb: int = 32,
                                   batch_size: int | None = None, *, pool=None,
                                   counter: PhaseCounters | None = None,
                                   singular_rtol: float | None = None):
    """||C (z I - A)^{-1} B||_2 over grid points; singular points -> +inf
    (solvers.py:508-530).  The spectral norms of the p x m values come from a
    device epilogue of the sweep (``ss_pspec_eval``: Gram matrix + Hermitian
    Jacobi per point) instead of the reference's numpy SVD."""
    del pool
    _check_chf(chf)
    grid = _shifts_in(grid)
    n, m, p = chf.n, chf.m, chf.p
    s = len(grid)
    if nb < 1:
        raise ValueError("window block size must be >= 1")
    rtol = default_singular_rtol(n) if singular_rtol is None else float(singular_rtol)
    host = all(D.is_host(a) for a in (chf.Ahat, chf.Bhat, chf.Chat, grid))
    dev = D.device_of(chf.Ahat, chf.Bhat, chf.Chat, grid)
    if s == 0 or p == 0:
        # empty values: ||.||_2 = 0 (two_norm_small), +inf where the shift is singular
        res = eval_transfer_function(chf, grid, nb=nb, batch_size=batch_size, counter=counter,
                                     on_singular="mark", singular_rtol=singular_rtol)
        out = torch.zeros(s, dtype=torch.float64, device=dev)
        if res.failures:
            out[torch.tensor(sorted(res.failures), device=dev)] = float("inf")
        return out.cpu().numpy() if host else out
    with torch.cuda.device(dev):
        A = D.fmat(chf.Ahat, torch.float64, dev)
        B = D.fmat(chf.Bhat, torch.float64, dev)
        C = D.fmat(chf.Chat, torch.float64, dev)
        sh = D.fvec(grid, torch.complex128, dev)
        G = torch.empty((s * m, p), dtype=torch.complex128, device=dev).t()
        norms = torch.empty(s, dtype=torch.float64, device=dev)
        fail = torch.empty(s, dtype=torch.int32, device=dev)
        h = _lib.handle(dev.index)
        L = _lib.load()
        with D.timed_call(h, counter):
            rc = L.ss_pspec_eval(h.ptr, n, m, p, D.ptr(A), D.ld(A), D.ptr(B), D.ld(B), D.ptr(C),
                                 D.ld(C), D.ptr(sh), s, int(nb), _batch(batch_size), rtol,
                                 D.ptr(G), p, D.ptr(norms), D.ptr(fail), D.stream_ptr(dev))
        D.check(h, rc)
    return norms.cpu().numpy() if host else norms


def residual_certificate(chf: ControllerHessForm, sigma: complex, x, rhs,
                         transpose: bool = False) -> float:
    """||(A - sigma I) x - rhs|| / (||A - sigma I||_F ||x|| + ||rhs||)
    (solvers.py:489-498); host-side test helper."""
    A = np.asarray(chf.Ahat.cpu() if isinstance(chf.Ahat, torch.Tensor) else chf.Ahat)
    M = A - sigma * np.eye(chf.n)
    if transpose:
        M = M.T
    x = np.asarray(x)
    rhs = np.asarray(rhs)
    num = np.linalg.norm(M @ x - rhs)
    den = np.linalg.norm(M, "fro") * np.linalg.norm(x) + np.linalg.norm(rhs)
    return float(num / den) if den else float(num)
