"""Controller-Hessenberg form and its one-time GPU reduction.

``ControllerHessForm`` mirrors the reference dataclass (hessenberg.py:53-67).
``reduce_controller_hessenberg`` keeps the reference signature
(hessenberg.py:260-265) and runs the blocked Householder reduction of
csrc/ss_reduce.cu on the GPU (there is no CPU path).  ``strategy``,
``pool_panel`` and ``pool_update`` are accepted for compatibility: the
reference's "overlapped" strategy overlaps task (c) with the next panel on a
second CPU thread; on the GPU both strategies run the same stream-ordered
kernels and give bitwise identical results, as the reference promises for
its two strategies (hessenberg.py:27-31).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _lib
from .counters import PhaseCounters
from .errors import DimensionMismatchError


@dataclass
class ControllerHessForm:
    """Reduced triple: banded-Hessenberg Ahat, upper-triangular Bhat, dense
    Chat (exact zero patterns); Q^T A Q = Ahat when Q is accumulated."""

    Ahat: object
    Bhat: object
    Chat: object
    m: int
    n: int
    p: int
    Q: object | None = None

    def to(self, device) -> "ControllerHessForm":
        """Device-resident copy (column-major torch tensors) for repeated solves."""
        dev = torch.device(device)
        return ControllerHessForm(
            Ahat=D.fmat(self.Ahat, torch.float64, dev), Bhat=D.fmat(self.Bhat, torch.float64, dev),
            Chat=D.fmat(self.Chat, torch.float64, dev), m=self.m, n=self.n, p=self.p,
            Q=None if self.Q is None else D.fmat(self.Q, torch.float64, dev))

    def numpy(self) -> "ControllerHessForm":
        def h(a):
            return a if a is None or isinstance(a, np.ndarray) else np.asfortranarray(a.cpu().numpy())
        return ControllerHessForm(Ahat=h(self.Ahat), Bhat=h(self.Bhat), Chat=h(self.Chat),
                                  m=self.m, n=self.n, p=self.p, Q=h(self.Q))


def _shape(a):
    return tuple(a.shape)


def reduce_controller_hessenberg(A, B, C, block_size: int = 64, strategy: str = "sequential", *,
                                 accumulate: bool = False, pool_panel=None, pool_update=None,
                                 counter: PhaseCounters | None = None) -> ControllerHessForm:
    """Orthogonally reduce (A, B, C): QR of B, similarity on A, band reduction
    of A with band width m = B.shape[1], and the matching right updates of C
    (hessenberg.py:260-328).  Inputs are never modified."""
    del pool_panel, pool_update
    if strategy not in ("sequential", "overlapped"):
        raise ValueError("strategy must be 'sequential' or 'overlapped'")
    if len(_shape(A)) != 2 or _shape(A)[0] != _shape(A)[1]:
        raise DimensionMismatchError("A must be square")
    n = _shape(A)[0]
    if len(_shape(B)) != 2 or _shape(B)[0] != n:
        raise DimensionMismatchError("B must have as many rows as A")
    if len(_shape(C)) != 2 or _shape(C)[1] != n:
        raise DimensionMismatchError("C must have as many columns as A")
    m, p = _shape(B)[1], _shape(C)[0]
    if not 1 <= m < n:
        raise DimensionMismatchError("need 1 <= m < n (inputs vs state dimension)")
    if block_size < 1:
        raise ValueError("block_size must be positive")
    host = all(D.is_host(a) for a in (A, B, C))
    dev = D.device_of(A, B, C)
    with torch.cuda.device(dev):
        # private column-major copies (the reference copies too, hessenberg.py:289-291)
        Ah = torch.empty((n, n), dtype=torch.float64, device=dev).t()
        Ah.copy_(A if isinstance(A, torch.Tensor) else torch.from_numpy(np.asarray(A, dtype=np.float64)))
        Bh = torch.empty((m, n), dtype=torch.float64, device=dev).t()
        Bh.copy_(B if isinstance(B, torch.Tensor) else torch.from_numpy(np.asarray(B, dtype=np.float64)))
        Ch = torch.empty((n, max(p, 1)), dtype=torch.float64, device=dev).t()[:p, :]
        if p:
            Ch.copy_(C if isinstance(C, torch.Tensor) else torch.from_numpy(np.asarray(C, dtype=np.float64)))
        Q = torch.empty((n, n), dtype=torch.float64, device=dev).t() if accumulate else None
        h = _lib.handle(dev.index)
        L = _lib.load()
        with D.timed_call(h, counter):
            rc = L.ss_reduce_chf(h.ptr, n, m, p, D.ptr(Ah), n, D.ptr(Bh), n, D.ptr(Ch),
                                 max(p, 1), D.ptr(Q), n, int(block_size), D.stream_ptr(dev))
        D.check(h, rc)
    chf = ControllerHessForm(Ahat=Ah, Bhat=Bh, Chat=Ch, m=m, n=n, p=p, Q=Q)
    return chf.numpy() if host else chf
