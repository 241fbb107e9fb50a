"""Device plumbing: torch owns device memory and streams, the C ABI does the
math.  Inputs may be numpy arrays or torch tensors (CPU or CUDA); they are
staged into column-major device tensors with explicit leading dimensions
(the reference's storage convention, kernels.py:1-11)."""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .counters import ALL_PHASES, PhaseCounters
from .errors import DeviceError, DimensionMismatchError


def device_of(*arrays) -> torch.device:
    """CUDA device to run on: that of the first CUDA tensor, else current."""
    for a in arrays:
        if isinstance(a, torch.Tensor) and a.is_cuda:
            return a.device
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1708_06290_b200 needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def is_host(a) -> bool:
    return not (isinstance(a, torch.Tensor) and a.is_cuda)


def fmat(a, dtype: torch.dtype, dev: torch.device, min_rows: int = 1) -> torch.Tensor:
    """Column-major device copy (or view) of a 2-D array; ld = stride(1)."""
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.asarray(a))
    if t.ndim == 1:
        t = t.reshape(-1, 1)
    if t.ndim != 2:
        raise DimensionMismatchError("expected a matrix")
    if t.dtype != dtype:
        t = t.to(dtype)
    rows, cols = t.shape
    if (t.device == dev and t.stride(0) == 1 and t.stride(1) >= max(rows, min_rows)
            and cols > 0):
        return t
    out = torch.empty((cols, max(rows, min_rows)), dtype=dtype, device=dev).t()[:rows, :]
    out.copy_(t, non_blocking=True)
    return out


def fvec(a, dtype: torch.dtype, dev: torch.device) -> torch.Tensor:
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(a)))
    t = t.reshape(-1)
    if t.dtype != dtype:
        t = t.to(dtype)
    if t.device != dev or not t.is_contiguous():
        t = t.to(dev, non_blocking=True).contiguous()
    return t


def ld(t: torch.Tensor) -> int:
    """Leading dimension of a column-major device matrix."""
    return max(int(t.stride(1)), int(t.shape[0]), 1)


def ptr(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() > 0 else None


def stream_ptr(dev: torch.device):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def check(h: _lib.Handle, rc: int) -> None:
    if rc == _lib.SS_OK:
        return
    msg = h.error()
    if rc == _lib.SS_EDIM:
        raise DimensionMismatchError(msg)
    if rc == _lib.SS_EARG:
        raise ValueError(msg)
    raise DeviceError(f"{msg} (code {rc})")


class timed_call:
    """Enable library event timing while a PhaseCounters is attached and fold
    the per-phase seconds/flops of this call into it."""

    def __init__(self, h: _lib.Handle, counter: PhaseCounters | None):
        self.h, self.counter = h, counter

    def __enter__(self):
        L = _lib.load()
        L.ss_reset_stats(self.h.ptr)
        L.ss_set_timing(self.h.ptr, 1 if self.counter is not None else 0)
        return self

    def __exit__(self, *exc):
        L = _lib.load()
        if self.counter is not None and exc[0] is None:
            sec = (ctypes.c_double * 5)()
            fl = (ctypes.c_double * 5)()
            L.ss_phase_stats(self.h.ptr, sec, fl)
            for i, ph in enumerate(ALL_PHASES):
                if fl[i] or sec[i]:
                    self.counter.add(ph, fl[i])
                    self.counter.add_seconds(ph, sec[i])
        L.ss_set_timing(self.h.ptr, 0)
        return False
