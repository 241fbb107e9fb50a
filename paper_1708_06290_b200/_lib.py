"""ctypes binding of libshiftsolve_b200.so (include/shiftsolve_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  There is deliberately no CPU fallback: if the library or a CUDA
device is missing every solver raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SS_LIB_PATH") or os.path.join(_HERE, "libshiftsolve_b200.so")

SS_OK, SS_EDIM, SS_EARG, SS_ECUDA, SS_ENOMEM = 0, 1, 2, 3, 4

#: every symbol include/shiftsolve_b200.h declares
EXPORTED = (
    "ss_version", "ss_create", "ss_destroy", "ss_last_error", "ss_greedy_schedule",
    "ss_tf_eval", "ss_tf_eval_stream", "ss_pspec_eval", "ss_solve_reduced", "ss_solve_transposed", "ss_reduce_chf", "ss_set_timing", "ss_phase_stats",
    "ss_reset_stats", "ss_launch_count", "ss_update_kernel_stats", "ss_probe_dfma_peak", "ss_probe_dmma_peak", "ss_dgemm",
)

_lib = None
_lock = threading.Lock()
_tls = threading.local()


def load():
    """Load and prototype the library (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P, I, I64, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
        L.ss_version.restype = I
        L.ss_create.argtypes = [ctypes.POINTER(P), I]
        L.ss_create.restype = I
        L.ss_destroy.argtypes = [P]
        L.ss_destroy.restype = None
        L.ss_last_error.argtypes = [P]
        L.ss_last_error.restype = ctypes.c_char_p
        L.ss_greedy_schedule.argtypes = [I, I, P, I64, P, I64, ctypes.POINTER(I), ctypes.POINTER(I)]
        L.ss_greedy_schedule.restype = I
        L.ss_tf_eval.argtypes = [P, I, I, I, P, I64, P, I64, P, I64, P, I64, I, I64, D, P, I64, P, P]
        L.ss_tf_eval.restype = I
        L.ss_solve_reduced.argtypes = [P, I, I, P, I64, P, I64, P, I64, P, I64, I, I64, D, P, I64,
                                       P, P]
        L.ss_solve_reduced.restype = I
        L.ss_tf_eval_stream.argtypes = [P, I, I, I, P, I64, P, I64, P, I64, P, I64, P, I64, I, I64,
                                        D, P, I64, P, P]
        L.ss_tf_eval_stream.restype = I
        L.ss_pspec_eval.argtypes = [P, I, I, I, P, I64, P, I64, P, I64, P, I64, I, I64, D, P, I64,
                                    P, P, P]
        L.ss_pspec_eval.restype = I
        L.ss_solve_transposed.argtypes = [P, I, I, P, I64, P, I64, P, I64, I, I64, D, P, I64, P, P]
        L.ss_solve_transposed.restype = I
        L.ss_reduce_chf.argtypes = [P, I, I, I, P, I64, P, I64, P, I64, P, I64, I, P]
        L.ss_reduce_chf.restype = I
        L.ss_set_timing.argtypes = [P, I]
        L.ss_set_timing.restype = I
        L.ss_phase_stats.argtypes = [P, P, P]
        L.ss_phase_stats.restype = I
        L.ss_reset_stats.argtypes = [P]
        L.ss_reset_stats.restype = None
        L.ss_launch_count.argtypes = [P]
        L.ss_launch_count.restype = ctypes.c_int64
        L.ss_update_kernel_stats.argtypes = [P, P, P, P]
        L.ss_update_kernel_stats.restype = I
        L.ss_probe_dfma_peak.argtypes = [P, P]
        L.ss_probe_dfma_peak.restype = I
        L.ss_probe_dmma_peak.argtypes = [P, P]
        L.ss_probe_dmma_peak.restype = I
        L.ss_dgemm.argtypes = [P, I, I, I, I, I, D, P, I64, P, I64, D, P, I64, P]
        L.ss_dgemm.restype = I
        _lib = L
    return _lib


class Handle:
    """Owns one ss_handle (device workspace + cached schedules)."""

    def __init__(self, device: int):
        L = load()
        h = ctypes.c_void_p()
        rc = L.ss_create(ctypes.byref(h), int(device))
        if rc != SS_OK:
            raise RuntimeError(f"ss_create(device={device}) failed with code {rc} "
                               "(no usable CUDA device?)")
        self.ptr = h
        self.device = int(device)

    def error(self) -> str:
        return load().ss_last_error(self.ptr).decode()

    def launches(self) -> int:
        return int(load().ss_launch_count(self.ptr))

    def __del__(self):
        try:
            if getattr(self, "ptr", None):
                load().ss_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass


def handle(device: int) -> Handle:
    """Per-thread, per-device handle (the C handle is not thread safe)."""
    hs = getattr(_tls, "handles", None)
    if hs is None:
        hs = _tls.handles = {}
    h = hs.get(device)
    if h is None:
        h = hs[device] = Handle(device)
    return h


def all_handles():
    return list(getattr(_tls, "handles", {}).values())
