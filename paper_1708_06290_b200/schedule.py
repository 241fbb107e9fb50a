"""Greedy step-parallel Givens annihilation plans (host precompute).

``greedy_schedule`` keeps the reference's name, result type and exact plan
(schedule.py:88-159); it is computed by the native host code of
libshiftsolve_b200.so (csrc/ss_api.cu, the same function the CUDA driver
uploads to the device) and cached per shape like the reference's lru_cache.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _lib


@dataclass(frozen=True)
class AnnihilationSchedule:
    """Step-grouped plan for one block shape (reference schedule.py:27-76):
    ``rot_info`` holds 1-based (r, c1, c2) triplets in execution order,
    ``job_size[t]`` the rotation count of step t."""

    n_rows: int
    n_cols: int
    num_steps: int
    num_rots: int
    job_size: np.ndarray
    rot_info: np.ndarray

    def steps(self):
        off = 0
        for size in self.job_size:
            yield [tuple(int(v) for v in self.rot_info[3 * k:3 * k + 3])
                   for k in range(off, off + int(size))]
            off += int(size)


@lru_cache(maxsize=None)
def greedy_schedule(n_rows: int, n_cols: int) -> AnnihilationSchedule:
    if n_rows < 1:
        raise ValueError("n_rows must be positive")
    if n_cols < n_rows:
        raise ValueError("n_cols must be at least n_rows")
    delta = n_cols - n_rows
    cap = n_rows * delta
    job = np.zeros(cap + 1, dtype=np.int64)
    info = np.zeros(3 * cap + 3, dtype=np.int64)
    steps, rots = ctypes.c_int(0), ctypes.c_int(0)
    rc = _lib.load().ss_greedy_schedule(n_rows, n_cols, job.ctypes.data_as(ctypes.c_void_p),
                                        len(job), info.ctypes.data_as(ctypes.c_void_p), len(info),
                                        ctypes.byref(steps), ctypes.byref(rots))
    if rc != _lib.SS_OK:
        raise ValueError("bad schedule shape")
    job = job[:steps.value].copy()
    info = info[:3 * rots.value].copy()
    job.setflags(write=False)
    info.setflags(write=False)
    return AnnihilationSchedule(n_rows, n_cols, steps.value, rots.value, job, info)


@lru_cache(maxsize=None)
def mirrored_schedule(n_rows: int, n_cols: int) -> AnnihilationSchedule:
    """Top-down plan for lower trapezoids (reference schedule.py:162-184): the
    greedy plan flipped in both axes, (r, c1, c2) -> (nr+1-r, nc+1-c1,
    nc+1-c2), same step structure."""
    base = greedy_schedule(n_rows, n_cols)
    info = np.asarray(base.rot_info).reshape(-1, 3).copy()
    info[:, 0] = n_rows + 1 - info[:, 0]
    info[:, 1:] = n_cols + 1 - info[:, 1:]
    info = info.reshape(-1)
    info.setflags(write=False)
    return AnnihilationSchedule(base.n_rows, base.n_cols, base.num_steps, base.num_rots,
                                base.job_size, info)
