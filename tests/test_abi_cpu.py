"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/shiftsolve_b200.h declares, the host schedule matches the
reference's plan, and the Python API validates arguments / fails loudly."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden, has_gpu

import paper_1708_06290_b200 as ss
from paper_1708_06290_b200 import _lib


def header_symbols():
    src = open(os.path.join(ROOT, "include", "shiftsolve_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(ss_[a-z_0-9]+)\s*\(", src))


def test_header_symbols_exported():
    L = _lib.load()
    names = header_symbols()
    assert names == set(_lib.EXPORTED)
    for name in names:
        assert hasattr(L, name), name


def test_library_is_sm100a():
    so = _lib.LIB_PATH
    data = open(so, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_dmma_only_in_the_reduction():
    """north_star: FP64 tensor-core DMMA only in the reduction's trailing
    updates.  Every kernel of the product library whose SASS holds a DMMA
    must be the reduction GEMM (ssr::k_dmma); the sweep is DFMA."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    with_dmma, fn = set(), None
    for line in sass.splitlines():
        if "Function :" in line:
            fn = line.split("Function :")[1].strip()
        elif "DMMA" in line and fn:
            with_dmma.add(fn)
    assert with_dmma, "the reduction GEMM should use DMMA"
    assert all("k_dmma" in f for f in with_dmma), sorted(f for f in with_dmma if "k_dmma" not in f)


def test_version():
    assert _lib.load().ss_version() == 100


def test_native_schedule_matches_reference():
    g = golden("schedules.npz")
    for nr, nc in g["shapes"]:
        s = ss.greedy_schedule(int(nr), int(nc))
        assert np.array_equal(s.job_size, g[f"job_{nr}_{nc}"])
        assert np.array_equal(s.rot_info, g[f"info_{nr}_{nc}"])


def test_schedule_counts_and_hand_trace():
    s = ss.greedy_schedule(8, 14)
    assert s.num_steps == 13 and s.num_rots == 48
    assert ss.greedy_schedule(5, 5).num_rots == 0
    steps = list(ss.greedy_schedule(1, 3).steps())
    assert steps == [[(1, 1, 3)], [(1, 2, 3)]]
    with pytest.raises(ValueError):
        ss.greedy_schedule(3, 2)


def test_schedule_properties_appendix_a():
    """steps / max parallel width at nb = 64."""
    for m, steps, width in [(1, 64, 1), (5, 68, 5), (10, 73, 10), (20, 83, 20), (50, 113, 42)]:
        s = ss.greedy_schedule(64, 64 + m)
        assert s.num_steps == steps and int(s.job_size.max()) == width
        assert s.num_rots == 64 * m


def test_abi_rejects_bad_arguments_without_device():
    L = _lib.load()
    job = np.zeros(4, dtype=np.int64)
    info = np.zeros(12, dtype=np.int64)
    st, rt = ctypes.c_int(), ctypes.c_int()
    assert L.ss_greedy_schedule(3, 2, job.ctypes.data_as(ctypes.c_void_p), 4,
                                info.ctypes.data_as(ctypes.c_void_p), 12,
                                ctypes.byref(st), ctypes.byref(rt)) == _lib.SS_EDIM
    # null handle -> SS_EARG, never a crash
    assert L.ss_tf_eval(None, 4, 1, 1, None, 4, None, 4, None, 1, None, 0, 4, 0, 0.0, None, 1,
                        None, None) == _lib.SS_EARG


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    chf = ss.ControllerHessForm(Ahat=np.array([[1.5]]), Bhat=np.array([[2.0]]),
                                Chat=np.array([[3.0]]), m=1, n=1, p=1)
    with pytest.raises(RuntimeError):
        ss.eval_transfer_function(chf, [2.0 + 0.5j], nb=4)
    with pytest.raises(RuntimeError):
        ss.reduce_controller_hessenberg(np.eye(3), np.ones((3, 1)), np.ones((1, 3)))


def test_argument_validation_before_device():
    chf = ss.ControllerHessForm(Ahat=np.eye(4), Bhat=np.ones((4, 1)), Chat=np.ones((1, 4)),
                                m=1, n=4, p=1)
    with pytest.raises(ValueError):
        ss.eval_transfer_function(chf, [1j], nb=0)
    bad = ss.ControllerHessForm(Ahat=np.eye(4), Bhat=np.ones((3, 1)), Chat=np.ones((1, 4)),
                                m=1, n=4, p=1)
    with pytest.raises(ss.DimensionMismatchError):
        ss.eval_transfer_function(bad, [1j])
    with pytest.raises(ss.DimensionMismatchError):
        ss.solve_shifted_reduced(chf, [1j, 2j], np.ones((1, 3)))
    with pytest.raises(ss.DimensionMismatchError):
        ss.reduce_controller_hessenberg(np.eye(3), np.ones((4, 1)), np.ones((1, 3)))
    with pytest.raises(ss.DimensionMismatchError):
        ss.reduce_controller_hessenberg(np.eye(3), np.ones((3, 3)), np.ones((1, 3)))
    with pytest.raises(ValueError):
        ss.reduce_controller_hessenberg(np.eye(3), np.ones((3, 1)), np.ones((1, 3)),
                                        strategy="bogus")


def test_error_types_mirror_reference():
    assert issubclass(ss.DimensionMismatchError, ValueError)
    e = ss.SingularShiftError([(3, 1), (1, 0)])
    assert e.failures == [(3, 1), (1, 0)] and "[1, 3]" in str(e)
    assert issubclass(ss.SingularShiftError, ArithmeticError)


def test_mirrored_schedule_matches_reference():
    """schedule.py:162-184 mirrored_schedule, bitwise against the reference's
    plans (tests/golden/transposed.npz) and the (3, 5) targets of
    test_schedule.py:106-120 (superdiagonal band, helpers to the left)."""
    g = golden("transposed.npz")
    for nr, nc in [(3, 5), (8, 14), (16, 26), (32, 42), (64, 74)]:
        sch = ss.mirrored_schedule(nr, nc)
        assert np.array_equal(np.asarray(sch.job_size), g[f"ms_{nr}_{nc}_job"])
        assert np.array_equal(np.asarray(sch.rot_info), g[f"ms_{nr}_{nc}_info"])
    sch = ss.mirrored_schedule(3, 5)
    for r, c1, c2 in np.asarray(sch.rot_info).reshape(-1, 3):
        assert c2 < c1 and c1 > r  # target above the diagonal, helper to its left
