import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def probe_shifts(rng, count, scale=1.0):
    """Complex probes kept off the real axis (reference tests/conftest.py:17-22)."""
    re = rng.uniform(-0.5, 1.5, count) * scale
    im = rng.uniform(0.4, 2.5, count) * scale * np.where(rng.uniform(size=count) < 0.5, -1, 1)
    return re + 1j * im


def bounded_shifts(rng, Ahat, count, cap=1e4):
    """test_acceptance.py:45-54 shifts_with_bounded_condition."""
    n = Ahat.shape[0]
    scale = np.linalg.norm(Ahat, "fro") / np.sqrt(n)
    out = []
    while len(out) < count:
        sig = complex(rng.uniform(-1, 1) * scale, rng.uniform(0.2, 2.0) * scale)
        if np.linalg.cond(Ahat - sig * np.eye(n)) <= cap:
            out.append(sig)
    return np.asarray(out)


EPS = float(np.finfo(np.float64).eps)


def shift_tolerance(n: int, kappa: float) -> float:
    """SURVEY 8(d) per-shift parity bound: max(1e-10, 10 n eps kappa), kappa =
    ||Ahat - sigma I||_F / min |R_ii| (from the oracle's sweep)."""
    return max(1e-10, 10.0 * n * EPS * kappa)


def assert_shift_parity(Y, fail, Y_ref, fail_ref, diag, n, cols_per_shift, rtol=None):
    """Per-shift parity of GPU results against the oracle on the same shifts.

    Y, Y_ref: (rows, s * cols_per_shift) arrays; fail, fail_ref: -1 or the
    failing pivot per shift; diag: the oracle's (s, 3) diagnostics.  A shift
    passes when both succeeded and ||Y_l - Yref_l||_F / ||Yref_l||_F <=
    max(1e-10, 10 n eps kappa_l), or both failed; the flags may disagree only
    when the smallest head pivot lies within 2x of the singular threshold
    rtol * ||Ahat - sigma I||_F (reference solvers.py:226-228).  Returns the
    worst (relative error, bound) pair."""
    rtol = 1e3 * n * EPS if rtol is None else rtol
    worst = (0.0, 1.0)
    for l in range(len(fail_ref)):
        gpu_bad, ref_bad = fail[l] >= 0, fail_ref[l] >= 0
        if gpu_bad != ref_bad:
            ratio = diag[l, 1] / rtol
            assert 0.5 <= ratio <= 2.0, (
                f"shift {l}: failure flags differ (gpu {fail[l]}, oracle {fail_ref[l]}) "
                f"and the head pivot is {ratio:.3g} x the threshold (> 2x away)")
            continue
        if ref_bad:
            assert np.isnan(Y[:, l * cols_per_shift:(l + 1) * cols_per_shift]).all()
            continue
        a = Y[:, l * cols_per_shift:(l + 1) * cols_per_shift]
        b = Y_ref[:, l * cols_per_shift:(l + 1) * cols_per_shift]
        err = np.linalg.norm(a - b) / np.linalg.norm(b)
        bound = shift_tolerance(n, diag[l, 0])
        assert err <= bound, f"shift {l}: rel err {err:.3e} > {bound:.3e} (kappa {diag[l, 0]:.3g})"
        if err / bound > worst[0] / worst[1]:
            worst = (err, bound)
    return worst
