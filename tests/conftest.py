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
