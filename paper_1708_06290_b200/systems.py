"""Synthetic test systems (reference systems.py:71-86) and the benchmark
configurations of BASELINE.json."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class SystemBundle:
    """State-space triple (A, B, C) (reference systems.py:12-36)."""

    A: np.ndarray
    B: np.ndarray
    C: np.ndarray
    name: str = ""

    @property
    def n(self) -> int:
        return self.A.shape[0]

    @property
    def m(self) -> int:
        return self.B.shape[1]

    @property
    def p(self) -> int:
        return self.C.shape[0]


def random_stable_system(n: int, m: int, p: int, seed: int = 0, margin: float = 0.05,
                         circular: bool = False) -> SystemBundle:
    """Seeded Gaussian triple with A shifted to a negative spectral abscissa.

    Default: the reference generator (systems.py:71-86) -- same rng call
    order and the eigenvalue-based shift, so the triple is identical to
    ``shiftsolve.random_stable_system(n, m, p, seed)``.

    ``circular=True`` replaces the O(n^3) eigenvalue computation by the
    circular-law bound: a standard Gaussian n x n matrix has spectral radius
    ~sqrt(n), so A - 1.1 sqrt(n) I is stable with abscissa ~ -0.1 sqrt(n).
    SURVEY.md 8(d) uses it for n >= 10000 (eigvals takes ~20 min at
    n = 20000); it is a documented deviation and carries a distinct name.
    """
    rng = np.random.default_rng(seed)
    A = np.asfortranarray(rng.standard_normal((n, n)))
    if circular:
        A -= 1.1 * np.sqrt(n) * np.eye(n)
    else:
        abscissa = float(np.max(np.real(np.linalg.eigvals(A))))
        A -= (abscissa + margin * np.sqrt(n)) * np.eye(n)
    B = np.asfortranarray(rng.standard_normal((n, m)))
    C = np.asfortranarray(rng.standard_normal((p, n)))
    tag = "circular" if circular else "random"
    return SystemBundle(A=A, B=B, C=C, name=f"{tag}-n{n}-m{m}-p{p}-s{seed}")


def config_shifts(cfg: int, n: int, seed: int | None = None) -> np.ndarray:
    """Shift sets of the five BASELINE.json configurations."""
    rt = np.sqrt(n)
    if cfg == 1:
        return 1j * np.logspace(-2, 2, 100) * rt
    if cfg == 2:
        return 1j * np.logspace(-2, 2, 1000) * rt
    if cfg == 3:
        re = np.linspace(-0.6 * rt, 0.4 * rt, 100)
        im = np.linspace(-1.2 * rt, 1.2 * rt, 100)
        return (re[None, :] + 1j * im[:, None]).ravel()
    if cfg in (4, 5):
        rng = np.random.default_rng(cfg if seed is None else seed)
        count = 1000 if cfg == 4 else 2000
        a = rng.uniform(0.05, 1.0, count) * rt
        b = rng.uniform(0.0, 1.5, count) * rt
        return np.stack([a + 1j * b, a - 1j * b], axis=1).ravel()
    raise ValueError("config must be 1..5")


#: (n, m, p, shifts) of BASELINE.json configs[0..4]
CONFIGS = {1: (500, 5, 5, 100), 2: (4000, 10, 10, 1000), 3: (2000, 1, 1, 10000),
           4: (10000, 20, 20, 2000), 5: (20000, 50, 50, 4000)}
