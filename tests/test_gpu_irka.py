"""IRKA on the GPU solvers (reference irka.py:179-262) against the
reference's own trajectories (tests/golden/irka.npz, generated from the
reference) and the independent LU oracle; mirrors test_irka.py:75-131."""

import numpy as np
import pytest

from conftest import golden

import paper_1708_06290_b200 as ss
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def case(i):
    g = golden("irka.npz")
    pre = f"i{i}_"
    n, m, p, seed, r, iters = (int(v) for v in g[pre + "dims"])
    chf = ss.ControllerHessForm(Ahat=g[pre + "Ahat"], Bhat=g[pre + "Bhat"], Chat=g[pre + "Chat"],
                                m=m, n=n, p=p)
    return g, pre, chf, r, iters


@pytest.mark.parametrize("i", range(5))
def test_trajectory_matches_reference(i):
    """Shift history per iteration within 1e-8 relative Hausdorff (the
    reference's own bound vs its LU oracle, test_irka.py:104-110), final
    reduced model within 1e-6."""
    g, pre, chf, r, iters = case(i)
    s0, b0, c0 = ss.default_initial_data(chf, r)
    model, state = ss.irka_iterate(chf, r, s0, b0, c0, maxiter=iters, fixed_iters=True, nb=8)
    assert state.iterations == iters
    for k, rec in enumerate(state.history):
        assert ss.relative_hausdorff(rec.shifts, g[pre + "hist"][k]) <= 1e-8
    assert ss.relative_hausdorff(state.shifts, g[pre + "final"]) <= 1e-8
    # the reduced model is basis-dependent; its transfer function is not
    for sv in (0.3j, 1.0 + 2j):
        Gr = model.transfer(sv)
        Gref = g[pre + "Cr"] @ np.linalg.solve(sv * np.eye(r) - g[pre + "Ar"], g[pre + "Br"])
        assert np.linalg.norm(Gr - Gref) <= 1e-6 * np.linalg.norm(Gref)


def test_single_iteration_shapes():
    _, _, chf, _, _ = case(2)
    model, state = ss.irka_iterate(chf, 3, maxiter=1, fixed_iters=True, nb=4)
    assert state.iterations == 1 and len(state.history) == 1
    assert model.Ar.shape == (3, 3) and model.Br.shape == (3, 2) and model.Cr.shape == (2, 3)
    assert np.all(np.isfinite(model.Ar))


def test_conjugate_closed_and_orthonormal():
    _, _, chf, _, _ = case(2)
    _, state = ss.irka_iterate(chf, 4, maxiter=6, fixed_iters=True, nb=8)
    for rec in state.history:
        assert np.allclose(np.sort_complex(rec.shifts), np.sort_complex(np.conj(rec.shifts)),
                           atol=0)
    for M in (state.V, state.W):
        assert np.linalg.norm(M.conj().T @ M - np.eye(4)) <= 1e-12


def test_mimo_tangential_interpolation():
    """test_irka.py:112-119: the reduced model interpolates G tangentially at
    the last iteration's points (LU oracle on the original triple)."""
    g, pre, chf, r, iters = case(1)
    model, state = ss.irka_iterate(chf, r, maxiter=10, fixed_iters=True, nb=8)
    rec = state.history[-1]
    A, B, C = g[pre + "A"], g[pre + "B"], g[pre + "C"]
    for i in range(r):
        gf = O.oracle_transfer_function(A, B, C, rec.shifts[i]) @ rec.b_dirs[:, i]
        gr = model.transfer(rec.shifts[i]) @ rec.b_dirs[:, i]
        assert np.linalg.norm(gr - gf) <= 1e-6 * np.linalg.norm(gf)


def test_early_stop_and_rejections():
    _, _, chf, _, _ = case(0)
    _, state = ss.irka_iterate(chf, 2, maxiter=60, tol=1e-8, nb=8)
    assert state.iterations < 60 and state.history[-1].shift_change < 1e-8
    with pytest.raises(ss.DimensionMismatchError):
        ss.irka_iterate(chf, chf.n)


def test_spectrum_collision_perturbed():
    """test_irka.py:127-131: a shift on an eigenvalue is nudged."""
    _, _, chf, _, _ = case(0)
    ev = np.linalg.eigvals(chf.Ahat)
    s0 = np.array([complex(ev[0]), 1.0 + 0j])
    b0 = np.ones((1, 2), dtype=complex)
    c0 = np.ones((1, 2), dtype=complex)
    _, state = ss.irka_iterate(chf, 2, s0, b0, c0, maxiter=2, fixed_iters=True, nb=4)
    assert state.perturbations and state.perturbations[0][0] == 0
