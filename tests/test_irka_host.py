"""Host-side IRKA helpers (reference test_irka.py:23-73): the r x r pencil
eigensolver contract, conjugate pairing, the Hausdorff distance."""

import numpy as np
import pytest

import paper_1708_06290_b200 as ss


def test_pencil_diagonal_identity():
    lam, Y, X = ss.small_eig_pencil(np.diag([3.0, -1.0, 2.0]), np.eye(3))
    assert np.allclose(np.sort(lam.real), [-1.0, 2.0, 3.0], atol=1e-13)


def test_pencil_2x2_quadratic_formula():
    a, b, c, d = 2.0, 1.0, 3.0, -1.0
    tr, det = a + d, a * d - b * c
    disc = np.sqrt(tr * tr - 4 * det + 0j)
    expect = np.sort_complex(np.array([(tr + disc) / 2, (tr - disc) / 2]))
    lam, _, _ = ss.small_eig_pencil(np.array([[a, b], [c, d]]), np.eye(2))
    assert np.allclose(np.sort_complex(lam), expect, atol=1e-12)


def test_pencil_residual_contract(rng):
    E = rng.standard_normal((8, 8))
    F = rng.standard_normal((8, 8)) + 8 * np.eye(8)
    lam, Y, X = ss.small_eig_pencil(E, F)
    for i in range(8):
        bound = 1e-10 * (np.linalg.norm(E) + abs(lam[i]) * np.linalg.norm(F))
        assert np.linalg.norm(E @ X[:, i] - lam[i] * (F @ X[:, i])) <= bound
        assert np.linalg.norm(Y[i, :] @ E - lam[i] * (Y[i, :] @ F)) <= bound


def test_pencil_rejections():
    with pytest.raises(ss.EigensolverError):
        ss.small_eig_pencil(np.eye(2), np.zeros((2, 2)))
    with pytest.raises(ValueError):
        ss.small_eig_pencil(np.eye(513), np.eye(513))


def test_pair_conjugates_enforces_closure(rng):
    shifts = np.array([1.0 + 2.0j, 1.0 - 2.0000001j, 3.0 + 1e-12j])
    bd = rng.standard_normal((2, 3)) + 1j * rng.standard_normal((2, 3))
    cd = rng.standard_normal((2, 3)) + 1j * rng.standard_normal((2, 3))
    s, b, c = ss.pair_conjugates(shifts, bd, cd)
    assert np.array_equal(np.sort_complex(s), np.sort_complex(np.conj(s)))
    assert s[2].imag == 0.0
    assert np.array_equal(b[:, 1], np.conj(b[:, 0]))


def test_relative_hausdorff():
    a = np.array([1.0 + 1j, 2.0])
    assert ss.relative_hausdorff(a, a) == 0.0
    b = np.array([1.0 + 1j, 2.2])
    assert ss.relative_hausdorff(a, b) == pytest.approx(0.2 / 2.2)
