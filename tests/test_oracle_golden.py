"""Pin the CPU oracle (oracle/shiftsolve_oracle.c) to the Python reference.

tests/golden/*.npz were produced by tests/golden/make_golden.py, which ran
the reference package itself.  Schedules must match bitwise (integer
plans); floating-point outputs within a few ulps-scaled tolerances (the
reference's BLAS and numpy use different summation orders than the C loops).
"""

import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O


def test_schedules_bitwise():
    g = golden("schedules.npz")
    for nr, nc in g["shapes"]:
        job, info = O.greedy_schedule(int(nr), int(nc))
        assert np.array_equal(job, g[f"job_{nr}_{nc}"]), (nr, nc)
        assert np.array_equal(info, g[f"info_{nr}_{nc}"]), (nr, nc)


def test_schedule_known_count():
    """test_schedule.py:12-16: (8,14) -> 13 steps / 48 rotations."""
    job, info = O.greedy_schedule(8, 14)
    assert len(job) == 13 and len(info) // 3 == 48


def test_batched_rq_matches_reference():
    b = golden("batched_rq.npz")
    for k in range(int(b["count"])):
        nr, nc, s = (int(v) for v in b[f"shape_{k}"])
        R, P = O.batched_rq(b[f"zin_{k}"], nr, nc)
        scale = max(np.abs(b[f"zin_{k}"]).max(), 1.0)
        assert np.abs(R - b[f"r_{k}"]).max() <= 1e-13 * scale * nc
        assert np.abs(P - b[f"p_{k}"]).max() <= 1e-13 * nc


def test_scalar_known_answer():
    g = golden("scalar.npz")
    G, fail = O.tf_eval(np.array([[1.5]]), np.array([[2.0]]), np.array([[3.0]]), g["sigma"], nb=4)
    assert fail[0] == -1
    assert abs(G[0, 0] - g["expect"][0]) <= 4 * np.finfo(float).eps * abs(g["expect"][0])


def _systems():
    S = golden("systems.npz")
    return [(S, k) for k in range(int(S["count"]))]


@pytest.mark.parametrize("case", range(17))
def test_tf_and_reduced_match_reference(case):
    S = golden("systems.npz")
    pre = f"s{case}_"
    n, m, p, seed, nb = (int(v) for v in S[pre + "dims"])
    G, fail = O.tf_eval(S[pre + "Ahat"], S[pre + "Bhat"], S[pre + "Chat"], S[pre + "shifts"], nb=nb)
    assert (fail < 0).all()
    Gr = S[pre + "G"]
    for l in range(len(S[pre + "shifts"])):
        a, b = G[:, l * m:(l + 1) * m], Gr[:, l * m:(l + 1) * m]
        assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b)
        lu = S[pre + "Glu"][:, l * m:(l + 1) * m]
        assert np.linalg.norm(a - lu) <= 1e-10 * np.linalg.norm(lu)
    x, fx = O.solve_reduced(S[pre + "Ahat"], S[pre + "Bhat"], S[pre + "shifts"], S[pre + "bdirs"],
                            nb=nb)
    assert (fx < 0).all()
    xr, xlu = S[pre + "x"], S[pre + "xlu"]
    for l in range(x.shape[1]):
        assert np.linalg.norm(x[:, l] - xr[:, l]) <= 1e-12 * np.linalg.norm(xr[:, l])
        assert np.linalg.norm(x[:, l] - xlu[:, l]) <= 1e-10 * np.linalg.norm(xlu[:, l])


@pytest.mark.parametrize("case", [0, 3, 9, 15, 16])
def test_reduction_matches_reference(case):
    S = golden("systems.npz")
    pre = f"s{case}_"
    n = int(S[pre + "dims"][0])
    m = int(S[pre + "dims"][1])
    Ah, Bh, Ch, Q = O.reduce_chf(S[pre + "A"], S[pre + "B"], S[pre + "C"], accumulate=True)
    nA = np.linalg.norm(S[pre + "A"])
    for ref in ("", "64"):
        assert np.abs(Ah - S[pre + "Ahat" + ref]).max() <= 1e-12 * nA
        assert np.abs(Bh - S[pre + "Bhat" + ref]).max() <= 1e-12 * np.linalg.norm(S[pre + "B"])
        assert np.abs(Ch - S[pre + "Chat" + ref]).max() <= 1e-12 * nA * np.linalg.norm(S[pre + "C"])
    for j in range(n):
        assert np.all(Ah[j + m + 1:, j] == 0.0)
    for j in range(m):
        assert np.all(Bh[j + 1:, j] == 0.0)
    sim = np.linalg.norm(Q.T @ S[pre + "A"] @ Q - Ah)
    assert sim <= 64 * n * np.finfo(float).eps * nA


def test_failure_isolation_matches_reference():
    F = golden("failure.npz")
    G, fail = O.tf_eval(F["Ahat"], F["Bhat"], F["Chat"], F["shifts"], nb=8)
    ref = {int(a): int(b) for a, b in F["failures"]}
    got = {int(l): int(f) for l, f in enumerate(fail) if f >= 0}
    assert got == ref == {7: 0}
    assert np.isnan(G[:, 7 * 2:8 * 2]).all()
    ok = ~np.isnan(F["G"])
    assert np.abs(G[ok] - F["G"][ok]).max() <= 1e-12 * np.abs(F["G"][ok]).max()
    x, fx = O.solve_reduced(F["Ahat"], F["Bhat"], F["shifts"], F["bdirs"], nb=8)
    rref = {int(a): int(b) for a, b in F["rfailures"]}
    assert {int(l): int(f) for l, f in enumerate(fx) if f >= 0} == rref


def test_config1_matches_reference():
    """BASELINE configs[0]: n=500, m=p=5, 100 i*omega shifts, full run."""
    import hashlib
    g = golden("config1.npz")
    n, m, p = (int(v) for v in g["dims"])
    A, B, C = O.random_stable_system(n, m, p, seed=int(g["seed"]))
    assert hashlib.sha256(np.asfortranarray(A).tobytes(order="F")).hexdigest() == str(g["sha_A"])
    Ah, Bh, Ch, _ = O.reduce_chf(A, B, C)
    G, fail = O.tf_eval(Ah, Bh, Ch, g["shifts"], nb=32)
    assert (fail < 0).all()
    Gr = g["G"]
    worst = max(np.linalg.norm(G[:, l * m:(l + 1) * m] - Gr[:, l * m:(l + 1) * m])
                / np.linalg.norm(Gr[:, l * m:(l + 1) * m]) for l in range(100))
    assert worst <= 1e-10
    for k, l in enumerate(g["lu_idx"]):
        lu = g["Glu"][:, k * m:(k + 1) * m]
        assert np.linalg.norm(G[:, l * m:(l + 1) * m] - lu) <= 1e-10 * np.linalg.norm(lu)


@pytest.mark.parametrize("n,m,p,nb", [(60, 3, 2, 8), (100, 5, 4, 16), (45, 1, 1, 7), (90, 12, 3, 32)])
def test_oracle_diagnostics_pin_the_R_diagonal(n, m, p, nb):
    """The condition estimate of the parity rule reads the R
    diagonal of every window block plus the head pivots; their log-magnitudes
    sum to log |det(Ahat - sigma I)| (the sweep is a unitary column
    transformation), for both the transfer-function and the reduced sweep."""
    rng = np.random.default_rng(n + m)
    A = np.triu(rng.standard_normal((n, n)), -m) - 1.1 * np.sqrt(n) * np.eye(n)
    B = np.zeros((n, m))
    B[:m, :m] = np.triu(rng.standard_normal((m, m))) + 2 * np.eye(m)
    C = rng.standard_normal((p, n))
    sh = np.array([3j, 2 + 5j, -1 + 0.3j])
    _, _, d = O.tf_eval(A, B, C, sh, nb=nb, diag=True)
    _, _, dr = O.solve_reduced(A, B, sh, np.ones((m, 3)), nb=nb, diag=True)
    for l, s in enumerate(sh):
        M = A - s * np.eye(n)
        ld = np.linalg.slogdet(M)[1]
        assert abs(d[l, 2] - ld) <= 1e-10 * abs(ld) + 1e-10
        assert abs(dr[l, 2] - ld) <= 1e-10 * abs(ld) + 1e-10
        # min |R_ii| >= sigma_min: the estimate never exceeds the Frobenius condition number
        kf = np.linalg.norm(M, "fro") * np.linalg.norm(np.linalg.inv(M), 2)
        assert 1.0 <= d[l, 0] <= kf * (1 + 1e-12)


def test_parity_rule_failure_flags():
    """assert_shift_parity: flags may differ only within 2x of the threshold."""
    from conftest import assert_shift_parity
    n, rt = 100, 1e3 * 100 * np.finfo(float).eps
    Y = np.ones((2, 2), complex)
    diag = np.array([[5.0, 1.5 * rt, 0.0], [5.0, 1.0, 0.0]])
    Yg = Y.copy()
    Yg[:, 0] = np.nan
    assert_shift_parity(Yg, np.array([0, -1]), Y, np.array([-1, -1]), diag, n, 1)
    diag[0, 1] = 3 * rt
    with pytest.raises(AssertionError):
        assert_shift_parity(Yg, np.array([0, -1]), Y, np.array([-1, -1]), diag, n, 1)
    Yb = Y.copy()
    Yb[0, 1] += 1e-6
    with pytest.raises(AssertionError):
        assert_shift_parity(Yb, np.array([-1, -1]), Y, np.array([-1, -1]), diag, n, 1)
