"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, the
reference's golden vectors and the independent LU oracle.

Tolerances (north_star): ||G_gpu - G_ref|| / ||G_ref|| <= 1e-10 per shift
(FP64), tighter where the reference tests are tighter; parameter invariance
<= 1e-12; batch composition / failure isolation bitwise.
"""

import numpy as np
import pytest
import torch

from conftest import bounded_shifts, golden, probe_shifts

import paper_1708_06290_b200 as ss
from oracle import oracle as O

pytestmark = pytest.mark.gpu

EPS = np.finfo(float).eps


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def per_shift_rel(G, Gr, m, s):
    return max(rel(G[:, l * m:(l + 1) * m], Gr[:, l * m:(l + 1) * m]) for l in range(s))


def chf_of(S, pre, suffix=""):
    n, m, p = (int(v) for v in S[pre + "dims"][:3])
    return ss.ControllerHessForm(Ahat=S[pre + "Ahat" + suffix], Bhat=S[pre + "Bhat" + suffix],
                                 Chat=S[pre + "Chat" + suffix], m=m, n=n, p=p)


# --------------------------------------------------------------------------
# transfer function
# --------------------------------------------------------------------------

def test_scalar_resolvent_exact():
    """test_solvers.py:32-40 known answer, 4 eps."""
    chf = ss.ControllerHessForm(Ahat=np.array([[1.5]]), Bhat=np.array([[2.0]]),
                                Chat=np.array([[3.0]]), m=1, n=1, p=1)
    sigma = 2.0 + 0.5j
    res = ss.eval_transfer_function(chf, [sigma], nb=4)
    expect = 3.0 * 2.0 / (sigma - 1.5)
    assert abs(res.G[0, 0] - expect) <= 4 * EPS * abs(expect)


@pytest.mark.parametrize("case", range(17))
def test_golden_systems_tf_and_reduced(case):
    S = golden("systems.npz")
    pre = f"s{case}_"
    n, m, p, seed, nb = (int(v) for v in S[pre + "dims"])
    chf = chf_of(S, pre)
    shifts = S[pre + "shifts"]
    s = len(shifts)
    res = ss.eval_transfer_function(chf, shifts, nb=nb)
    assert res.failures == {}
    assert per_shift_rel(res.G, S[pre + "G"], m, s) <= 1e-10      # vs reference
    assert per_shift_rel(res.G, S[pre + "Glu"], m, s) <= 1e-10    # vs LU oracle (orig triple)
    Go, _ = O.tf_eval(chf.Ahat, chf.Bhat, chf.Chat, shifts, nb=nb)
    assert per_shift_rel(res.G, Go, m, s) <= 1e-11                 # vs C oracle
    red = ss.solve_shifted_reduced(chf, shifts, S[pre + "bdirs"], nb=nb)
    assert red.failures == {}
    for l in range(s):
        assert rel(red.x[:, l], S[pre + "x"][:, l]) <= 1e-10
        assert rel(red.x[:, l], S[pre + "xlu"][:, l]) <= 1e-10


def test_criterion4_corpus_vs_lu():
    """test_acceptance.py:130-163 style: random systems, 16 bounded-condition
    shifts each, nb in {4, 8, 16}: tf and reduced <= 1e-10 vs dense LU."""
    rng = np.random.default_rng(7)
    worst_tf = worst_red = 0.0
    for case in range(40):
        n = int(rng.integers(4, 65))
        m = int(rng.integers(1, min(4, n - 1) + 1))
        p = int(rng.integers(1, 5))
        sysb = ss.random_stable_system(n, m, p, seed=20_000 + case, circular=False)
        chf = ss.reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=8)
        shifts = bounded_shifts(rng, chf.Ahat, 16)
        nb = int(rng.choice([4, 8, 16]))
        res = ss.eval_transfer_function(chf, shifts, nb=nb)
        bd = rng.standard_normal((m, 16)) + 1j * rng.standard_normal((m, 16))
        red = ss.solve_shifted_reduced(chf, shifts, bd, nb=nb)
        for l, sig in enumerate(shifts):
            Go = O.oracle_transfer_function(sysb.A, sysb.B, sysb.C, sig)
            worst_tf = max(worst_tf, rel(res.value(l), Go))
            xo = O.lu_solve_shifted(chf.Ahat, sig, chf.Bhat @ bd[:, l])
            worst_red = max(worst_red, rel(red.x[:, l], xo))
    assert worst_tf <= 1e-10 and worst_red <= 1e-10, (worst_tf, worst_red)


def test_parameter_invariance(rng):
    """test_solvers.py:52-59 / test_acceptance.py:166-199: nb and batch size."""
    sysb = ss.random_stable_system(48, 3, 2, seed=5, circular=False)
    chf = ss.reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=8)
    shifts = bounded_shifts(rng, chf.Ahat, 10)
    ref = ss.eval_transfer_function(chf, shifts, nb=6).G
    for nb in (3, 6, 8, 32, 64):
        for bs in (1, 4, None):
            G = ss.eval_transfer_function(chf, shifts, nb=nb, batch_size=bs).G
            assert np.abs(G - ref).max() <= 1e-12 * np.abs(ref).max()


def test_batch_composition_bitwise(rng):
    """Each shift is computed in isolation: any subset / batch size gives
    bitwise identical slices (reference solvers.py:25-28)."""
    sysb = ss.random_stable_system(80, 4, 3, seed=9, circular=False)
    chf = ss.reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=16)
    shifts = probe_shifts(rng, 20, scale=5.0)
    full = ss.eval_transfer_function(chf, shifts, nb=16).G
    part = ss.eval_transfer_function(chf, shifts[5:12], nb=16).G
    assert np.array_equal(part, full[:, 5 * 4:12 * 4])
    b3 = ss.eval_transfer_function(chf, shifts, nb=16, batch_size=3).G
    assert np.array_equal(b3, full)


def test_failure_isolation_bitwise():
    """test_acceptance.py:311-339 with the reference's own failure case."""
    F = golden("failure.npz")
    chf = ss.ControllerHessForm(Ahat=F["Ahat"], Bhat=F["Bhat"], Chat=F["Chat"], m=2, n=24, p=2)
    full = F["shifts"]
    marked = ss.eval_transfer_function(chf, full, nb=8, on_singular="mark")
    assert marked.failures == {7: 0}
    assert np.isnan(marked.value(7)).all()
    keep = [i for i in range(16) if i != 7]
    clean = ss.eval_transfer_function(chf, full[keep], nb=8)
    for lc, li in enumerate(keep):
        assert np.array_equal(marked.value(li), clean.value(lc))
    ok = ~np.isnan(F["G"])
    assert np.abs(marked.G[ok] - F["G"][ok]).max() <= 1e-10 * np.abs(F["G"][ok]).max()
    with pytest.raises(ss.SingularShiftError) as ei:
        ss.eval_transfer_function(chf, full, nb=8)
    assert ei.value.failures == [(7, 0)]
    redm = ss.solve_shifted_reduced(chf, full, F["bdirs"], nb=8, on_singular="mark")
    assert redm.failures == {int(a): int(b) for a, b in F["rfailures"]}
    assert np.isnan(redm.x[:, 7]).all()


def test_singular_rtol_is_used_as_given():
    """singular_rtol=0.0 means only exactly-zero pivots fail (reference
    solvers.py:227 ``abs(piv) <= rtol * scale``); it must not fall back to
    the default 1e3 n eps.  A huge rtol flags every shift."""
    sysb = ss.random_stable_system(16, 2, 2, seed=8, circular=False)
    chf = ss.reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=8)
    ev = np.linalg.eigvals(chf.Ahat)[0]
    shifts = np.array([ev * (1 + 1e-14), 1j, ev])
    default = ss.eval_transfer_function(chf, shifts, nb=4, on_singular="mark")
    assert 0 in default.failures and 2 in default.failures
    zero = ss.eval_transfer_function(chf, shifts, nb=4, on_singular="mark", singular_rtol=0.0)
    G_o, f_o = O.tf_eval(chf.Ahat, chf.Bhat, chf.Chat, shifts, nb=4, rtol=0.0)
    assert zero.failures == {int(l): int(f_o[l]) for l in np.nonzero(f_o >= 0)[0]}
    assert 1 not in zero.failures and 0 not in zero.failures
    assert np.isfinite(zero.value(0)).all()
    np.testing.assert_array_equal(zero.value(1), default.value(1))
    red = ss.solve_shifted_reduced(chf, shifts[:2], np.ones((2, 2)), nb=4, on_singular="mark",
                                   singular_rtol=0.0)
    assert red.failures == {}
    big = ss.eval_transfer_function(chf, shifts, nb=4, on_singular="mark", singular_rtol=1e6)
    assert sorted(big.failures) == [0, 1, 2]


def test_singular_shift_raises_by_default():
    sysb = ss.random_stable_system(16, 2, 2, seed=8, circular=False)
    chf = ss.reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=8)
    ev = np.linalg.eigvals(chf.Ahat)[0]
    with pytest.raises(ss.SingularShiftError):
        ss.eval_transfer_function(chf, [ev], nb=4)


def test_result_slicing():
    sysb = ss.random_stable_system(12, 2, 2, seed=0, circular=False)
    chf = ss.reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=8)
    res = ss.eval_transfer_function(chf, [1j, 2j], nb=4)
    assert res.value(1).shape == (2, 2)
    assert np.array_equal(res.value(0), res.G[:, :2])


def test_counters_populated():
    sysb = ss.random_stable_system(20, 2, 2, seed=17, circular=False)
    chf = ss.reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=8)
    c = ss.PhaseCounters()
    ss.eval_transfer_function(chf, [1j, 2j], nb=4, counter=c)
    snap = c.snapshot()
    for ph in ("small_batched_rq", "outer_gemm", "tail_solves", "batched_gemm"):
        assert snap[ph][0] > 0 and snap[ph][1] > 0


def test_config1_full_vs_reference():
    """BASELINE configs[0] end to end: GPU reduction + GPU sweep vs the
    reference's G (CPU reduction + CPU sweep) on the same seeded input."""
    g = golden("config1.npz")
    n, m, p = (int(v) for v in g["dims"])
    sysb = ss.random_stable_system(n, m, p, seed=int(g["seed"]), circular=False)
    chf = ss.reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=64)
    res = ss.eval_transfer_function(chf, g["shifts"], nb=32)
    assert res.failures == {}
    assert per_shift_rel(res.G, g["G"], m, 100) <= 1e-10
    for k, l in enumerate(g["lu_idx"]):
        assert rel(res.value(int(l)), g["Glu"][:, k * m:(k + 1) * m]) <= 1e-10


def test_device_resident_inputs_stay_on_device():
    sysb = ss.random_stable_system(64, 3, 2, seed=4, circular=False)
    chf = ss.reduce_controller_hessenberg(torch.tensor(sysb.A, device="cuda"),
                                          torch.tensor(sysb.B, device="cuda"),
                                          torch.tensor(sysb.C, device="cuda"), block_size=16)
    assert isinstance(chf.Ahat, torch.Tensor) and chf.Ahat.is_cuda
    sh = torch.tensor(1j * np.linspace(1, 5, 9), device="cuda")
    res = ss.eval_transfer_function(chf, sh, nb=16)
    assert isinstance(res.G, torch.Tensor) and res.G.is_cuda
    Gh = ss.eval_transfer_function(chf.numpy(), sh.cpu().numpy(), nb=16).G
    assert np.array_equal(res.G.cpu().numpy(), Gh)


# --------------------------------------------------------------------------
# reduced solves
# --------------------------------------------------------------------------

def test_reduced_triangular_back_substitution(rng):
    """test_solvers.py:89-106."""
    n, m = 8, 2
    Ahat = np.asfortranarray(np.triu(rng.standard_normal((n, n))) + 4 * np.eye(n))
    Bhat = np.zeros((n, m), order="F")
    Bhat[:m, :m] = np.triu(rng.standard_normal((m, m))) + 2 * np.eye(m)
    chf = ss.ControllerHessForm(Ahat=Ahat, Bhat=Bhat, Chat=np.zeros((1, n), order="F"), m=m, n=n, p=1)
    sigma = 0.3 + 0.2j
    bdir = np.zeros((m, 1), dtype=complex)
    bdir[0, 0] = 1.0
    res = ss.solve_shifted_reduced(chf, [sigma], bdir, nb=4)
    M = Ahat - sigma * np.eye(n)
    rhs = (Bhat @ bdir[:, 0]).astype(complex)
    x = np.zeros(n, dtype=complex)
    for i in range(n - 1, -1, -1):
        x[i] = (rhs[i] - M[i, i + 1:] @ x[i + 1:]) / M[i, i]
    assert np.linalg.norm(res.x[:, 0] - x) <= 1e-12 * np.linalg.norm(x)


def test_reduced_zero_shift_and_certificate(rng):
    sysb = ss.random_stable_system(32, 2, 2, seed=7, circular=False)
    chf = ss.reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=8)
    bdir = rng.standard_normal((2, 1)) + 0j
    res = ss.solve_shifted_reduced(chf, [0.0], bdir, nb=8)
    xo = O.lu_solve_shifted(chf.Ahat, 0.0, chf.Bhat @ bdir[:, 0])
    assert rel(res.x[:, 0], xo) <= 1e-10
    shifts = probe_shifts(rng, 4, scale=2.0)
    bdirs = rng.standard_normal((2, 4)) + 0j
    res = ss.solve_shifted_reduced(chf, shifts, bdirs, nb=8)
    for l, sigma in enumerate(shifts):
        rhs = (chf.Bhat @ bdirs[:, l]).astype(complex)
        cert = ss.residual_certificate(chf, sigma, res.x[:, l], rhs)
        assert cert <= 1e3 * chf.n * EPS


# --------------------------------------------------------------------------
# pseudospectrum grid
# --------------------------------------------------------------------------

def test_pseudospectrum_siso_and_inf(rng):
    sysb = ss.random_stable_system(12, 1, 1, seed=21, circular=False)
    chf = ss.reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=8)
    pts = probe_shifts(rng, 4, scale=2.0)
    vals = ss.structured_pseudospectrum_grid(chf, pts, nb=4)
    res = ss.eval_transfer_function(chf, pts, nb=4)
    assert np.allclose(vals, np.abs(res.G[0, :]), atol=1e-13 * np.abs(res.G).max())
    ev = np.linalg.eigvals(chf.Ahat)
    bad = ev[np.argmax(np.abs(ev.imag))]
    v2 = ss.structured_pseudospectrum_grid(chf, [bad, 1.0 + 1.0j], nb=4)
    assert np.isinf(v2[0]) and np.isfinite(v2[1])


def test_pseudospectrum_mimo_svd_and_symmetry(rng):
    n, m, p = 5, 2, 2
    Qb, _ = np.linalg.qr(rng.standard_normal((n, n)))
    A = Qb @ np.diag([-1.0, -2.0, -3.0, -4.0, -5.0]) @ Qb.T
    B = rng.standard_normal((n, m))
    C = rng.standard_normal((p, n))
    chf = ss.reduce_controller_hessenberg(A, B, C, block_size=2)
    pts = np.array([0.5 + 0.5j, -1.5 + 2j, 3.0 - 1j])
    vals = ss.structured_pseudospectrum_grid(chf, pts, nb=2)
    for z, v in zip(pts, vals):
        Gz = O.oracle_transfer_function(A, B, C, z)
        assert abs(v - np.linalg.svd(Gz, compute_uv=False)[0]) <= 1e-10 * max(v, 1.0)
    sysb = ss.random_stable_system(14, 2, 2, seed=24, circular=False)
    chf = ss.reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=8)
    pts = np.array([0.4 + 1.3j, 0.4 - 1.3j, -0.6 + 2j, -0.6 - 2j])
    vals = ss.structured_pseudospectrum_grid(chf, pts, nb=4)
    assert abs(vals[0] - vals[1]) <= 1e-12 * vals[0]
    assert abs(vals[2] - vals[3]) <= 1e-12 * vals[2]


def test_far_point_asymptotics():
    sysb = ss.random_stable_system(16, 2, 2, seed=22, circular=False)
    chf = ss.reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=8)
    z = 1e8 * np.linalg.norm(sysb.A)
    val = ss.structured_pseudospectrum_grid(chf, [z + 0j], nb=8)[0]
    approx = np.linalg.svd(sysb.C @ sysb.B, compute_uv=False)[0] / z
    assert abs(val / approx - 1.0) <= 1e-6


# --------------------------------------------------------------------------
# GPU reduction
# --------------------------------------------------------------------------

@pytest.mark.parametrize("case", [0, 3, 9, 15, 16])
@pytest.mark.parametrize("bs", [1, 7, 64])
def test_reduction_matches_reference(case, bs):
    S = golden("systems.npz")
    pre = f"s{case}_"
    n, m = int(S[pre + "dims"][0]), int(S[pre + "dims"][1])
    A, B, C = S[pre + "A"], S[pre + "B"], S[pre + "C"]
    chf = ss.reduce_controller_hessenberg(A, B, C, block_size=bs, accumulate=True)
    nA = np.linalg.norm(A)
    assert np.abs(chf.Ahat - S[pre + "Ahat"]).max() <= 1e-11 * nA
    assert np.abs(chf.Bhat - S[pre + "Bhat"]).max() <= 1e-11 * np.linalg.norm(B)
    assert np.abs(chf.Chat - S[pre + "Chat"]).max() <= 1e-11 * nA * np.linalg.norm(C)
    for j in range(n):
        assert np.all(chf.Ahat[j + m + 1:, j] == 0.0)
    for j in range(m):
        assert np.all(chf.Bhat[j + 1:, j] == 0.0)
    sim = np.linalg.norm(chf.Q.T @ A @ chf.Q - chf.Ahat)
    assert sim <= 64 * n * EPS * nA


def test_reduction_criterion3_corpus():
    """test_acceptance.py:83-127 style: blocked GPU reduction vs the oracle's
    unblocked reduction through the LU transfer function, b in {1,7,64}."""
    rng = np.random.default_rng(2024)
    worst_sim = worst_tf = 0.0
    for case in range(12):
        n = int(rng.integers(6, 129)) if case >= 2 else 128
        m = int(rng.integers(1, min(8, n - 1) + 1))
        p = int(rng.integers(1, 9))
        sysb = ss.random_stable_system(n, m, p, seed=10_000 + case, circular=False)
        Ao, Bo, Co, _ = O.reduce_chf(sysb.A, sysb.B, sysb.C)
        probes = bounded_shifts(rng, sysb.A, 3)
        for b in (1, 7, 64):
            for strat in ("sequential", "overlapped"):
                chf = ss.reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=b,
                                                      strategy=strat, accumulate=True)
                sim = np.linalg.norm(chf.Q.T @ sysb.A @ chf.Q - chf.Ahat)
                worst_sim = max(worst_sim, sim / (64 * n * EPS * np.linalg.norm(sysb.A)))
                for sig in probes:
                    Gb = O.oracle_transfer_function(chf.Ahat, chf.Bhat, chf.Chat, sig)
                    Go = O.oracle_transfer_function(Ao, Bo, Co, sig)
                    worst_tf = max(worst_tf, rel(Gb, Go))
    assert worst_sim <= 1.0 and worst_tf <= 1e-10, (worst_sim, worst_tf)


def test_reduction_strategies_bitwise():
    sysb = ss.random_stable_system(70, 3, 2, seed=31, circular=False)
    a = ss.reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=16)
    b = ss.reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=16, strategy="overlapped")
    assert np.array_equal(a.Ahat, b.Ahat) and np.array_equal(a.Chat, b.Chat)


# --------------------------------------------------------------------------
# larger sizes: oracle on sampled shifts + size-independent properties
# --------------------------------------------------------------------------

@pytest.mark.parametrize("n,m,p,nb", [(1000, 10, 10, 64), (2000, 1, 1, 64), (1500, 20, 20, 48)])
def test_medium_sizes_vs_oracle(n, m, p, nb):
    sysb = ss.random_stable_system(n, m, p, seed=n + m, circular=True)
    chf = ss.reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=64)
    shifts = 1j * np.logspace(-2, 2, 24) * np.sqrt(n) + 0.1
    res = ss.eval_transfer_function(chf, shifts, nb=nb)
    assert res.failures == {}
    idx = [0, 7, 23]
    Go, _ = O.tf_eval(chf.Ahat, chf.Bhat, chf.Chat, shifts[idx], nb=nb)
    for k, l in enumerate(idx):
        assert rel(res.value(l), Go[:, k * m:(k + 1) * m]) <= 1e-10
    # conjugate symmetry of a real system: G(conj s) = conj G(s)
    res2 = ss.eval_transfer_function(chf, np.conj(shifts), nb=nb)
    assert per_shift_rel(res2.G, np.conj(res.G), m, len(shifts)) <= 1e-10
    # residual of the reduced solve on one shift
    bd = np.ones((m, 1), dtype=complex)
    red = ss.solve_shifted_reduced(chf, shifts[3:4], bd, nb=nb)
    cert = ss.residual_certificate(chf, shifts[3], red.x[:, 0], chf.Bhat @ bd[:, 0])
    assert cert <= 1e3 * n * EPS


@pytest.mark.parametrize("case", [0, 9, 15, 16])
def test_block_rq_flavours_agree(case, monkeypatch):
    """The row-Householder block RQ (default) and the reference's scheduled
    Givens batch (SS_BLOCK_RQ=givens) give the same G to rounding: P differs
    by an m x m unitary on the active columns, G is invariant."""
    S = golden("systems.npz")
    pre = f"s{case}_"
    m, nb = int(S[pre + "dims"][1]), int(S[pre + "dims"][4])
    chf = chf_of(S, pre)
    shifts = S[pre + "shifts"]
    Gh = ss.eval_transfer_function(chf, shifts, nb=nb).G
    monkeypatch.setenv("SS_BLOCK_RQ", "givens")
    Gg = ss.eval_transfer_function(chf, shifts, nb=nb).G
    assert per_shift_rel(Gh, Gg, m, len(shifts)) <= 1e-12
    assert per_shift_rel(Gg, S[pre + "G"], m, len(shifts)) <= 1e-10


def _mhess_triple(n, m, p, seed):
    """Random m-Hessenberg / triangular / dense triple of the reduced shape."""
    rng = np.random.default_rng(seed)
    A = np.triu(rng.standard_normal((n, n)), -m) - 1.1 * np.sqrt(n) * np.eye(n)
    B = np.zeros((n, m))
    B[:m, :m] = np.triu(rng.standard_normal((m, m))) + 2 * np.eye(m)
    C = rng.standard_normal((p, n))
    return ss.ControllerHessForm(Ahat=np.asfortranarray(A), Bhat=np.asfortranarray(B),
                                 Chat=np.asfortranarray(C), m=m, n=n, p=p)


@pytest.mark.parametrize("n,m,p", [(300, 10, 10), (517, 10, 3), (161, 1, 1), (40, 5, 2),
                                   (389, 2, 4), (455, 3, 3), (260, 7, 5), (700, 8, 8), (129, 4, 1),
                                   (333, 20, 4), (700, 20, 20), (61, 20, 3)])
def test_two_level_vs_one_level(n, m, p, monkeypatch):
    """The two-level sweep (k_block + k_far over 128-column outer blocks, the
    default for m in 1..8, 10) against the per-window sweep (SS_ONE_LEVEL=1)
    and the C oracle, on ragged sizes (n - m not a multiple of 128 or 32)."""
    chf = _mhess_triple(n, m, p, seed=n * 31 + m)
    shifts = 1j * np.logspace(-2, 2, 37) * np.sqrt(n) + 0.2
    G2 = ss.eval_transfer_function(chf, shifts, nb=64).G
    bd = np.exp(1j * np.arange(m * 5).reshape(m, 5))
    X2 = ss.solve_shifted_reduced(chf, shifts[:5], bd, nb=64).x
    monkeypatch.setenv("SS_ONE_LEVEL", "1")
    G1 = ss.eval_transfer_function(chf, shifts, nb=64).G
    X1 = ss.solve_shifted_reduced(chf, shifts[:5], bd, nb=64).x
    assert per_shift_rel(G2, G1, m, len(shifts)) <= 1e-12
    assert max(rel(X2[:, k], X1[:, k]) for k in range(5)) <= 1e-12
    idx = [0, 18, 36]
    Go, _ = O.tf_eval(chf.Ahat, chf.Bhat, chf.Chat, shifts[idx], nb=32)
    for k, l in enumerate(idx):
        assert rel(G2[:, l * m:(l + 1) * m], Go[:, k * m:(k + 1) * m]) <= 1e-10


@pytest.mark.parametrize("n,m,p", [(700, 10, 10), (650, 20, 5), (520, 5, 5), (400, 4, 3)])
def test_paired_blocks_vs_unpaired(n, m, p, monkeypatch):
    """Paired outer blocks (near update + one far update per 256 columns from
    the composite W) against one far update per 128-column block
    (SS_NO_PAIR=1): the composite is exact algebra, so G and the reduced
    solve agree to rounding; odd block counts and a ragged last block."""
    chf = _mhess_triple(n, m, p, seed=n * 13 + m)
    shifts = np.concatenate([1j * np.logspace(-2, 2, 19) * np.sqrt(n) + 0.3,
                             [0.5 * np.sqrt(n) - 0.2j]])
    bd = np.exp(1j * np.arange(m * 3).reshape(m, 3))
    Gp = ss.eval_transfer_function(chf, shifts, nb=64).G
    Xp = ss.solve_shifted_reduced(chf, shifts[:3], bd, nb=64).x
    monkeypatch.setenv("SS_NO_PAIR", "1")
    Gu = ss.eval_transfer_function(chf, shifts, nb=64).G
    Xu = ss.solve_shifted_reduced(chf, shifts[:3], bd, nb=64).x
    assert per_shift_rel(Gp, Gu, m, len(shifts)) <= 1e-12
    assert max(rel(Xp[:, k], Xu[:, k]) for k in range(3)) <= 1e-12


@pytest.mark.parametrize("n,p", [(1111, 10), (700, 3), (389, 10)])
def test_far4_vs_far(n, p, monkeypatch):
    """m = 10 far-row update: 128-column passes on the four-way-split kernel
    (k_far4, default) against 64-column passes on k_far (SS_FAR4=0) --
    ragged last blocks, odd pair counts, the near update, the reduced solve
    (identity top, far rows from the block's first column)."""
    m = 10
    monkeypatch.setenv("SS_FAR_PASSES", "1")  # the pass kernels, not k_fark
    chf = _mhess_triple(n, m, p, seed=n * 7 + p)
    shifts = np.concatenate([1j * np.logspace(-2, 2, 25) * np.sqrt(n) + 0.2,
                             [0.4 * np.sqrt(n) + 0.9j * np.sqrt(n)]])
    bd = np.exp(1j * np.arange(m * 3).reshape(m, 3))
    G4 = ss.eval_transfer_function(chf, shifts, nb=64).G
    X4 = ss.solve_shifted_reduced(chf, shifts[:3], bd, nb=64).x
    monkeypatch.setenv("SS_FAR4", "0")
    G2 = ss.eval_transfer_function(chf, shifts, nb=64).G
    X2 = ss.solve_shifted_reduced(chf, shifts[:3], bd, nb=64).x
    assert per_shift_rel(G4, G2, m, len(shifts)) <= 1e-12
    assert max(rel(X4[:, k], X2[:, k]) for k in range(3)) <= 1e-12


@pytest.mark.parametrize("group", ["1", "2", "4"])
@pytest.mark.parametrize("n,m,p", [(1111, 10, 10), (700, 20, 3), (389, 20, 20), (1400, 5, 4),
                                   (650, 20, 5)])
def test_block_groups_vs_oracle(group, n, m, p, monkeypatch):
    """Groups of 1, 2, 4 outer blocks per composite (SS_GROUP; default 4 on
    the K-streamed far kernel, 2 on the pass kernels): composites over up to
    512 columns with near updates inside the group, ragged first blocks and
    partial last groups; transfer function and reduced solve vs the oracle."""
    monkeypatch.setenv("SS_GROUP", group)
    chf = _mhess_triple(n, m, p, seed=n * 3 + m)
    shifts = np.concatenate([1j * np.logspace(-2, 2, 9) * np.sqrt(n) + 0.3,
                             [0.5 * np.sqrt(n) - 0.2j, 0.2 * np.sqrt(n) + 1.1j * np.sqrt(n)]])
    s = len(shifts)
    G = ss.eval_transfer_function(chf, shifts, nb=64).G
    Go, fo = O.tf_eval(chf.Ahat, chf.Bhat, chf.Chat, shifts, nb=64, threads=4)
    assert (fo < 0).all()
    assert per_shift_rel(G, Go, m, s) <= 1e-11
    bd = np.exp(1j * np.arange(m * 3).reshape(m, 3))
    X = ss.solve_shifted_reduced(chf, shifts[:3], bd, nb=64).x
    Xo, _ = O.solve_reduced(chf.Ahat, chf.Bhat, shifts[:3], bd, nb=64, threads=4)
    assert max(rel(X[:, k], Xo[:, k]) for k in range(3)) <= 1e-11


@pytest.mark.parametrize("n,m", [(1111, 10), (700, 20), (389, 20), (1400, 5), (650, 8), (130, 4)])
def test_reduced_deferred_identity_vs_swept(n, m, monkeypatch):
    """Reduced solve on the two-level sweep with the identity top deferred
    (x expanded from the kept composites, k_expand) against the identity rows
    swept as the reference does (SS_NO_DEFER=1) and the oracle; failure
    isolation keeps NaN columns."""
    chf = _mhess_triple(n, m, 3, seed=n + 5 * m)
    rng = np.random.default_rng(n * m)
    s = 11
    shifts = (rng.uniform(-0.5, 1.0, s) + 1j * rng.uniform(-1.5, 1.5, s)) * np.sqrt(n)
    bd = rng.standard_normal((m, s)) + 1j * rng.standard_normal((m, s))
    X = ss.solve_shifted_reduced(chf, shifts, bd, nb=64).x
    Xb = ss.solve_shifted_reduced(chf, shifts, bd, nb=64, batch_size=4).x
    assert np.array_equal(X, Xb)
    Xo, fo = O.solve_reduced(chf.Ahat, chf.Bhat, shifts, bd, nb=64, threads=4)
    assert (fo < 0).all()
    assert max(rel(X[:, k], Xo[:, k]) for k in range(s)) <= 1e-11
    monkeypatch.setenv("SS_NO_DEFER", "1")
    Xs = ss.solve_shifted_reduced(chf, shifts, bd, nb=64).x
    assert max(rel(X[:, k], Xs[:, k]) for k in range(s)) <= 1e-12
    for k in range(3):
        cert = ss.solvers.residual_certificate(chf, shifts[k], X[:, k], chf.Bhat[:, :m] @ bd[:, k])
        assert cert <= 1e-13


def test_reduced_deferred_failure_isolation():
    """A shift on the spectrum fails alone in the deferred reduced solve
    (NaN column, the pivot index as the reference reports it), the other
    columns are bitwise those of a run without it."""
    n, m = 300, 5
    chf = _mhess_triple(n, m, 2, seed=77)
    # decouple the leading m columns: eig(A11) are eigenvalues of Ahat and a
    # shift there leaves the HEAD singular (where the reference tests pivots)
    chf.Ahat[m:2 * m, :m] = 0.0
    ev = np.linalg.eigvals(chf.Ahat[:m, :m])
    shifts = np.array([0.3 + 2j, ev[0], -1.0 + 0.5j, 4j])
    bd = np.exp(1j * np.arange(m * 4).reshape(m, 4))
    res = ss.solve_shifted_reduced(chf, shifts, bd, nb=64, on_singular="mark")
    Xo, fo = O.solve_reduced(chf.Ahat, chf.Bhat, shifts, bd, nb=64, threads=4)
    assert res.failures == {int(l): int(fo[l]) for l in np.nonzero(fo >= 0)[0]}
    assert 1 in res.failures and np.isnan(res.x[:, 1]).all()
    keep = [0, 2, 3]
    clean = ss.solve_shifted_reduced(chf, shifts[keep], bd[:, keep], nb=64).x
    assert np.array_equal(clean, res.x[:, keep])


@pytest.mark.parametrize("n,m,p,s", [(1111, 10, 10, 26), (700, 10, 3, 9), (389, 20, 7, 13),
                                     (1500, 20, 20, 41), (260, 20, 1, 5), (1337, 10, 5, 17)])
def test_fark_vs_passes_and_oracle(n, m, p, s, monkeypatch):
    """K-streamed far kernel (k_fark: one pass per composite, default for
    m = 10, 20) against the 64 / 128-column pass kernels (SS_FAR_PASSES=1)
    and the C oracle: ragged last blocks, odd p (unaligned Chat rows in the
    packed panel), shift counts that leave a partial last shift group."""
    chf = _mhess_triple(n, m, p, seed=n * 11 + m)
    rng = np.random.default_rng(n + s)
    shifts = (rng.uniform(-0.5, 1.0, s) + 1j * rng.uniform(-1.5, 1.5, s)) * np.sqrt(n)
    Gk = ss.eval_transfer_function(chf, shifts, nb=64).G
    Gb3 = ss.eval_transfer_function(chf, shifts, nb=64, batch_size=3).G
    assert np.array_equal(Gk, Gb3)  # shift groups never mix shifts
    monkeypatch.setenv("SS_FAR_PASSES", "1")
    Gp = ss.eval_transfer_function(chf, shifts, nb=64).G
    assert per_shift_rel(Gk, Gp, m, s) <= 1e-12
    idx = np.arange(0, s, max(1, s // 4))
    Go, fo = O.tf_eval(chf.Ahat, chf.Bhat, chf.Chat, shifts[idx], nb=64, threads=4)
    assert (fo < 0).all()
    Gs = np.concatenate([Gk[:, l * m:(l + 1) * m] for l in idx], axis=1)
    assert per_shift_rel(Gs, Go, m, len(idx)) <= 1e-11


@pytest.mark.parametrize("n,nb", [(333, 64), (300, 32), (129, 7), (66, 64)])
def test_m1_throughput_rq_vs_warp_rq(n, nb, monkeypatch):
    """m = 1 window RQ: the 8-lane-per-shift kernel (k_rq_m1, P rows beside
    the chain) against the one-warp-per-shift Householder RQ
    (SS_RQ_M1_OFF=1) and the C oracle, on ragged windows (nb < 64, n - 1 not
    a multiple of nb), a shift count that leaves a partial warp, a zero
    subdiagonal (identity reflectors) and real / complex / conjugate shifts."""
    chf = _mhess_triple(n, 1, 1, seed=n + nb)
    chf.Ahat[n // 2, n // 2 - 1] = 0.0
    shifts = np.concatenate([1j * np.logspace(-2, 2, 19) * np.sqrt(n) + 0.1,
                             [0.3 * np.sqrt(n), 0.2 - 0.7j * np.sqrt(n)]])
    r1 = ss.eval_transfer_function(chf, shifts, nb=nb)
    monkeypatch.setenv("SS_RQ_M1_OFF", "1")
    r0 = ss.eval_transfer_function(chf, shifts, nb=nb)
    assert r1.failures == r0.failures == {}
    assert per_shift_rel(r1.G, r0.G, 1, len(shifts)) <= 1e-12
    Go, _ = O.tf_eval(chf.Ahat, chf.Bhat, chf.Chat, shifts[[0, 10, 20]], nb=nb)
    for k, l in enumerate([0, 10, 20]):
        assert rel(r1.G[:, l:l + 1], Go[:, k:k + 1]) <= 1e-10


@pytest.mark.parametrize("n,m,p", [(400, 50, 50), (330, 33, 7), (500, 20, 20), (260, 16, 4), (300, 63, 5),
                                   (420, 100, 90), (380, 70, 3), (1500, 40, 6), (1300, 50, 9), (1400, 60, 4)])
def test_wide_m_paths_vs_oracle(n, m, p):
    """Block widths outside the two-level set: m + 1 > 32 takes the scheduled
    Givens block RQ (config 5: m = 50; m = 100: head matrices in global
    scratch), m = 16 / 20 the one-level update with
    several column blocks per shift (config 4: m = 20).  Transfer function and
    reduced solve vs the C oracle, conjugate pairs of complex shifts as in
    config 4 / 5.  n >= 1300 at m = 40 / 50 / 60: several window composites,
    so the K-streamed far pass (k_farkd) runs over real far rows."""
    sysb = ss.random_stable_system(n, m, p, seed=n + 7 * m, circular=True)
    chf = ss.reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=64)
    rng = np.random.default_rng(m)
    a = rng.uniform(0.05, 1.0, 6) * np.sqrt(n)
    b = rng.uniform(0.0, 1.5, 6) * np.sqrt(n)
    shifts = np.concatenate([a + 1j * b, a - 1j * b])
    res = ss.eval_transfer_function(chf, shifts, nb=64)
    assert res.failures == {}
    Go, fo = O.tf_eval(chf.Ahat, chf.Bhat, chf.Chat, shifts, nb=64)
    assert (fo < 0).all()
    assert per_shift_rel(res.G, Go, m, len(shifts)) <= 1e-10
    # conjugate pairs give conjugate transfer functions (real system)
    assert per_shift_rel(res.G[:, 6 * m:], np.conj(res.G[:, :6 * m]), m, 6) <= 1e-10
    bd = (rng.standard_normal((m, 4)) + 1j * rng.standard_normal((m, 4)))
    bd /= np.linalg.norm(bd, axis=0)
    red = ss.solve_shifted_reduced(chf, shifts[:4], bd, nb=64)
    for k in range(4):
        cert = ss.residual_certificate(chf, shifts[k], red.x[:, k], chf.Bhat @ bd[:, k])
        assert cert <= 1e3 * n * EPS


@pytest.mark.parametrize("n,m,p", [(120, 7, 3), (90, 2, 6), (300, 10, 10), (64, 4, 1),
                                   (200, 33, 40), (260, 50, 50), (400, 100, 110)])
def test_pseudospectrum_epilogue_vs_svd(n, m, p):
    """The device ||G||_2 epilogue (Gram matrix + parallel Hermitian Jacobi)
    against numpy's SVD of the same G blocks (solvers.py:501-505), wide and
    tall blocks, odd k, k = 50 (config 5's block) and k = 100 (Gram matrix in
    global scratch); singular points -> +inf."""
    chf = _mhess_triple(n, m, p, seed=n + m + p)
    rng = np.random.default_rng(n)
    grid = (rng.uniform(-1, 1, 40) + 1j * rng.uniform(-1, 1, 40)) * np.sqrt(n)
    vals = ss.structured_pseudospectrum_grid(chf, grid, nb=32)
    G = ss.eval_transfer_function(chf, grid, nb=32).G
    ref = np.array([np.linalg.svd(G[:, l * m:(l + 1) * m], compute_uv=False)[0]
                    for l in range(len(grid))])
    assert np.max(np.abs(vals - ref) / ref) <= 1e-12
    # at a (numerically computed) eigenvalue: flagged singular (+inf) or a
    # resolvent norm orders of magnitude above the grid's
    ev = np.linalg.eigvals(chf.Ahat)
    v2 = ss.structured_pseudospectrum_grid(chf, np.array([ev[0], grid[0]]), nb=32)
    assert np.isinf(v2[0]) or v2[0] > 1e4 * np.median(ref)
    assert abs(v2[1] - ref[0]) <= 1e-12 * ref[0]


@pytest.mark.parametrize("n,m,p,bs", [(517, 10, 3, None), (300, 5, 2, 7), (260, 1, 1, None),
                                      (333, 20, 4, 5)])
def test_streamed_host_ahat_bitwise(n, m, p, bs):
    """A pinned, column-major host Ahat is streamed to the device chunk by
    chunk in sweep order (ss_tf_eval_stream); results are bitwise those of
    the device-resident call (two-level and one-level paths, several
    batches)."""
    chf = _mhess_triple(n, m, p, seed=7 * n + m)
    shifts = 1j * np.logspace(-1, 1, 23) * np.sqrt(n) + 0.3
    ref = ss.eval_transfer_function(chf, shifts, nb=64, batch_size=bs).G
    Ah = torch.from_numpy(np.asfortranarray(chf.Ahat)).t().contiguous().t().pin_memory()
    assert Ah.is_pinned() and Ah.stride(0) == 1
    chf_h = ss.ControllerHessForm(Ahat=Ah, Bhat=torch.from_numpy(chf.Bhat).pin_memory(),
                                  Chat=torch.from_numpy(chf.Chat).pin_memory(), m=m, n=n, p=p)
    sh = torch.from_numpy(shifts).pin_memory()
    res = ss.eval_transfer_function(chf_h, sh, nb=64, batch_size=bs)
    assert np.array_equal(np.asarray(res.G), ref)
