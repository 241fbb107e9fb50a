"""Generate golden vectors by running the Python reference itself.

Run in the build container (the reference is only present there):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``shiftsolve`` read-only from /root/reference/pkg/src and writes
small .npz fixtures next to this script.  The fixtures travel with the repo;
nothing at test time reads /root/reference.

Cases (each cites the reference test it mirrors):
  schedules.npz      greedy_schedule(nr, nc) for a set of shapes
                     (test_schedule.py:12-16, SURVEY Appendix A shapes)
  batched_rq.npz     batched_rq inputs/outputs (test_batched.py:38-98)
  scalar.npz         the scalar resolvent known answer (test_solvers.py:32-40)
  systems.npz        small random systems: inputs A,B,C, the reference's
                     reduced triple, shifts, reference G / reduced x, LU oracle
                     values (test_solvers.py:42-50, test_acceptance.py:130-163)
  failure.npz        failure-isolation case with an eigenvalue shift
                     (test_solvers.py:73-85)
  config1.npz        config 1 (n=500, m=p=5, 100 i*omega shifts) reference G
                     and input checksums (BASELINE.json configs[0])
  irka.npz           irka_iterate trajectories (shift history per iteration,
                     final reduced model) on reduced triples
                     (test_irka.py:81-131)
  cli/               a reference CLI session: `gen` -> `reduce` (archive with
                     manifest) -> `tf` and `pspec` CSVs (test_sysio_cli.py)
  transposed.npz     solve_shifted_transposed on reduced triples (general
                     right-hand sides), the scalar known answer, a failure
                     case, and mirrored_schedule plans (test_solvers.py:139-189,
                     test_schedule.py:106-120)
  transposed_wide.npz  the same for m + 1 > 32 (m = 33..100) and one IRKA run at m = 40
"""

from __future__ import annotations

import hashlib
import os
import sys

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from shiftsolve import (  # noqa: E402
    BlockBatch,
    batched_rq,
    eval_transfer_function,
    greedy_schedule,
    random_stable_system,
    reduce_controller_hessenberg,
    solve_shifted_reduced,
    solve_shifted_transposed,
)
from shiftsolve.schedule import mirrored_schedule  # noqa: E402
from shiftsolve.hessenberg import ControllerHessForm  # noqa: E402
from shiftsolve.oracles import lu_solve_shifted, oracle_transfer_function  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.asfortranarray(a).tobytes(order="F")).hexdigest()


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


def schedules():
    shapes = [(1, 1), (1, 3), (4, 7), (8, 14), (13, 16), (16, 17), (32, 42),
              (64, 65), (64, 69), (64, 74), (64, 84), (64, 114), (100, 110)]
    d = {}
    for nr, nc in shapes:
        s = greedy_schedule(nr, nc)
        d[f"job_{nr}_{nc}"] = np.asarray(s.job_size, dtype=np.int64)
        d[f"info_{nr}_{nc}"] = np.asarray(s.rot_info, dtype=np.int64)
    d["shapes"] = np.asarray(shapes, dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "schedules.npz"), **d)


def batched():
    rng = np.random.default_rng(4321)
    d = {}
    cases = [(6, 9, 3), (8, 14, 2), (16, 26, 2), (5, 5, 1), (1, 4, 2)]
    for idx, (nr, nc, s) in enumerate(cases):
        batch = BlockBatch.zeros(nr, nc, s)
        for l in range(s):
            Z = rng.standard_normal((nr, nc)) + 1j * rng.standard_normal((nr, nc))
            for r in range(nr):
                Z[r, :r] = 0.0
            batch.z_block(l)[:, :] = Z
        Zin = batch.Z.copy()
        batched_rq(batch, greedy_schedule(nr, nc))
        d[f"shape_{idx}"] = np.asarray([nr, nc, s])
        d[f"zin_{idx}"] = Zin
        d[f"r_{idx}"] = batch.Z.copy()
        d[f"p_{idx}"] = batch.P.copy()
    d["count"] = np.asarray(len(cases))
    np.savez_compressed(os.path.join(OUT, "batched_rq.npz"), **d)


def scalar():
    chf = ControllerHessForm(Ahat=np.array([[1.5]], order="F"), Bhat=np.array([[2.0]], order="F"),
                             Chat=np.array([[3.0]], order="F"), m=1, n=1, p=1)
    sigma = 2.0 + 0.5j
    res = eval_transfer_function(chf, [sigma], nb=4)
    np.savez_compressed(os.path.join(OUT, "scalar.npz"), G=res.G, sigma=np.asarray([sigma]),
                        expect=np.asarray([3.0 * 2.0 / (sigma - 1.5)]))


def systems():
    rng = np.random.default_rng(7)
    d = {}
    specs = [(50, 2, 3, 11, 8, "iw")]
    for case in range(14):
        n = int(rng.integers(4, 65))
        m = int(rng.integers(1, min(4, n - 1) + 1))
        p = int(rng.integers(1, 5))
        nb = int(rng.choice([4, 8, 16]))
        specs.append((n, m, p, 20_000 + case, nb, "bounded"))
    specs.append((96, 6, 4, 31, 16, "bounded"))
    specs.append((128, 8, 3, 32, 32, "bounded"))
    for idx, (n, m, p, seed, nb, kind) in enumerate(specs):
        sysb = random_stable_system(n, m, p, seed=seed)
        chf = reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=8)
        if kind == "iw":
            shifts = 1j * np.logspace(-1, 1, 7)
        else:
            shifts = bounded_shifts(rng, chf.Ahat, 16)
        res = eval_transfer_function(chf, shifts, nb=nb)
        bd = rng.standard_normal((m, len(shifts))) + 1j * rng.standard_normal((m, len(shifts)))
        red = solve_shifted_reduced(chf, shifts, bd, nb=nb)
        Glu = np.concatenate([oracle_transfer_function(sysb.A, sysb.B, sysb.C, s_)
                              for s_ in shifts], axis=1)
        xlu = np.stack([lu_solve_shifted(chf.Ahat, s_, chf.Bhat @ bd[:, l])
                        for l, s_ in enumerate(shifts)], axis=1)
        chf64 = reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=64)
        pre = f"s{idx}_"
        d[pre + "dims"] = np.asarray([n, m, p, seed, nb])
        d[pre + "A"], d[pre + "B"], d[pre + "C"] = sysb.A, sysb.B, sysb.C
        d[pre + "Ahat"], d[pre + "Bhat"], d[pre + "Chat"] = chf.Ahat, chf.Bhat, chf.Chat
        d[pre + "Ahat64"], d[pre + "Bhat64"], d[pre + "Chat64"] = chf64.Ahat, chf64.Bhat, chf64.Chat
        d[pre + "shifts"] = shifts
        d[pre + "G"] = res.G
        d[pre + "Glu"] = Glu
        d[pre + "bdirs"] = bd
        d[pre + "x"] = red.x
        d[pre + "xlu"] = xlu
    d["count"] = np.asarray(len(specs))
    np.savez_compressed(os.path.join(OUT, "systems.npz"), **d)


def failure():
    sysb = random_stable_system(24, 2, 2, seed=9)
    chf = reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=8)
    rng = np.random.default_rng(23)
    good = bounded_shifts(rng, chf.Ahat, 15)
    ev = np.linalg.eigvals(chf.Ahat)
    bad = ev[int(np.argmax(np.abs(ev.imag)))]
    full = np.concatenate([good[:7], [bad], good[7:]])
    marked = eval_transfer_function(chf, full, nb=8, on_singular="mark")
    bd = rng.standard_normal((2, 16)) + 1j * rng.standard_normal((2, 16))
    redm = solve_shifted_reduced(chf, full, bd, nb=8, on_singular="mark")
    fails = np.asarray(sorted(marked.failures.items()), dtype=np.int64).reshape(-1, 2)
    rfails = np.asarray(sorted(redm.failures.items()), dtype=np.int64).reshape(-1, 2)
    np.savez_compressed(os.path.join(OUT, "failure.npz"), Ahat=chf.Ahat, Bhat=chf.Bhat,
                        Chat=chf.Chat, shifts=full, G=marked.G, failures=fails,
                        bdirs=bd, x=redm.x, rfailures=rfails)


def config1():
    n, m, p = 500, 5, 5
    sysb = random_stable_system(n, m, p, seed=1)
    chf = reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=64)
    omega = np.logspace(-2, 2, 100) * np.sqrt(n)
    shifts = 1j * omega
    res = eval_transfer_function(chf, shifts, nb=32)
    Glu = np.concatenate([oracle_transfer_function(sysb.A, sysb.B, sysb.C, shifts[l])
                          for l in (0, 37, 99)], axis=1)
    np.savez_compressed(os.path.join(OUT, "config1.npz"), shifts=shifts, G=res.G,
                        lu_idx=np.asarray([0, 37, 99]), Glu=Glu,
                        sha_A=np.asarray(sha(sysb.A)), sha_B=np.asarray(sha(sysb.B)),
                        sha_C=np.asarray(sha(sysb.C)), seed=np.asarray(1),
                        dims=np.asarray([n, m, p]))


def transposed():
    rng = np.random.default_rng(17)
    d = {}
    specs = [(40, 3, 2, 12, 8), (30, 2, 2, 13, 8), (33, 3, 2, 14, 8), (64, 4, 3, 40, 16),
             (96, 6, 4, 41, 16), (128, 8, 3, 42, 32), (75, 1, 1, 43, 8), (57, 5, 2, 44, 4),
             (200, 10, 10, 45, 32)]
    for idx, (n, m, p, seed, nb) in enumerate(specs):
        sysb = random_stable_system(n, m, p, seed=seed)
        chf = reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=8)
        shifts = bounded_shifts(rng, chf.Ahat, 6)
        rhs = rng.standard_normal((n, 6)) + 1j * rng.standard_normal((n, 6))
        res = solve_shifted_transposed(chf, shifts, rhs, nb=nb)
        xlu = np.stack([lu_solve_shifted(chf.Ahat, s_, rhs[:, l], transpose=True)
                        for l, s_ in enumerate(shifts)], axis=1)
        pre = f"t{idx}_"
        d[pre + "dims"] = np.asarray([n, m, p, seed, nb])
        d[pre + "Ahat"], d[pre + "Bhat"], d[pre + "Chat"] = chf.Ahat, chf.Bhat, chf.Chat
        d[pre + "shifts"], d[pre + "rhs"], d[pre + "x"], d[pre + "xlu"] = shifts, rhs, res.x, xlu
    d["count"] = np.asarray(len(specs))
    # scalar known answer (test_solvers.py:139-142)
    chf1 = ControllerHessForm(Ahat=np.array([[2.0]], order="F"), Bhat=np.array([[1.0]], order="F"),
                              Chat=np.array([[1.0]], order="F"), m=1, n=1, p=1)
    r1 = solve_shifted_transposed(chf1, [0.5], np.array([[3.0 + 0j]]), nb=4)
    d["scalar_x"] = r1.x
    # failure isolation (test_solvers.py:173-184)
    sysb = random_stable_system(24, 2, 2, seed=15)
    chf = reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=8)
    good = bounded_shifts(rng, chf.Ahat, 5)
    ev = np.linalg.eigvals(chf.Ahat)
    bad = ev[int(np.argmax(np.abs(ev.imag)))]
    full = np.concatenate([good, [bad]])
    rhs = rng.standard_normal((24, 6)) + 1j * rng.standard_normal((24, 6))
    rf = solve_shifted_transposed(chf, full, rhs, nb=4, on_singular="mark")
    d["f_Ahat"], d["f_Bhat"], d["f_Chat"] = chf.Ahat, chf.Bhat, chf.Chat
    d["f_shifts"], d["f_rhs"], d["f_x"] = full, rhs, rf.x
    d["f_failures"] = np.asarray(sorted(rf.failures.items()), dtype=np.int64).reshape(-1, 2)
    # mirrored schedules
    for nr, nc in [(3, 5), (8, 14), (16, 26), (32, 42), (64, 74)]:
        sch = mirrored_schedule(nr, nc)
        d[f"ms_{nr}_{nc}_job"] = np.asarray(sch.job_size, dtype=np.int64)
        d[f"ms_{nr}_{nc}_info"] = np.asarray(sch.rot_info, dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "transposed.npz"), **d)


def transposed_wide():
    """Windows wider than one warp (m + 1 > 32): the shared-memory LQ path,
    and IRKA on such a system (solve_shifted_transposed every iteration)."""
    from shiftsolve.irka import default_initial_data, irka_iterate
    rng = np.random.default_rng(23)
    d = {}
    specs = [(90, 33, 2, 60, 8), (120, 40, 3, 61, 16), (160, 50, 5, 62, 32), (200, 63, 4, 63, 32),
             (260, 100, 3, 64, 16)]
    for idx, (n, m, p, seed, nb) in enumerate(specs):
        sysb = random_stable_system(n, m, p, seed=seed)
        chf = reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=8)
        shifts = bounded_shifts(rng, chf.Ahat, 4)
        rhs = rng.standard_normal((n, 4)) + 1j * rng.standard_normal((n, 4))
        res = solve_shifted_transposed(chf, shifts, rhs, nb=nb)
        xlu = np.stack([lu_solve_shifted(chf.Ahat, s_, rhs[:, l], transpose=True)
                        for l, s_ in enumerate(shifts)], axis=1)
        pre = f"t{idx}_"
        d[pre + "dims"] = np.asarray([n, m, p, seed, nb])
        d[pre + "Ahat"], d[pre + "Bhat"], d[pre + "Chat"] = chf.Ahat, chf.Bhat, chf.Chat
        d[pre + "shifts"], d[pre + "rhs"], d[pre + "x"], d[pre + "xlu"] = shifts, rhs, res.x, xlu
    d["count"] = np.asarray(len(specs))
    n, m, p, seed, r, iters = 120, 40, 3, 66, 6, 4
    sysb = random_stable_system(n, m, p, seed=seed)
    chf = reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=8)
    s0, b0, c0 = default_initial_data(chf, r)
    model, state = irka_iterate(chf, r, s0, b0, c0, maxiter=iters, fixed_iters=True, nb=8)
    d["irka_dims"] = np.asarray([n, m, p, seed, r, iters])
    d["irka_Ahat"], d["irka_Bhat"], d["irka_Chat"] = chf.Ahat, chf.Bhat, chf.Chat
    d["irka_hist"] = np.stack([rec.shifts for rec in state.history])
    d["irka_Ar"], d["irka_Br"], d["irka_Cr"] = model.Ar, model.Br, model.Cr
    np.savez_compressed(os.path.join(OUT, "transposed_wide.npz"), **d)


def cli():
    import shutil

    from shiftsolve.cli import main as ref_main
    root = os.path.join(OUT, "cli")
    shutil.rmtree(root, ignore_errors=True)
    os.makedirs(root)
    sysdir, arch = os.path.join(root, "sys"), os.path.join(root, "archive")
    assert ref_main(["gen", "--n", "40", "--m", "3", "--p", "2", "--seed", "5", "--out", sysdir]) == 0
    assert ref_main(["reduce", *(os.path.join(sysdir, f) for f in ("A.mtx", "B.mtx", "C.mtx")),
                     "--out", arch, "--block-size", "8"]) == 0
    assert ref_main(["tf", arch, "--out", os.path.join(root, "tf.csv"), "--w-min", "0.1",
                     "--w-max", "100", "--count", "9", "--nb", "8"]) == 0
    assert ref_main(["pspec", arch, "--out", os.path.join(root, "pspec.csv"), "--re-min", "-3",
                     "--re-max", "1", "--re-count", "4", "--im-min", "-2", "--im-max", "2",
                     "--im-count", "3", "--nb", "8"]) == 0
    shutil.rmtree(sysdir)  # the archive is the fixture; gen is re-run by the test


def irka():
    from shiftsolve.irka import default_initial_data, irka_iterate
    d = {}
    specs = [(30, 1, 1, 4, 4, 8), (30, 2, 2, 5, 4, 10), (24, 2, 2, 2, 4, 6), (60, 3, 2, 50, 6, 6),
             (120, 4, 3, 51, 8, 5)]
    for idx, (n, m, p, seed, r, iters) in enumerate(specs):
        sysb = random_stable_system(n, m, p, seed=seed)
        chf = reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=8)
        s0, b0, c0 = default_initial_data(chf, r)
        model, state = irka_iterate(chf, r, s0, b0, c0, maxiter=iters, fixed_iters=True, nb=8)
        pre = f"i{idx}_"
        d[pre + "dims"] = np.asarray([n, m, p, seed, r, iters])
        d[pre + "A"], d[pre + "B"], d[pre + "C"] = sysb.A, sysb.B, sysb.C
        d[pre + "Ahat"], d[pre + "Bhat"], d[pre + "Chat"] = chf.Ahat, chf.Bhat, chf.Chat
        d[pre + "hist"] = np.stack([rec.shifts for rec in state.history])
        d[pre + "final"] = state.shifts
        d[pre + "Ar"], d[pre + "Br"], d[pre + "Cr"] = model.Ar, model.Br, model.Cr
    d["count"] = np.asarray(len(specs))
    np.savez_compressed(os.path.join(OUT, "irka.npz"), **d)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[name]()
        sys.exit(0)
    schedules()
    batched()
    scalar()
    systems()
    failure()
    config1()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
