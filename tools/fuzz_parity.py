"""Randomised parity sweep of the GPU sweep against the C oracle (experiment
tooling): random (n, m, p, nb, batch), transfer function and reduced solve,
<= 1e-10 per shift; prints failures."""
import os, sys, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1708_06290_b200 as ss
from oracle import oracle as O

def triple(n, m, p, rng):
    A = np.triu(rng.standard_normal((n, n)), -m) - 1.1 * np.sqrt(n) * np.eye(n)
    B = np.zeros((n, m)); B[:m, :m] = np.triu(rng.standard_normal((m, m))) + 2 * np.eye(m)
    C = rng.standard_normal((p, n))
    return ss.ControllerHessForm(Ahat=np.asfortranarray(A), Bhat=B, Chat=C, m=m, n=n, p=p)

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
ms = [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 16, 20, 24, 29, 31, 32, 40, 50, 59, 60, 63, 70]
worst, bad = 0.0, 0
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    m = int(rng.choice(ms))
    n = int(rng.integers(m + 2, int(os.environ.get("FUZZ_NMAX", "900"))))
    p = int(rng.integers(1, 12))
    nb = int(rng.choice([4, 7, 16, 32, 64]))
    bs = [None, 3, 17][int(rng.integers(0, 3))]
    chf = triple(n, m, p, rng)
    s = int(rng.integers(1, 40))
    sh = (rng.uniform(-0.5, 0.5, s) + 1j * rng.uniform(-1.5, 1.5, s)) * np.sqrt(n)
    try:
        G = ss.eval_transfer_function(chf, sh, nb=nb, batch_size=bs).G
    except Exception as e:
        print(f"EXC n={n} m={m} p={p} nb={nb} bs={bs}: {e}"); bad += 1; continue
    idx = sorted(set([0, s // 2, s - 1]))
    Go, _ = O.tf_eval(chf.Ahat, chf.Bhat, chf.Chat, sh[idx], nb=nb)
    err = max(np.linalg.norm(G[:, l * m:(l + 1) * m] - Go[:, k * m:(k + 1) * m]) /
              np.linalg.norm(Go[:, k * m:(k + 1) * m]) for k, l in enumerate(idx))
    # reduced solve (identity top) and the transposed solve
    k2 = [0, s - 1]
    bd = rng.standard_normal((m, len(k2))) + 1j * rng.standard_normal((m, len(k2)))
    try:
        X = ss.solve_shifted_reduced(chf, sh[k2], bd, nb=nb, batch_size=bs).x
        for k, l in enumerate(k2):
            xo = O.lu_solve_shifted(chf.Ahat, sh[l], chf.Bhat @ bd[:, k])
            err = max(err, np.linalg.norm(X[:, k] - xo) / np.linalg.norm(xo))
        if m + 1 <= 256:
            rhs = rng.standard_normal((n, len(k2))) + 1j * rng.standard_normal((n, len(k2)))
            Xt = ss.solve_shifted_transposed(chf, sh[k2], rhs, nb=min(nb, 32), batch_size=bs).x
            for k, l in enumerate(k2):
                xo = O.lu_solve_shifted(chf.Ahat, sh[l], rhs[:, k], transpose=True)
                err = max(err, np.linalg.norm(Xt[:, k] - xo) / np.linalg.norm(xo))
    except Exception as e:
        print(f"EXC(solve) n={n} m={m} p={p} nb={nb} bs={bs}: {e}"); bad += 1; continue
    worst = max(worst, err)
    flag = "FAIL" if err > 1e-10 else "ok"
    if err > 1e-10:
        bad += 1
    print(f"{flag} n={n} m={m} p={p} nb={nb} bs={bs} s={s}: {err:.2e}", flush=True)
print(f"worst {worst:.2e}, failures {bad}")
