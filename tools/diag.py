#!/usr/bin/env python
"""Diagnostics for the sweep on one GPU (not part of the product or bench).

    python tools/diag.py [--cfg 2] [--nb 64] [--shifts S] [--reps 5]

Times ss_tf_eval on a synthetic m-Hessenberg triple of the config shape
under the env variants given by --variants (comma list of NAME=VAL;...),
with per-kernel event timing off (wall time of the whole call, CUDA events)
and on (phase split)."""

from __future__ import annotations

import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--nb", type=int, default=64)
    ap.add_argument("--shifts", type=int, default=0)
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--variants", default="")
    ap.add_argument("--profile", action="store_true", help="one call, no timing (for ncu)")
    args = ap.parse_args()
    import torch

    from bench import synthetic_triple
    from paper_1708_06290_b200 import _device as D
    from paper_1708_06290_b200 import _lib
    from paper_1708_06290_b200.systems import CONFIGS

    n, m, p, s = CONFIGS[args.cfg]
    s = args.shifts or s
    A, B, C = synthetic_triple(n, m, p, seed=args.cfg)
    dev = torch.device("cuda", 0)
    A, B, C = (torch.from_numpy(x).to(dev) for x in (A, B, C))
    sh = torch.from_numpy(1j * np.logspace(-2, 2, s) * np.sqrt(n)).to(dev)
    G = torch.empty((s * m, p), dtype=torch.complex128, device=dev).t()
    fail = torch.empty(s, dtype=torch.int32, device=dev)
    h = _lib.handle(0)
    L = _lib.load()
    st = torch.cuda.current_stream(dev)

    def call():
        rc = L.ss_tf_eval(h.ptr, n, m, p, D.ptr(A), D.ld(A), D.ptr(B), D.ld(B), D.ptr(C), D.ld(C),
                          D.ptr(sh), s, args.nb, 0, float("nan"), D.ptr(G), p, D.ptr(fail),
                          ctypes.c_void_p(st.cuda_stream))
        D.check(h, rc)

    if args.profile:
        call()
        torch.cuda.synchronize()
        return
    f_alg = 2.0 * n * n * m + 4.0 * n * m * (m + p)
    variants = [v for v in args.variants.split(",") if v] or [""]
    for var in variants:
        saved = {}
        for kv in [x for x in var.split(";") if x]:
            k, v = kv.split("=")
            saved[k] = os.environ.get(k)
            os.environ[k] = v
        call()
        call()
        torch.cuda.synchronize()
        per = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            call()
            e1.record(st)
            torch.cuda.synchronize()
            per.append(e0.elapsed_time(e1))
        per.sort()
        ms = per[len(per) // 2]
        L.ss_reset_stats(h.ptr)
        L.ss_set_timing(h.ptr, 1)
        call()
        torch.cuda.synchronize()
        L.ss_set_timing(h.ptr, 0)
        sec5 = (ctypes.c_double * 5)()
        fl5 = (ctypes.c_double * 5)()
        L.ss_phase_stats(h.ptr, sec5, fl5)
        ul, us, ua = ctypes.c_int64(0), ctypes.c_double(0.0), ctypes.c_double(0.0)
        L.ss_update_kernel_stats(h.ptr, ctypes.byref(ul), ctypes.byref(us), ctypes.byref(ua))
        ach = ua.value / us.value / 1e12 if us.value else 0
        print(f"cfg{args.cfg} n={n} m={m} s={s} nb={args.nb} [{var or 'default'}] "
              f"{ms:.3f} ms/call (median; min {per[0]:.3f} max {per[-1]:.3f})  {s / ms * 1e3:.0f} shifts/s  sweep {f_alg * s / ms / 1e9:.2f} TF | "
              f"timed: rq {sec5[1]*1e3:.2f} ms, update {(sec5[2]+sec5[3])*1e3:.2f} ms "
              f"({ach:.2f} TF alg), head {sec5[4]*1e3:.3f} ms", flush=True)
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    # parity spot check vs a dense solve of a few shifts (large n: complex128
    # LU on the device through torch -- a checker, not the product path)
    if n > 4000:
        Ad = A.to(torch.complex128)
        for l in (0, s - 1):
            sig = sh[l].item()
            Ms = Ad - sig * torch.eye(n, dtype=torch.complex128, device=A.device)
            X = torch.linalg.solve(Ms, B.to(torch.complex128))
            Gr = -(C.to(torch.complex128) @ X)
            err = float(torch.linalg.norm(G[:, l * m:(l + 1) * m] - Gr) / torch.linalg.norm(Gr))
            print(f"  shift {l}: rel err vs dense solve {err:.2e}", flush=True)
            del Ms, X
        return
    Ah, Bh, Ch = (x.cpu().numpy() for x in (A, B, C))
    Gh = G.cpu().numpy()
    for l in (0, s // 2, s - 1):
        sig = sh[l].item()
        X = np.linalg.solve(Ah - sig * np.eye(n), Bh)
        Gr = -Ch @ X
        err = np.linalg.norm(Gh[:, l * m:(l + 1) * m] - Gr) / np.linalg.norm(Gr)
        print(f"  shift {l}: rel err vs dense solve {err:.2e}")


if __name__ == "__main__":
    main()
