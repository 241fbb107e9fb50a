#!/usr/bin/env python
"""Transposed-solve timing (IRKA's inner solve) on one GPU, experiment
tooling: solve_shifted_transposed on a synthetic m-Hessenberg triple.
    python tools/lq_probe.py [--n 10000] [--m 20] [--s 40] [--profile]"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10000)
    ap.add_argument("--m", type=int, default=20)
    ap.add_argument("--s", type=int, default=40)
    ap.add_argument("--profile", action="store_true")
    a = ap.parse_args()
    import torch

    import paper_1708_06290_b200 as ss
    from bench import synthetic_triple

    A, B, C = synthetic_triple(a.n, a.m, a.m, seed=5)
    dev = torch.device("cuda", 0)
    chf = ss.ControllerHessForm(Ahat=torch.from_numpy(A).to(dev), Bhat=torch.from_numpy(B).to(dev),
                                Chat=torch.from_numpy(C).to(dev), m=a.m, n=a.n, p=a.m)
    rng = np.random.default_rng(0)
    sh = torch.from_numpy((rng.uniform(0.05, 1, a.s) + 1j * rng.uniform(0, 1.5, a.s)) * np.sqrt(a.n)).to(dev)
    rhs = torch.from_numpy(rng.standard_normal((a.n, a.s)) + 1j * rng.standard_normal((a.n, a.s))).to(dev)
    call = lambda: ss.solve_shifted_transposed(chf, sh, rhs, nb=32, on_singular="mark")
    call()
    torch.cuda.synchronize()
    if a.profile:
        return
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(json.dumps({"n": a.n, "m": a.m, "shifts": a.s, "ms": ms, "shifts_per_s": a.s / ms * 1e3}))


if __name__ == "__main__":
    main()
