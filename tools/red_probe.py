#!/usr/bin/env python
"""Controller-Hessenberg reduction timing on one GPU (experiment tooling).

    python tools/red_probe.py [--n 10000] [--m 20] [--p 20] [--reps 2] [--profile]

Times ss_reduce_chf (CUDA events, after one warm call at the same size) on a
seeded dense Gaussian system and prints ms, the reference flop count
(the figure the phase counters report) and TFLOP/s.
--profile: one call, no timing (for ncu)."""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10000)
    ap.add_argument("--m", type=int, default=20)
    ap.add_argument("--p", type=int, default=20)
    ap.add_argument("--b", type=int, default=64)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--profile", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_1708_06290_b200 as ss

    n, m, p = args.n, args.m, args.p
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(n + m)
    A0 = torch.randn((n, n), dtype=torch.float64, device=dev, generator=g) - 1.1 * np.sqrt(n) * torch.eye(
        n, dtype=torch.float64, device=dev)
    B0 = torch.randn((n, m), dtype=torch.float64, device=dev, generator=g)
    C0 = torch.randn((p, n), dtype=torch.float64, device=dev, generator=g)

    def call():
        return ss.reduce_controller_hessenberg(A0.clone(), B0.clone(), C0.clone(), block_size=args.b)

    if args.profile:
        call()
        torch.cuda.synchronize()
        return
    call()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.reps):
        A, B, C = A0.clone(), B0.clone(), C0.clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ss.reduce_controller_hessenberg(A, B, C, block_size=args.b)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    b = min(args.b, 128)
    fl = 10 / 3 * n ** 3 + 2.5 * n * n * b - 4.5 * n * n * m + n * n * m * m / (2 * b)
    ms = min(ts)
    print(json.dumps({"n": n, "m": m, "p": p, "b": args.b, "ms": ms, "all_ms": ts,
                      "ref_flops": fl, "tflops": fl / ms / 1e9}))


if __name__ == "__main__":
    main()
