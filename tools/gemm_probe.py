#!/usr/bin/env python
"""Reduction GEMM shapes on one GPU (experiment tooling): ss_dgemm (DMMA)
vs torch float64 matmul (cuBLAS, reference only), and the measured DMMA /
DFMA peaks.   python tools/gemm_probe.py"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1708_06290_b200 import _lib  # noqa: E402

SHAPES = [  # (name, ta, tb, M, N, K)
    ("rank64_NT (task a)", 0, 1, 12000, 12000, 64),
    ("rank64_NN (apply_left)", 0, 0, 12000, 12000, 64),
    ("VtM (TN, 64 x n)", 1, 0, 64, 12000, 12000),
    ("MV (NN, n x 64)", 0, 0, 12000, 64, 12000),
    ("Yext (NN, n x 50)", 0, 0, 12000, 50, 12000),
    ("Yext m=20", 0, 0, 8000, 20, 8000),
    ("Yext m=1", 0, 0, 2000, 1, 2000),
]


def main():
    only = sys.argv[1] if len(sys.argv) > 1 else None  # profile mode: one call of one shape
    h = _lib.handle(0)
    L = _lib.load()
    st = torch.cuda.current_stream()
    pk = ctypes.c_double(0)
    pf = ctypes.c_double(0)
    if not only:
        L.ss_probe_dmma_peak(h.ptr, ctypes.byref(pk))
        L.ss_probe_dfma_peak(h.ptr, ctypes.byref(pf))
    out = {"dmma_peak_tflops": pk.value, "dfma_peak_tflops": pf.value, "shapes": []}
    for name, ta, tb, M, N, K in SHAPES:
        dev = torch.device("cuda", 0)
        A = torch.randn((M, K) if not ta else (K, M), dtype=torch.float64, device=dev).t().contiguous().t()
        B = torch.randn((K, N) if not tb else (N, K), dtype=torch.float64, device=dev).t().contiguous().t()
        C = torch.randn(M, N, dtype=torch.float64, device=dev).t().contiguous().t()

        def ours():
            L.ss_dgemm(h.ptr, ta, tb, M, N, K, -1.0, ctypes.c_void_p(A.data_ptr()), A.stride(1),
                       ctypes.c_void_p(B.data_ptr()), B.stride(1), 1.0, ctypes.c_void_p(C.data_ptr()),
                       C.stride(1), ctypes.c_void_p(st.cuda_stream))

        if only:
            if only in name:
                ours()
                torch.cuda.synchronize()
            continue
        opA = A.t() if ta else A
        opB = B.t() if tb else B

        def lib():
            torch.addmm(C, opA, opB, beta=1.0, alpha=-1.0, out=C)

        res = {"name": name, "M": M, "N": N, "K": K}
        for tag, fn in (("ours", ours), ("torch_cublas", lib)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            res[tag + "_ms"] = ms
            res[tag + "_tflops"] = 2.0 * M * N * K / ms / 1e9
        out["shapes"].append(res)
        print(json.dumps(res), flush=True)
    if not only:
        print(json.dumps({"dmma_peak_tflops": pk.value, "dfma_peak_tflops": pf.value}))


if __name__ == "__main__":
    main()
