"""The reduction's FP64 tensor-core GEMM (csrc/ss_gemm.cuh, C ABI ss_dgemm)
against a plain PyTorch float64 matmul: every transpose combination, the
tile shapes the host picks (N <= 8, <= 32, <= 64, M <= 64, wide), ragged and
unaligned sub-matrices (offset pointers, odd leading dimensions), split-K
(long K, small output) and alpha / beta.  Tolerance: 1e-13 relative to
|alpha| |op(A)| |op(B)| + |beta| |C| elementwise (FP64 accumulation in a
different order)."""

import ctypes

import numpy as np
import pytest
import torch

from paper_1708_06290_b200 import _device as D
from paper_1708_06290_b200 import _lib

pytestmark = pytest.mark.gpu


def run(ta, tb, M, N, K, alpha, beta, off=0, pad=0, seed=0, pad_fn=None):
    g = torch.Generator(device="cuda").manual_seed(seed)
    dev = torch.device("cuda", 0)
    ra, ca = (K, M) if ta else (M, K)
    rb, cb = (N, K) if tb else (K, N)

    def mat(r, c):  # column-major with an odd leading dimension and an offset start
        ld = r + off + (pad if pad_fn is None else pad_fn(r + off))
        buf = torch.randn(ld * c + off + 8, dtype=torch.float64, device=dev, generator=g)
        return buf, ld

    Ab, lda = mat(ra, ca)
    Bb, ldb = mat(rb, cb)
    Cb, ldc = mat(M, N)
    view = lambda b, ld, r, c: b[off:off + ld * c].view(c, ld).t()[:r, :]
    A, B, C0 = view(Ab, lda, ra, ca), view(Bb, ldb, rb, cb), view(Cb, ldc, M, N).clone()
    opA = A.t() if ta else A
    opB = B.t() if tb else B
    ref = alpha * (opA @ opB) + beta * C0
    bound = abs(alpha) * (opA.abs() @ opB.abs()) + abs(beta) * C0.abs()
    h = _lib.handle(0)
    L = _lib.load()
    ptr = lambda b: ctypes.c_void_p(b.data_ptr() + off * 8)
    rc = L.ss_dgemm(h.ptr, int(ta), int(tb), M, N, K, alpha, ptr(Ab), lda, ptr(Bb), ldb, beta,
                    ptr(Cb), ldc, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    D.check(h, rc)
    torch.cuda.synchronize()
    out = view(Cb, ldc, M, N)
    err = ((out - ref).abs() / bound.clamp_min(1e-300)).max().item()
    return err


@pytest.mark.parametrize("ta", [0, 1])
@pytest.mark.parametrize("tb", [0, 1])
@pytest.mark.parametrize("M,N,K", [(300, 5, 257), (517, 30, 96), (1000, 50, 64), (40, 700, 333),
                                   (1100, 900, 64), (257, 129, 4000), (64, 1500, 2000),
                                   (3000, 1, 3000), (1, 1, 1), (130, 70, 0)])
def test_dgemm_vs_torch(ta, tb, M, N, K):
    err = run(ta, tb, M, N, K, alpha=-1.0, beta=1.0, off=3, pad=1, seed=M + N + K)
    assert err <= 1e-13


@pytest.mark.parametrize("alpha,beta", [(1.0, 0.0), (0.5, -2.0), (2.0, 1.0)])
def test_dgemm_alpha_beta(alpha, beta):
    assert run(0, 1, 700, 300, 128, alpha, beta, off=1, pad=3, seed=7) <= 1e-13
    assert run(1, 0, 64, 900, 3000, alpha, beta, off=0, pad=0, seed=8) <= 1e-13


def test_dgemm_deterministic():
    """Split-K partials are summed in a fixed order: bitwise repeatable."""
    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cuda").manual_seed(3)
    M, N, K = 300, 40, 20000
    A = torch.randn(K, M, dtype=torch.float64, device=dev, generator=g)
    B = torch.randn(N, K, dtype=torch.float64, device=dev, generator=g)
    h = _lib.handle(0)
    L = _lib.load()
    outs = []
    for _ in range(3):
        C = torch.zeros(N, M, dtype=torch.float64, device=dev)  # column-major M x N
        rc = L.ss_dgemm(h.ptr, 1, 1, M, N, K, 1.0, ctypes.c_void_p(A.data_ptr()), K,
                        ctypes.c_void_p(B.data_ptr()), N, 0.0, ctypes.c_void_p(C.data_ptr()), M,
                        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        D.check(h, rc)
        outs.append(C.clone())
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])


@pytest.mark.parametrize("ta", [0, 1])
@pytest.mark.parametrize("tb", [0, 1])
@pytest.mark.parametrize("M,N,K", [(301, 7, 257), (516, 30, 96), (1000, 51, 64), (41, 700, 333),
                                   (1100, 901, 64), (64, 1500, 2001), (3001, 1, 3000)])
def test_dgemm_aligned_path(ta, tb, M, N, K):
    """Even leading dimensions and 16-byte aligned bases take the paired
    16-byte copies (odd extents end in a half-filled pair)."""
    def pad_even(r):  # leading dimension r + pad made even
        return 0 if r % 2 == 0 else 1
    err = run(ta, tb, M, N, K, alpha=-1.0, beta=1.0, off=0, pad=0, seed=M * 3 + N + K,
              pad_fn=pad_even)
    assert err <= 1e-13
