"""Host enqueue time vs GPU time per ss_tf_eval call for configs 1-3 (experiment tooling)."""
import ctypes, os, sys, time
import numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1708_06290_b200 import _device as D, _lib
from bench import synthetic_triple
from paper_1708_06290_b200.systems import CONFIGS
for cfg in (1, 3, 2):
    n, m, p, s = CONFIGS[cfg]
    A, B, C = synthetic_triple(n, m, p, seed=cfg)
    dev = torch.device("cuda", 0)
    A, B, C = (torch.as_tensor(x).to(dev) for x in (A, B, C))
    sh = torch.from_numpy(1j * np.logspace(-2, 2, s) * np.sqrt(n)).to(dev)
    G = torch.empty((s * m, p), dtype=torch.complex128, device=dev).t()
    fail = torch.empty(s, dtype=torch.int32, device=dev)
    h = _lib.handle(0); L = _lib.load(); st = torch.cuda.current_stream(dev)
    def call():
        D.check(h, L.ss_tf_eval(h.ptr, n, m, p, D.ptr(A), D.ld(A), D.ptr(B), D.ld(B), D.ptr(C), D.ld(C),
                                D.ptr(sh), s, 64, 0, float("nan"), D.ptr(G), p, D.ptr(fail), ctypes.c_void_p(st.cuda_stream)))
    for _ in range(3): call()
    torch.cuda.synchronize()
    enq, gpu = [], []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter(); e0.record(st); call(); e1.record(st); t1 = time.perf_counter()
        torch.cuda.synchronize()
        enq.append(1e3 * (t1 - t0)); gpu.append(e0.elapsed_time(e1))
    print(f"cfg{cfg}: enqueue median {np.median(enq):.3f} ms, gpu median {np.median(gpu):.3f} ms, launches/call {h.launches() if hasattr(h,'launches') else '?'}")
