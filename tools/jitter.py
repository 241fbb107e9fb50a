"""Host-jitter diagnostic for the bench step (not part of the product):
per-step host enqueue time vs GPU time, and per-call e2e wall time."""
import ctypes, os, sys, time, statistics
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1708_06290_b200 as ss
from paper_1708_06290_b200 import _device as D, _lib
from bench import synthetic_triple

n, m, p, s = 4000, 10, 10, 1000
A, B, C = synthetic_triple(n, m, p, seed=2)
dev = torch.device("cuda", 0)
A, B, C = (torch.as_tensor(x).to(dev) for x in (A, B, C))
sh = torch.from_numpy(1j * np.logspace(-2, 2, s) * np.sqrt(n)).to(dev)
G = torch.empty((s * m, p), dtype=torch.complex128, device=dev).t()
fail = torch.empty(s, dtype=torch.int32, device=dev)
h = _lib.handle(0); L = _lib.load()
stream = torch.cuda.current_stream(dev)
def step():
    D.check(h, L.ss_tf_eval(h.ptr, n, m, p, D.ptr(A), D.ld(A), D.ptr(B), D.ld(B), D.ptr(C), D.ld(C),
                            D.ptr(sh), s, 64, 0, float("nan"), D.ptr(G), p, D.ptr(fail),
                            ctypes.c_void_p(stream.cuda_stream)))
for _ in range(3): step()
torch.cuda.synchronize()
for i in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(stream); step(); e1.record(stream); t1 = time.perf_counter()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"step {i}: enqueue {1e3*(t1-t0):.2f} ms  gpu {e0.elapsed_time(e1):.2f} ms  wall {1e3*(t2-t0):.2f} ms")
# back-to-back
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
t0 = time.perf_counter()
for _ in range(5): step()
t1 = time.perf_counter()
e1.record(stream); torch.cuda.synchronize()
print(f"5 back-to-back: enqueue {1e3*(t1-t0):.2f} ms, gpu {e0.elapsed_time(e1)/5:.2f} ms/step")
# e2e
A_h = A.cpu().t().contiguous().t().pin_memory(); B_h = B.cpu().pin_memory(); C_h = C.cpu().pin_memory()
sh_h = sh.cpu().pin_memory()
chf = ss.ControllerHessForm(Ahat=A_h, Bhat=B_h, Chat=C_h, m=m, n=n, p=p)
ss.eval_transfer_function(chf, sh_h, nb=64, on_singular="mark")
for i in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ss.eval_transfer_function(chf, sh_h, nb=64, on_singular="mark")
    t1 = time.perf_counter()
    print(f"e2e {i}: {1e3*(t1-t0):.2f} ms")
