"""Where the e2e time of eval_transfer_function (pinned host inputs) goes,
beyond the device sweep (experiment tooling, not part of the product)."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1708_06290_b200 as ss
from paper_1708_06290_b200 import _device as D, _lib
from bench import synthetic_triple

n, m, p, s = 4000, 10, 10, 1000
A, B, C = synthetic_triple(n, m, p, seed=2)
A_h = torch.as_tensor(A).t().contiguous().t().pin_memory()
B_h = torch.as_tensor(B).pin_memory(); C_h = torch.as_tensor(C).pin_memory()
sh_h = torch.from_numpy(1j * np.logspace(-2, 2, s) * np.sqrt(n)).pin_memory()
chf = ss.ControllerHessForm(Ahat=A_h, Bhat=B_h, Chat=C_h, m=m, n=n, p=p)
for _ in range(3):
    ss.eval_transfer_function(chf, sh_h, nb=64, on_singular="mark")
ts = []
for _ in range(7):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ss.eval_transfer_function(chf, sh_h, nb=64, on_singular="mark")
    ts.append(time.perf_counter() - t0)
print("e2e ms", [round(1e3 * t, 2) for t in ts])
# device-only sweep on resident inputs for comparison
dev = torch.device("cuda", 0)
chf_d = ss.ControllerHessForm(Ahat=A_h.to(dev), Bhat=B_h.to(dev), Chat=C_h.to(dev), m=m, n=n, p=p)
sh_d = sh_h.to(dev)
ts = []
for _ in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = ss.eval_transfer_function(chf_d, sh_d, nb=64, on_singular="mark")
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print("device-resident API ms", [round(1e3 * t, 2) for t in ts])
# pieces
torch.cuda.synchronize(); t0 = time.perf_counter()
Bd = D.fmat(B_h, torch.float64, dev); Cd = D.fmat(C_h, torch.float64, dev); sd = D.fvec(sh_h, torch.complex128, dev)
torch.cuda.synchronize(); t1 = time.perf_counter()
G = torch.empty((s * m, p), dtype=torch.complex128, device=dev).t()
t2 = time.perf_counter(); Gh = G.cpu(); t3 = time.perf_counter()
print(f"small H2D {1e3*(t1-t0):.3f} ms, G D2H {1e3*(t3-t2):.3f} ms")
