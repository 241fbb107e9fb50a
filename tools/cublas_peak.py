import torch, time
a=torch.randn(8192,8192,dtype=torch.float64,device='cuda'); b=torch.randn_like(a)
for _ in range(3): c=a@b
torch.cuda.synchronize()
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): c=a@b
e1.record(); torch.cuda.synchronize()
ms=e0.elapsed_time(e1)/10
print("cublas dgemm 8192^3:", 2*8192**3/ms/1e9, "TFLOP/s")
