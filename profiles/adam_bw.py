import torch, time
n = 3_000_000 * 87
p = torch.randn(n, device='cuda'); g = torch.randn(n, device='cuda')
p.grad = g
opt = torch.optim.Adam([p], lr=1e-3, fused=True)
for _ in range(3): opt.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): opt.step()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("torch fused adam ms", ms, "GB/s (7 streams of 4B)", 28 * n / ms / 1e6)
a = torch.empty(n, device='cuda'); b = torch.empty(n, device='cuda')
e0.record()
for _ in range(10): b.copy_(a)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("copy ms", ms, "GB/s", 8 * n / ms / 1e6)

# the library's fused Adam over the [N, 87] records (train.Adam -> gsx_adam_step)
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07782_b200.train import Adam
P = torch.rand((3_000_000, 87), device='cuda') + 0.5
G_ = torch.randn((3_000_000, 87), device='cuda') * 1e-3
opt2 = Adam(P, 0.01, None)
for _ in range(3): opt2.step(G_)
torch.cuda.synchronize()
e0.record()
for _ in range(10): opt2.step(G_)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("gsx_adam_step ms", ms, "GB/s", 28 * P.numel() / ms / 1e6)
