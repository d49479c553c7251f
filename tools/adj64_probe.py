"""Config-4 shape SA with float64 A (the reference's dtype): K2 gather path timing."""
import sys
import torch
sys.path.insert(0, "/root/repo")
from paper_2508_21189_b200.sketch import SparseUniformTM  # noqa: E402

dev = torch.device("cuda", 0)
n, d, k = 4194304, 512, 2048
a = torch.randn(n, d, device=dev, dtype=torch.float64)
tm = SparseUniformTM(n, k, 8, seed=0)
print("path", tm.adjoint_path(a))
y = tm.apply_adjoint(a)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(3):
    y = tm.apply_adjoint(a)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"f64 SA {ms:.2f} ms  {n * d * 8 / ms / 1e6:.0f} GB/s")
