"""Config-2 shape SRTT with float64 A (the reference's dtype)."""
import sys
import torch
sys.path.insert(0, "/root/repo")
from paper_2508_21189_b200.sketch import SparseRttTM  # noqa: E402
dev = torch.device("cuda", 0)
a = torch.randn(65536, 8192, device=dev, dtype=torch.float64)
tm = SparseRttTM(8192, 512, 1, "wht", seed=0)
tm.apply_right(a)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(5):
    tm.apply_right(a)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"f64 SRTT {ms:.3f} ms  {a.numel() * 8 / ms / 1e6:.0f} GB/s")
