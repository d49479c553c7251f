"""Config-4 S*A launch-by-launch times over a long back-to-back series (drift / bimodality check)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_21189_b200 import sketch as skb  # noqa: E402

tm = skb.SparseUniformTM(4194304, 2048, 8, seed=0)
a = torch.randn(4194304, 512, device="cuda")
tm.apply_adjoint(a)
torch.cuda.synchronize()
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(60)]
for s, e in evs:
    s.record()
    tm.apply_adjoint(a)
    e.record()
torch.cuda.synchronize()
t = [s.elapsed_time(e) for s, e in evs]
print(" ".join(f"{x:.2f}" for x in t))
print(f"first10 {sum(t[:10]) / 10:.3f}  last10 {sum(t[-10:]) / 10:.3f}  min {min(t):.3f}")
