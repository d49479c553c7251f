"""Config-4 S*A (K2g): piece size sweep, sizes interleaved launch by launch (medians of 15)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_21189_b200 import sketch as skb  # noqa: E402

tm = skb.SparseUniformTM(4194304, 2048, 8, seed=0)
a = torch.randn(4194304, 512, device="cuda")
sizes = [int(x) for x in (sys.argv[1:] or ["48", "56", "64", "72"])]
times = {s: [] for s in sizes}
for s in sizes:
    os.environ["SKETCH_B200_K2G_PIECE_MB"] = str(s)
    tm.apply_adjoint(a)
torch.cuda.synchronize()
for it in range(15):
    for s in sizes:
        os.environ["SKETCH_B200_K2G_PIECE_MB"] = str(s)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        tm.apply_adjoint(a)
        ev[1].record()
        torch.cuda.synchronize()
        times[s].append(ev[0].elapsed_time(ev[1]))
for s in sizes:
    print(f"piece {s} MB: median {statistics.median(times[s]):.3f} ms  min {min(times[s]):.3f}  max {max(times[s]):.3f}")
