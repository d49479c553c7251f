"""Host-side cost of one apply_right call (Python + ctypes) against the kernel time, config 1."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_21189_b200 import sketch as skb  # noqa: E402

tm = skb.SparseUniformTM(4096, 256, 4, seed=0)
a = torch.randn(16384, 4096, dtype=torch.float64, device="cuda")
small = torch.randn(64, 4096, dtype=torch.float64, device="cuda")
for _ in range(5):
    tm.apply_right(a)
torch.cuda.synchronize()
# host cost: tiny input so the GPU never backs up the launch queue
t0 = time.perf_counter()
for _ in range(200):
    tm.apply_right(small)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host per call (64 rows): {(t1 - t0) / 200 * 1e6:.1f} us")
import cProfile  # noqa: E402
import pstats  # noqa: E402

pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    tm.apply_right(small)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(50):
    tm.apply_right(a)
ev[1].record()
torch.cuda.synchronize()
print(f"back-to-back kernel-bound: {ev[0].elapsed_time(ev[1]) / 50 * 1e3:.1f} us per call")
