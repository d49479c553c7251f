"""K1c vs K1r / K1 timing on sparse-sign right applies (config 1 and neighbours), CUDA events."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_21189_b200 import sketch as skb  # noqa: E402


def t_apply(tm, a, reps=20):
    for _ in range(3):
        tm.apply_right(a)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(reps):
        tm.apply_right(a)
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps


shapes = [(16384, 4096, 256, 4, torch.float64), (16384, 4096, 256, 4, torch.float32), (65536, 2048, 128, 2, torch.float64),
          (8192, 8192, 256, 8, torch.float64), (65536, 16384, 200, 8, torch.float64)]
for n, d, k, z, dt in shapes:
    a = torch.randn(n, d, dtype=dt, device="cuda")
    gb = (a.numel() + n * k) * a.element_size() / 1e9
    res = {}
    for mode in ("cols", "ring", "classic"):
        if mode == "ring" and dt == torch.float32:
            continue
        os.environ["SKETCH_B200_K1"] = mode
        tm = skb.SparseUniformTM(d, k, z, seed=0)
        ms = t_apply(tm, a)
        res[mode] = ms
    ref = None
    print(f"n={n} d={d} k={k} zeta={z} {str(dt)[6:]}: " + "  ".join(f"{m} {v:.4f} ms ({gb / v:.0f} GB/s)" for m, v in res.items()),
          flush=True)
