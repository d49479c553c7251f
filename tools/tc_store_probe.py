"""Dense tensor-core engine legs (config 3 sparse sign, Gaussian, DCT SRTT at the config-2 shape):
back-to-back kernel time over 20 launches (for the epilogue store-pattern change)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_21189_b200 import sketch as skb  # noqa: E402

legs = [("cfg3", skb.SparseUniformTM(16384, 200, 8, seed=0), torch.randn(131072, 16384, device="cuda")),
        ("dct", skb.SparseRttTM(8192, 512, 1, "dct", seed=0), torch.randn(65536, 8192, device="cuda"))]
for name, tm, a in legs:
    for _ in range(3):
        tm.apply_right(a)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(20):
        tm.apply_right(a)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"{name}: {ev[0].elapsed_time(ev[1]) / 20:.4f} ms", flush=True)
    del a
    torch.cuda.empty_cache()
