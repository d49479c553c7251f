"""Config 5 Khatri-Rao: sign-bit weights (sk_kr_right_signs) vs float32 weights (sk_kr_right), CUDA events."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_21189_b200 import sketch as skb  # noqa: E402

tm = skb.KhatriRaoTM(256, 2, 512, "real_rademacher", seed=0)
a = torch.randn(16384, 65536, device="cuda")
for mode in ("1", "0", "1", "0"):
    os.environ["SKETCH_B200_KR_SIGNS"] = mode
    for _ in range(3):
        tm.apply_right(a)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(10):
        tm.apply_right(a)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"signs={mode}: {ev[0].elapsed_time(ev[1]) / 10:.4f} ms", flush=True)
