"""SparseRttTM with the DCT transform (the reference's real-field default) at the config-2 shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_21189_b200 import sketch as skb  # noqa: E402

dev = torch.device("cuda", 0)
a = torch.randn(65536, 8192, device=dev)
for tr in ("wht", "dct"):
    tm = skb.SparseRttTM(8192, 512, 1, tr, seed=0)
    tm.apply_right(a)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        tm.apply_right(a)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"{tr}: {ms:.3f} ms  {(a.numel() + 65536 * 512) * 4 / ms / 1e6:.0f} GB/s")
