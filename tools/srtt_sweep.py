"""SRTT right-apply throughput over d (float32 and float64, ~1-2 GB inputs, k = 512 or d/2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_21189_b200 import sketch as skb  # noqa: E402

dev = torch.device("cuda", 0)
for dt in (torch.float32, torch.float64):
    for L in (6, 8, 9, 10, 11, 12, 13, 14, 15, 16):
        d = 1 << L
        esz = torch.empty((), dtype=dt).element_size()
        n = (1 << 31) // (d * esz) if dt == torch.float32 else (1 << 30) // (d * esz)
        k = min(512, d // 2)
        a = torch.randn(n, d, device=dev, dtype=dt)
        tm = skb.SparseRttTM(d, k, 1, "wht", seed=0)
        tm.apply_right(a[:8])
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            tm.apply_right(a)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 5
        gbs = (a.numel() + n * k) * esz / ms / 1e6
        print(f"{str(dt)[6:]:8s} d={d:6d} n={n:8d} k={k:4d}  {ms:7.3f} ms  {gbs:7.0f} GB/s  {100 * gbs / 6550.4:5.1f}% HBM")
        del a
