"""Headline kernel (config-2 SRTT) timing forms: one launch after idle vs back-to-back launches.

    python tools/headline_timing.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_21189_b200 import sketch as skb  # noqa: E402

dev = torch.device("cuda", 0)
a = torch.randn(65536, 8192, device=dev)
a /= torch.arange(1, 8193, device=dev, dtype=torch.float32)
tm = skb.SparseRttTM(8192, 512, 1, "wht", seed=0)
y = tm.apply_right(a)
alg = a.numel() * 4 + y.numel() * 4
for _ in range(5):
    tm.apply_right(a)
torch.cuda.synchronize()


def ev():
    return torch.cuda.Event(enable_timing=True)


singles = []
for _ in range(10):
    time.sleep(0.05)
    s, e = ev(), ev()
    s.record()
    tm.apply_right(a)
    e.record()
    torch.cuda.synchronize()
    singles.append(s.elapsed_time(e))
for reps in (2, 10, 50):
    s, e = ev(), ev()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        tm.apply_right(a)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    print(f"back-to-back x{reps}: {ms:.4f} ms/launch  {alg / ms / 1e6:.0f} GB/s", flush=True)
singles.sort()
print(f"single after idle: min {singles[0]:.4f} median {singles[5]:.4f} ms  ({alg / singles[5] / 1e6:.0f} GB/s)")

# per-launch kernel time with the host well ahead (events enqueued around each launch, no host gap
# inside the timed region) after a GPU-side idle gap of `gap_ms`
for gap_ms in (0.0, 0.2, 1.0, 5.0):
    ts = []
    for _ in range(10):
        if gap_ms:
            torch.cuda._sleep(int(gap_ms * 1.9e6))  # GPU-side spin (cycles at ~1.9 GHz)
        s, e = ev(), ev()
        s.record()
        tm.apply_right(a)
        e.record()
        ts.append((s, e))
    torch.cuda.synchronize()
    v = sorted(s.elapsed_time(e) for s, e in ts)
    print(f"gap {gap_ms} ms: per-launch median {v[5]:.4f} min {v[0]:.4f} ms", flush=True)
