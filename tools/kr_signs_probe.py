"""Config 5 Khatri-Rao A/B timing (CUDA events, modes interleaved launch by launch so clock drift hits
all equally; medians): sign-bit weights (sk_kr_right_signs) vs float32 weights
(SKETCH_B200_KR_SIGNS=0), with and without the partner-pair lockstep (SKETCH_B200_KR_LOCKSTEP=off)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_21189_b200 import sketch as skb  # noqa: E402

tm = skb.KhatriRaoTM(256, 2, 512, "real_rademacher", seed=0)
a = torch.randn(16384, 65536, device="cuda")
modes = [("1", None), ("1", "off"), ("0", None), ("0", "off")]


def setm(signs, lock):
    os.environ["SKETCH_B200_KR_SIGNS"] = signs
    if lock:
        os.environ["SKETCH_B200_KR_LOCKSTEP"] = lock
    else:
        os.environ.pop("SKETCH_B200_KR_LOCKSTEP", None)


times = {m: [] for m in modes}
for m in modes:
    setm(*m)
    tm.apply_right(a)
torch.cuda.synchronize()
for it in range(15):
    for m in modes:
        setm(*m)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        tm.apply_right(a)
        ev[1].record()
        torch.cuda.synchronize()
        times[m].append(ev[0].elapsed_time(ev[1]))
for m in modes:
    print(f"signs={m[0]} lockstep={'off' if m[1] else 'on'}: median {statistics.median(times[m]):.4f} ms "
          f"min {min(times[m]):.4f}", flush=True)
