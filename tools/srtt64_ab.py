"""Float64 SRTT-WHT at the config-2 shape: the wide kernel (2 phases + gather fold) vs the 3-phase
fast path (SKETCH_B200_SRTT64=3), interleaved; parity of the two against each other."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_21189_b200.sketch import SparseRttTM  # noqa: E402

a = torch.randn(65536, 8192, device="cuda", dtype=torch.float64)
tm = SparseRttTM(8192, 512, 1, "wht", seed=0)
res = {}
outs = {}
for m in ("wide", "3"):
    os.environ["SKETCH_B200_SRTT64"] = m
    outs[m] = tm.apply_right(a)
print("max rel diff", float((outs["wide"] - outs["3"]).norm() / outs["3"].norm()))
for it in range(5):
    for m in ("wide", "3"):
        os.environ["SKETCH_B200_SRTT64"] = m
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        tm.apply_right(a)
        ev[0].record()
        for _ in range(5):
            tm.apply_right(a)
        ev[1].record()
        torch.cuda.synchronize()
        res.setdefault(m, []).append(ev[0].elapsed_time(ev[1]) / 5)
for m, v in res.items():
    ms = statistics.median(v)
    print(f"{m}: {ms:.3f} ms  {65536 * 8192 * 8 / ms / 1e6:.0f} GB/s")
