"""Fused two-sided sketch at the DESIGN section-6 shape: lane-pair sector adds of the Y partials
(default) vs per-lane row adds (SKETCH_B200_TS_DBG=16), interleaved; outputs compared."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_21189_b200 import rand_nla as rn  # noqa: E402
from paper_2508_21189_b200 import sketch as skb  # noqa: E402

n, d, k, p = 1 << 21, 512, 64, 96
a = torch.randn(n, d, device="cuda")
om = skb.SparseRttTM(d, k, 1, "wht", seed=1)
ps = skb.SparseUniformTM(n, p, 8, seed=2)
outs = {}
for m in ("0", "16"):
    os.environ["SKETCH_B200_TS_DBG"] = m
    outs[m] = rn.two_sided_sketch(a, om, ps, fused=True)
    torch.cuda.synchronize()
print("Y rel diff", float((outs["0"][0] - outs["16"][0]).norm() / outs["16"][0].norm()))
t = {"0": [], "16": []}
for it in range(8):
    for m in ("0", "16"):
        os.environ["SKETCH_B200_TS_DBG"] = m
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        rn.two_sided_sketch(a, om, ps, fused=True)
        ev[0].record()
        for _ in range(5):
            rn.two_sided_sketch(a, om, ps, fused=True)
        ev[1].record()
        torch.cuda.synchronize()
        t[m].append(ev[0].elapsed_time(ev[1]) / 5)
for m in ("0", "16"):
    print(f"dbg={m}: median {statistics.median(t[m]):.3f} ms  min {min(t[m]):.3f}")
