"""Config-5 Khatri-Rao timing probe: sk_kr_right variants vs the materialised-Omega dense engine.

    python tools/kr_probe.py [--reps 10]

`kr` = sk_kr_right (F^T resident, per-P fold with W, Omega never formed).  `dense` = the round-1 path: Omega^T (512 x 65536 bf16)
formed on the device and streamed as the B operand of sk_dense_right_tc.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2508_21189_b200.sketch import KhatriRaoTM  # noqa: E402
from paper_2508_21189_b200.sketch.tensorcore import dense_right_tc  # noqa: E402


def time_fn(fn, reps, trials=5):
    """min over trials of the mean kernel time of `reps` back-to-back calls (CUDA events)"""
    for _ in range(3):
        fn()
    best = float("inf")
    for _ in range(trials):
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(reps):
            fn()
        ev[1].record()
        torch.cuda.synchronize()
        best = min(best, ev[0].elapsed_time(ev[1]) / reps)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--n", type=int, default=16384)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    n, d, k = args.n, 65536, 512
    tm = KhatriRaoTM(256, 2, k, "real_rademacher", seed=0)
    a = torch.randn(n, d, device=dev)
    out = {}
    y0 = None
    out["kr_ms"] = time_fn(lambda: tm.apply_right(a), args.reps)
    y0 = tm.apply_right(a)

    om = torch.as_tensor(tm.materialize(), device=dev)  # d x k float64 (probe only)
    bt = (om.T * np.sqrt(k)).contiguous().to(torch.bfloat16)  # exact +-1
    del om
    out["dense_ms"] = time_fn(lambda: dense_right_tc(a, bt, None, k, 1.0 / np.sqrt(k)), args.reps)
    yd = dense_right_tc(a, bt, None, k, 1.0 / np.sqrt(k))
    out["kr_vs_dense_rel"] = float(torch.linalg.norm(y0 - yd) / torch.linalg.norm(yd))
    out["tflops_executed_kr"] = 2 * 2.0 * n * d * k / (out["kr_ms"] / 1e3) / 1e12
    print(json.dumps(out))


if __name__ == "__main__":
    main()
