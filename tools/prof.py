"""Profiling driver: run one config's kernel a few times (for ncu / compute-sanitizer on one GPU)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--rows", type=int, default=0, help="truncate the input to this many rows (0 = full)")
args = ap.parse_args()
dev = torch.device("cuda", 0)
w = bench.WORKLOADS[args.config](torch, dev, 0)
if args.rows:
    w["a"] = w["a"][: args.rows].contiguous()
    w["n"] = args.rows
for _ in range(args.reps):
    bench._apply(w, w["a"])
torch.cuda.synchronize()
print("ok", args.config, tuple(w["a"].shape))
