"""Probe tcgen05 accumulation precision: error of the K-TC engine vs K for exact +-1 B."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2508_21189_b200.sketch.tensorcore import bt_from_triplets, dense_right_tc
dev = torch.device("cuda", 0)
rng = np.random.default_rng(0)
k = 256
for d in (1024, 4096, 16384, 65536):
    for kind in ("iid", "lowrank"):
        n = 64
        if kind == "iid":
            a = rng.standard_normal((n, d))
        else:
            r = int(np.sqrt(d))
            u = rng.standard_normal((n, 5, r)); v = rng.standard_normal((n, 5, r))
            a = np.einsum("nrp,nrq->npq", u, v).reshape(n, d) + 1e-2 * rng.standard_normal((n, d))
        a = a.astype(np.float32)
        b = np.where(rng.random((d, k)) < 0.5, -1.0, 1.0)
        rows, cols = np.nonzero(b)
        hi, lo = bt_from_triplets(rows, cols, b[rows, cols] < 0, d, k, dev)
        y = dense_right_tc(torch.from_numpy(a).to(dev), hi, lo, k, 1.0).double().cpu().numpy()
        ref = a.astype(np.float64) @ b
        # emulate BF16x2 input rounding only
        a_hi = torch.from_numpy(a).to(torch.bfloat16).float().numpy()
        a_lo = torch.from_numpy(a - a_hi).to(torch.bfloat16).float().numpy()
        emu = (a_hi.astype(np.float64) + a_lo) @ b
        e = np.linalg.norm(y - ref) / np.linalg.norm(ref)
        e2 = np.linalg.norm(emu - ref) / np.linalg.norm(ref)
        # fp32 sequential accumulation emulation
        print(f"d={d:6d} {kind:8s} tc_err={e:.2e} input_rounding_err={e2:.2e}", flush=True)
