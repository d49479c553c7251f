"""End-to-end drop-in call with NumPy input (the reference's calling convention): config-2 SRTT on a
pageable float32 / float64 NumPy array, wall clock per call (host staging, PCIe, kernel, result)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_21189_b200.sketch import SparseRttTM  # noqa: E402

tm = SparseRttTM(8192, 512, 1, "wht", seed=0)
rng = np.random.default_rng(0)
for dt in (np.float32, np.float64):
    a = rng.standard_normal((65536, 8192)).astype(dt)
    tm.apply_right(a[:1024])
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        y = tm.apply_right(a)
        ts.append(time.perf_counter() - t0)
    gb = a.nbytes / 1e9
    print(f"numpy {np.dtype(dt).name}: {[round(t * 1e3, 1) for t in ts]} ms per call; best {gb / min(ts):.1f} GB/s of A "
          f"(out {y.dtype}, {y.shape})", flush=True)
