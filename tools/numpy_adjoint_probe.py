"""NumPy drop-in S*A at the config-4 shape (pageable float32 A, 8.6 GB): wall clock per call with the
staged pinned upload vs a plain pageable upload (STAGED_UPLOAD_MIN_BYTES raised)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_21189_b200 import _device  # noqa: E402
from paper_2508_21189_b200.sketch import SparseUniformTM  # noqa: E402

tm = SparseUniformTM(4194304, 2048, 8, seed=0)
a = np.random.default_rng(0).standard_normal((4194304, 512), dtype=np.float32)
for label, thr in (("staged", 64 << 20), ("pageable", 1 << 62), ("staged", 64 << 20)):
    _device.STAGED_UPLOAD_MIN_BYTES = thr
    tm.apply_adjoint(a[:1000].repeat(4194, axis=0)[:4194304] if False else a)
    t0 = time.perf_counter()
    sa = tm.apply_adjoint(a)
    dt = time.perf_counter() - t0
    print(f"{label}: {dt * 1e3:.1f} ms per call ({a.nbytes / dt / 1e9:.1f} GB/s of A), out {sa.dtype} {sa.shape}",
          flush=True)
