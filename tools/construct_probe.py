"""Config-4 operator construction: host NumPy draws vs device draws (devrng), then the K2w encoding."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_21189_b200 import sketch as skb  # noqa: E402

torch.zeros(1, device="cuda")
for mode in ("1", "0"):
    os.environ["SKETCH_B200_HOST_RNG"] = mode
    t0 = time.perf_counter()
    tm = skb.SparseUniformTM(4194304, 2048, 8, seed=0)
    tm._triplets()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    tm._adjoint_wide_on(torch.device("cuda", 0))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{'host' if mode == '1' else 'device'} draws: {t1 - t0:.3f} s; wide encoding + upload: {t2 - t1:.3f} s")
