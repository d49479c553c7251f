"""Config-4 operator setup: host draws + host K2w encoding vs device draws + device encoding."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_21189_b200 import sketch as skb  # noqa: E402

dev = torch.device("cuda", 0)
torch.zeros(1, device=dev)
for mode in ("1", "0"):
    os.environ["SKETCH_B200_HOST_RNG"] = mode
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tm = skb.SparseUniformTM(4194304, 2048, 8, seed=0)
    if mode == "1":
        tm._triplets()
    else:
        tm._device_draw()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    tm._adjoint_wide_on(dev)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{'host' if mode == '1' else 'device'} draws: {t1 - t0:.3f} s; K2w encoding on the "
          f"{'host + upload' if mode == '1' else 'device'}: {t2 - t1:.3f} s")
