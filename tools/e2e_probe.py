"""Per-step end-to-end timings of apply_right(pinned host A) at the config-2 shape."""
import sys
import time

import torch

sys.path.insert(0, "/root/repo")
from paper_2508_21189_b200.sketch import SparseRttTM  # noqa: E402

dev = torch.device("cuda", 0)
tm = SparseRttTM(8192, 512, 1, "wht", seed=0)
a = torch.randn(65536, 8192, device=dev)
a_host = torch.empty(a.shape, dtype=a.dtype, pin_memory=True)
a_host.copy_(a)
for i in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    y = tm.apply_right(a_host)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"step {i}: {dt * 1e3:7.2f} ms  {a_host.numel() * 4 / dt / 1e9:6.1f} GB/s", flush=True)
