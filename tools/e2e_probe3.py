"""End-to-end steps after a bench-like device section; flags slow pinned / device allocations and GC."""
import gc
import sys
import time

import torch

sys.path.insert(0, "/root/repo")
from paper_2508_21189_b200.sketch import SparseRttTM  # noqa: E402

dev = torch.device("cuda", 0)
tm = SparseRttTM(8192, 512, 1, "wht", seed=0)
a = torch.randn(65536, 8192, device=dev)
for _ in range(13):
    y = tm.apply_right(a)
torch.cuda.synchronize()
tm2 = SparseRttTM(8192, 512, 1, "wht", seed=0)
y2 = tm2.apply_right(a)
del tm2, y2
a_host = torch.empty(a.shape, dtype=a.dtype, pin_memory=True)
a_host.copy_(a)
orig_empty = torch.empty


def timed_empty(*args, **kw):
    t0 = time.perf_counter()
    r = orig_empty(*args, **kw)
    dt = time.perf_counter() - t0
    if dt > 0.002:
        print(f"   slow torch.empty {args} pin={kw.get('pin_memory')} dev={kw.get('device')} {dt * 1e3:.1f} ms", flush=True)
    return r


torch.empty = timed_empty
gc.callbacks.append(lambda phase, info: print(f"   gc {phase} gen{info['generation']}", flush=True) if info["generation"] == 2 else None)
for rep in range(3):
    for i in range(3):
        y = tm.apply_right(a_host)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range(5):
        y = tm.apply_right(a_host)
        t2 = time.perf_counter()
        print(f"rep {rep} step {i}: {1e3 * (t2 - t):.2f} ms", flush=True)
        t = t2
