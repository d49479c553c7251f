"""PCIe H2D: one stream vs two streams (two copy engines) over a pinned 2 GiB buffer."""
import time

import torch

dev = torch.device("cuda", 0)
n, d = 65536, 8192
h = torch.randn(n, d).pin_memory()
g = torch.empty(n, d, device=dev)
ss = [torch.cuda.Stream() for _ in range(4)]


def run(nstreams, chunk_rows=4096):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, r0 in enumerate(range(0, n, chunk_rows)):
        with torch.cuda.stream(ss[i % nstreams]):
            g[r0:r0 + chunk_rows].copy_(h[r0:r0 + chunk_rows], non_blocking=True)
    torch.cuda.synchronize()
    return h.numel() * 4 / (time.perf_counter() - t0) / 1e9


for ns in (1, 2, 4, 1, 2):
    print(f"{ns} stream(s): " + " ".join(f"{run(ns):.1f}" for _ in range(3)) + " GB/s", flush=True)
