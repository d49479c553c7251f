"""PCIe / end-to-end pipeline probe for the config-2 host path (what bounds bench.py's e2e)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_21189_b200 import _device  # noqa: E402
from paper_2508_21189_b200.sketch import SparseRttTM  # noqa: E402

dev = torch.device("cuda", 0)
n, d = 65536, 8192
a_host = torch.randn(n, d).pin_memory()
a_dev = torch.empty(n, d, device=dev)


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


gb = a_host.numel() * 4 / 1e9
print(f"one 2 GiB H2D copy          {gb / t(lambda: a_dev.copy_(a_host, non_blocking=True)):.1f} GB/s")
rows = _device.PIPELINE_CHUNK_BYTES // (d * 4)


def chunked():
    for r0 in range(0, n, rows):
        a_dev[r0:r0 + rows].copy_(a_host[r0:r0 + rows], non_blocking=True)


print(f"{n // rows} x {rows * d * 4 >> 20} MB H2D copies    {gb / t(chunked):.1f} GB/s")
y_dev = torch.empty(n, 512, device=dev)
y_host = torch.empty(n, 512).pin_memory()
print(f"one 128 MB D2H copy         {y_dev.numel() * 4 / 1e9 / t(lambda: y_host.copy_(y_dev, non_blocking=True)):.1f} GB/s")


def both():
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        a_dev.copy_(a_host, non_blocking=True)
    with torch.cuda.stream(s2):
        for _ in range(16):
            y_host.copy_(y_dev, non_blocking=True)
    torch.cuda.synchronize()


print(f"H2D 2 GiB || D2H 16x128 MB  {t(both):.4f} s")
tm = SparseRttTM(d, 512, 1, "wht", seed=0)
tm.apply_right(a_dev[:256])
for cb in (16, 32, 48, 64, 128, 256, 32, 128):
    _device.PIPELINE_CHUNK_BYTES = cb << 20
    r = [(gb + n * 512 * 4 / 1e9) / t(lambda: tm.apply_right(a_host), reps=5) for _ in range(2)]
    print(f"apply_right(host), chunk {cb:3d} MB  " + " ".join(f"{x:.1f}" for x in r) + " GB/s")
