"""The BASELINE configurations with float64 A (the reference's dtype): kernel path and time."""
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_2508_21189_b200.sketch import KhatriRaoTM, SparseRttTM, SparseUniformTM  # noqa: E402

dev = torch.device("cuda", 0)


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


cases = [("cfg2 SRTT f64", SparseRttTM(8192, 512, 1, "wht", seed=0), (65536, 8192)),
         ("cfg3 sparse f64", SparseUniformTM(16384, 200, 8, seed=0), (65536, 16384)),
         ("cfg5 KR f64", KhatriRaoTM(256, 2, 512, "real_rademacher", seed=0), (8192, 65536))]
for name, tm, shape in cases:
    a = torch.randn(*shape, device=dev, dtype=torch.float64)
    ms = timeit(lambda: tm.apply_right(a))
    gb = a.numel() * 8 / 1e9
    print(f"{name:18s} A {shape} {gb:.1f} GB: {ms:8.2f} ms  {gb / ms * 1e3:7.0f} GB/s", flush=True)
    del a
    torch.cuda.empty_cache()
