"""Gram matrix Y^T Y of a tall float64 Y (2M x 64 and 131072 x 200): one cuBLAS GEMM vs a split-K
batched form (bmm over row blocks, then a sum)."""
import time

import torch

dev = torch.device("cuda", 0)


def t(name, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    print(f"{name:36s} {(time.perf_counter() - t0) / reps * 1e3:8.3f} ms", flush=True)
    return r


for n, k in ((1 << 21, 64), (131072, 200)):
    y = torch.randn(n, k, dtype=torch.float64, device=dev)
    g0 = t(f"y.T @ y  ({n} x {k})", lambda: y.T @ y)
    for nb in (64, 256, 1024):
        if n % nb:
            continue
        yb = y.reshape(nb, n // nb, k)
        g1 = t(f"  bmm split-K nb={nb}", lambda: torch.bmm(yb.transpose(1, 2), yb).sum(0))
        print("     rel diff", float((g1 - g0).norm() / g0.norm()))
