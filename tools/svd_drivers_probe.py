"""SVD options for the rsvd core factor B (200 x 16384 float64): cuSOLVER drivers, tall/wide, host."""
import time

import torch

dev = torch.device("cuda", 0)
k, d = 200, 16384
b = (torch.randn(k, d, device=dev, dtype=torch.float64).T * torch.arange(1, k + 1, device=dev) ** -2.0).T.contiguous()
ref = torch.linalg.svdvals(b.cpu())


def t(name, fn):
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
    s = out[1].cpu()
    print(f"{name:34s} {el * 1e3:8.2f} ms   max rel sv err {float(((s - ref) / ref).abs().max()):.2e}", flush=True)


t("gesvd wide", lambda: torch.linalg.svd(b, full_matrices=False, driver="gesvd"))
t("gesvdj wide", lambda: torch.linalg.svd(b, full_matrices=False, driver="gesvdj"))
bt = b.T.contiguous()
t("gesvd tall (B^T)", lambda: torch.linalg.svd(bt, full_matrices=False, driver="gesvd"))
t("gesvdj tall (B^T)", lambda: torch.linalg.svd(bt, full_matrices=False, driver="gesvdj"))
bc = b.cpu()
t("host (LAPACK) wide", lambda: torch.linalg.svd(bc, full_matrices=False))
