"""Timing of the rsvd core SVD (B = Q^T A, 200 x 16384 float64) through the cuSOLVER drivers."""
import time

import numpy as np
import torch

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
k, d = 200, 16384
u0, _ = torch.linalg.qr(torch.randn(d, k, dtype=torch.float64, device=dev, generator=g))
b = (torch.diag(torch.arange(1, k + 1, dtype=torch.float64, device=dev) ** -2.0) @ u0.T).contiguous()
ref = torch.linalg.svdvals(b.cpu())


def t(name, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / reps * 1e3
    s = out[1].cpu()
    print(f"{name:34s} {ms:7.2f} ms   max rel sigma err {float(((s - ref).abs() / ref).max()):.2e}")


t("svd(B) default", lambda: torch.linalg.svd(b, full_matrices=False))
for drv in ("gesvd", "gesvdj", "gesvda"):
    try:
        t(f"svd(B) {drv}", lambda: torch.linalg.svd(b, full_matrices=False, driver=drv))
    except Exception as e:
        print(drv, "failed", e)


def qr_svd(drv=None):
    q, r = torch.linalg.qr(b.T)
    ur, s, vrh = torch.linalg.svd(r, full_matrices=False, driver=drv)
    return vrh.T, s, (q @ ur).T


def chol2_svd(drv=None):
    x = b.T
    rr = None
    for _ in range(2):
        gm = x.T @ x
        r = torch.linalg.cholesky(gm, upper=True)
        x = torch.linalg.solve_triangular(r, x, upper=True, left=False)
        rr = r if rr is None else r @ rr
    ur, s, vrh = torch.linalg.svd(rr, full_matrices=False, driver=drv)
    return vrh.T, s, (x @ ur).T


for drv in (None, "gesvdj", "gesvd"):
    t(f"qr + svd(R) {drv}", lambda: qr_svd(drv))
    t(f"cholqr2 + svd(R) {drv}", lambda: chol2_svd(drv))


def host_r(fn):
    def go():
        x = b.T
        q, r = torch.linalg.qr(x)
        ur, s, vrh = np.linalg.svd(r.cpu().numpy())
        ur = torch.from_numpy(ur).to(dev)
        return torch.from_numpy(vrh.T).to(dev), torch.from_numpy(s), (q @ ur).T
    return go


t("qr + host svd(R)", host_r(None))
