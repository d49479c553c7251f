"""SVD of a 200 x 200 float64 matrix (the rsvd's small factor): cuSOLVER drivers vs host LAPACK."""
import time

import numpy as np
import torch

dev = torch.device("cuda", 0)
rng = np.random.default_rng(0)
u, _ = np.linalg.qr(rng.standard_normal((200, 200)))
v, _ = np.linalg.qr(rng.standard_normal((200, 200)))
s = np.arange(1, 201, dtype=np.float64) ** -2.0
m = (u * s) @ v.T
mt = torch.from_numpy(m).to(dev)


def t(name, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    print(f"{name:34s} {(time.perf_counter() - t0) / reps * 1e3:8.3f} ms", flush=True)
    return r


for drv in (None, "gesvd", "gesvdj", "gesvda"):
    try:
        r = t(f"torch.linalg.svd driver={drv}", lambda: torch.linalg.svd(mt, full_matrices=False, driver=drv))
        print("   sigma rel err", float(np.abs(r[1].cpu().numpy() - s).max() / s.max()),
              "min-sigma rel err", float(abs(r[1].cpu().numpy()[-1] - s[-1]) / s[-1]))
    except Exception as e:  # noqa: BLE001
        print(drv, "failed", e)
t("torch.linalg.eigh (Gram)", lambda: torch.linalg.eigh(mt.T @ mt))
t("numpy svd (host, incl. copies)", lambda: np.linalg.svd(mt.cpu().numpy(), full_matrices=False))
t("torch cpu svd (incl. copies)", lambda: torch.linalg.svd(mt.cpu(), full_matrices=False))

# SVD through the symmetric eigenproblem of the augmented [[0, M], [M^T, 0]] (eigenvalues +-sigma: no
# squaring of the condition number, unlike the Gram matrix)
aug = torch.zeros((400, 400), dtype=torch.float64, device=dev)
aug[:200, 200:] = mt
aug[200:, :200] = mt.T
ev = t("torch.linalg.eigh (augmented 400)", lambda: torch.linalg.eigh(aug))
sig = ev[0][200:].flip(0).cpu().numpy()
print("   sigma rel err", float(np.abs(sig - s).max() / s.max()), "min-sigma rel err", float(abs(sig[-1] - s[-1]) / s[-1]))
vecs = ev[1][:, 200:].flip(1) * np.sqrt(2.0)
uu, vv = vecs[:200], vecs[200:]
rec = (uu * torch.from_numpy(sig).to(dev)) @ vv.T
print("   reconstruction rel err", float((rec - mt).norm() / mt.norm()))
