"""Tall-skinny QR of a 2M x 64 float64 matrix: cuSOLVER Householder (torch.linalg.qr) vs a TSQR over
batched QRs (rank-deficient input: duplicated columns, as an SRTT sketch with replacement gives)."""
import time

import torch

dev = torch.device("cuda", 0)
n, k = 1 << 21, 64
g = torch.Generator(device=dev).manual_seed(0)
y = torch.randn(n, k, dtype=torch.float64, device=dev, generator=g)
y[:, 5] = -y[:, 9]  # a duplicated column (rank deficiency)


def t(name, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    print(f"{name:28s} {(time.perf_counter() - t0) / reps * 1e3:8.2f} ms", flush=True)
    return r


def tsqr(y, mb=2048):
    n, k = y.shape
    nb = n // mb
    yb = y[:nb * mb].reshape(nb, mb, k)
    q1, r1 = torch.linalg.qr(yb, mode="reduced")          # nb x mb x k, nb x k x k
    rs = r1.reshape(nb * k, k)
    if nb * k > 4 * mb:
        q2, r = tsqr(rs, mb)
    else:
        q2, r = torch.linalg.qr(rs, mode="reduced")
    q = torch.bmm(q1, q2.reshape(nb, k, k)).reshape(nb * mb, k)
    return q, r


for mb in (512, 1024, 2048, 4096):
    t(f"batched qr (n/{mb}, {mb}, 64)", lambda: torch.linalg.qr(y.reshape(-1, mb, k), mode="reduced"))
q0, r0 = t("torch.linalg.qr", lambda: torch.linalg.qr(y, mode="reduced"))
for mb in (1024, 2048):
    q, r = t(f"tsqr mb={mb}", lambda: tsqr(y, mb))
    eye = torch.eye(k, dtype=torch.float64, device=dev)
    print("   orth err", float((q.T @ q - eye).norm()), "recon err", float((q @ r - y).norm() / y.norm()))
