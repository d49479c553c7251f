"""CholeskyQR2 pieces for the config-3 rsvd sketch Y (131072 x 200, float64): Gram, Cholesky,
triangular solve vs multiplication by R^-1, and the whole orth / _svd_wide / rsvd (warm)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_21189_b200 import rand_nla  # noqa: E402
from paper_2508_21189_b200.sketch import SparseUniformTM  # noqa: E402

dev = torch.device("cuda", 0)
n, d, k = 131072, 16384, 200
a = torch.randn(n, d, device=dev)
tm = SparseUniformTM(d, k, 8, seed=0)
y = tm.apply_right(a)
rand_nla.rsvd(a, k, tm)


def t(name, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    print(f"{name:34s} {1e3 * (time.perf_counter() - t0) / reps:8.3f} ms", flush=True)
    return r


y64 = t("Y -> float64", lambda: y.double())
g = t("Gram Y^T Y (f64)", lambda: y64.T @ y64)
r = t("cholesky", lambda: torch.linalg.cholesky_ex(g, upper=True)[0])
t("solve_triangular", lambda: torch.linalg.solve_triangular(r, y64, upper=True, left=False))
ri = t("R^-1 (trtri via solve on I)", lambda: torch.linalg.solve_triangular(r, torch.eye(k, dtype=torch.float64, device=dev), upper=True))
t("Y @ R^-1 (DGEMM)", lambda: y64 @ ri)
t("isfinite(Y).all()", lambda: bool(torch.isfinite(y64).all()))
q = t("orth(Y)", lambda: rand_nla.orth(y))
b = t("B = Q^T A", lambda: rand_nla._qt_a(q, a))
t("_svd_wide(B)", lambda: rand_nla._svd_wide(b.double()))
t("rsvd total", lambda: rand_nla.rsvd(a, k, tm), reps=3)
b64 = b.double()
res = t("  _cholqr2_qr(B^T)", lambda: rand_nla._cholqr2_qr(b64.T))
print("   fast path taken:", res is not None)
if res is not None:
    rr = res[1]
    t("  svd(R) 200x200 default", lambda: torch.linalg.svd(rr, full_matrices=False))
    t("  svd(R) gesvdj", lambda: torch.linalg.svd(rr, full_matrices=False, driver="gesvdj"))
    t("  svd(R) host numpy", lambda: __import__("numpy").linalg.svd(rr.cpu().numpy()))
    t("  eigh(R^T R)", lambda: torch.linalg.eigh(rr.T @ rr))
t("  svd(B) direct", lambda: torch.linalg.svd(b64, full_matrices=False))
