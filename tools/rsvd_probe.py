"""Config-3 rsvd stage timings (warm): sketch, orth (QR of Y in f64), B = Q^T A, SVD(B), Q U."""
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
rand_nla.rsvd(a, k, tm)
torch.cuda.synchronize()


def t(name, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print(f"{name:28s} {1e3 * (time.perf_counter() - t0):8.2f} ms", flush=True)
    return r


for _ in range(2):
    y = t("sketch", lambda: tm.apply_right(a))
    q = t("orth (f64 QR of Y)", lambda: rand_nla.orth(y))
    with rand_nla._no_tf32():
        b = t("B = Q^T A (fp32 cuBLAS)", lambda: (q.to(a.dtype).T @ a).to(q.dtype))
    b2 = t("B = Q^T A (sk_dense_tn_tc)", lambda: rand_nla._qt_a(q, a))
    print("   rel diff", float((b2 - b).norm() / b.norm()))
    usv = t("SVD(B) f64 direct", lambda: torch.linalg.svd(b.double(), full_matrices=False))
    t("SVD(B) f64 gesvdj", lambda: torch.linalg.svd(b.double(), full_matrices=False, driver="gesvdj"))
    bt = b.double().T.contiguous()
    t("  QR(B^T) 16384x200", lambda: torch.linalg.qr(bt, mode="reduced"))
    rr = torch.randn(200, 200, device=dev, dtype=torch.float64)
    t("  SVD 200x200", lambda: torch.linalg.svd(rr, full_matrices=False))
    t("Q U", lambda: q @ usv[0].to(q.dtype))
    t("rsvd total", lambda: rand_nla.rsvd(a, k, tm))
