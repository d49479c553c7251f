import sys, time, torch
sys.path.insert(0, "/root/repo")
from paper_2508_21189_b200 import rand_nla
from paper_2508_21189_b200.sketch import SparseUniformTM
dev = torch.device("cuda", 0)
n, d, k = 4194304, 512, 2048
a = torch.randn(n, d, device=dev)
b = torch.randn(n, device=dev)
tm = SparseUniformTM(n, k, 8, seed=0)
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sb = tm.apply_adjoint(b); torch.cuda.synchronize(); t1 = time.perf_counter()
    x = rand_nla.sketch_and_solve(a, b, tm); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"S b {1e3*(t1-t0):.2f} ms  path {tm.adjoint_path(b[:, None])}; sketch_and_solve {1e3*(t2-t1):.2f} ms")
a_sk = tm.apply_adjoint(a)
b_sk = tm.apply_adjoint(b)
for drv in (None, "gesvd", "gesvdj"):
    for _ in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        u, s, vh = torch.linalg.svd(a_sk.double(), full_matrices=False, driver=drv)
        torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"SVD 2048x512 driver={drv}: {1e3*(t1-t0):.2f} ms")
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    q, r = torch.linalg.qr(a_sk.double())
    torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"QR 2048x512: {1e3*(t1-t0):.2f} ms")
for drv in (None, "gesvdj"):
    for _ in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        torch.linalg.svd(r, full_matrices=False, driver=drv)
        torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"SVD 512x512 driver={drv}: {1e3*(t1-t0):.2f} ms")
