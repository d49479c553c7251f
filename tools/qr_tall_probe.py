import os, sys, time, torch
sys.path.insert(0, os.getcwd())
from paper_2508_21189_b200 import rand_nla as rn, sketch as skb
a = torch.randn(1 << 21, 512, device="cuda")
om = skb.SparseRttTM(512, 64, 1, "wht", seed=1); ps = skb.SparseUniformTM(1 << 21, 96, 8, seed=2)
y, x = rn.two_sided_sketch(a, om, ps)
print("y", y.shape, y.dtype, y.stride(), "x", x.shape, x.dtype)
y64 = y.double()
res = rn._cholqr2_qr(y64)
print("cholqr2 None?", res is None)
g = y64.T @ y64
r, info = torch.linalg.cholesky_ex(g, upper=True)
d = r.diagonal()
print("info", int(info), "diag min/max", float(d.min()), float(d.max()))
for f in (lambda: rn._qr_tall(y64), lambda: torch.linalg.qr(y64, mode="reduced")):
    torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); print(f"{(time.perf_counter()-t0)*1e3:.2f} ms")
