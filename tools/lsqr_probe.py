"""Config-4 LSQR time breakdown: whole driver vs its fused steps and the QR of SA."""
import sys, time, torch, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2508_21189_b200 import rand_nla
from paper_2508_21189_b200.sketch import SparseUniformTM
dev = torch.device("cuda", 0)
n, d, k = 4194304, 512, 2048
g = torch.Generator(device=dev).manual_seed(0)
gen = np.random.default_rng(0)
w = torch.from_numpy(1.0 + gen.pareto(1.5, size=n).astype(np.float32)).to(dev)
a = torch.randn(n, d, device=dev, dtype=torch.float32, generator=g) * w[:, None]
x0 = torch.randn(d, device=dev, dtype=torch.float64, generator=g)
b = (a.double() @ x0 + 1e-3 * torch.randn(n, device=dev, dtype=torch.float64, generator=g)).float()
tm = SparseUniformTM(n, k, 8, seed=0)
tm.apply_adjoint(a)
def timed(fn):
    torch.cuda.synchronize(); t = time.perf_counter(); r = fn(); torch.cuda.synchronize(); return r, (time.perf_counter() - t) * 1e3
res, t1 = timed(lambda: rand_nla.sketch_precondition_lsqr(a, b, tm, atol=1e-6, btol=0.0))
res, t2 = timed(lambda: rand_nla.sketch_precondition_lsqr(a, b, tm, atol=1e-6, btol=0.0))
print("lsqr", t1, t2, "itn", res.itn, "t_sketch", res.t_sketch * 1e3 if hasattr(res, "t_sketch") else None)
v = torch.randn(d, dtype=torch.float64, device=dev); u = torch.randn(n, dtype=torch.float64, device=dev)
_, ts = timed(lambda: [rand_nla._lsqr_step(a, v, 0.5, u) for _ in range(35)])
print("35 fused steps", ts)
sa = tm.apply_adjoint(torch.cat([a, b[:, None]], 1)) if False else None
_, tq = timed(lambda: torch.linalg.qr(torch.randn(2048, 512, dtype=torch.float64, device=dev), mode="reduced"))
print("qr 2048x512", tq)
