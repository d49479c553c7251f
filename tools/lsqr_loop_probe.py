"""Config-4 LSQR loop overheads: fused steps alone, steps + device recurrences back to back (no host
sync), and the driver (device loop vs host loop)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_21189_b200 import _lib, rand_nla  # noqa: E402
from paper_2508_21189_b200.sketch import SparseUniformTM  # noqa: E402

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
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t) * 1e3


v = torch.randn(d, dtype=torch.float64, device=dev)
u = torch.randn(n, dtype=torch.float64, device=dev)
_, ts = timed(lambda: [rand_nla._lsqr_step(a, v, 1.0, u) for _ in range(35)])
print(f"35 fused steps            {ts:.2f} ms")
lib = _lib.load()
R = torch.linalg.qr(torch.randn(2048, d, dtype=torch.float64, device=dev))[1]
rinv = torch.linalg.inv(R).contiguous()
rinvt = rinv.T.contiguous()
vv, ww, xx, vn = (torch.randn(d, dtype=torch.float64, device=dev) for _ in range(4))
state = torch.tensor([1.0, 1.0, 1.0, 1.0, 0, 0, 1.0, 0.0, 0.0, 0, 0], dtype=torch.float64, device=dev)
scal = torch.zeros(8, dtype=torch.float64, device=dev)
zb = torch.rand(d + 1, dtype=torch.float64, device=dev)
st = torch.cuda.current_stream().cuda_stream


def recur():
    state[9] = 0.0
    lib.sk_lsqr_recur_f64(d, rinv.data_ptr(), rinvt.data_ptr(), zb.data_ptr(), vv.data_ptr(), ww.data_ptr(),
                          xx.data_ptr(), vn.data_ptr(), state.data_ptr(), scal.data_ptr(), st)


ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(35):
    recur()
ev[1].record()
torch.cuda.synchronize()
print(f"35 recurrences (GPU)      {ev[0].elapsed_time(ev[1]):.2f} ms (incl. the state reset copies)")
for mode in ("1", "0", "1", "0"):
    os.environ["SKETCH_B200_LSQR_DEVLOOP"] = mode
    res, tl = timed(lambda: rand_nla.sketch_precondition_lsqr(a, b, tm, atol=1e-6, btol=0.0))
    print(f"driver devloop={mode}: {tl:.2f} ms, itn {res.itn}, sketch {res.sketch_seconds * 1e3:.2f} ms")
