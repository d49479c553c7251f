"""Config-4 LSQR matvec timings: fused one-pass step vs A v + A^T u (float32 A 4194304 x 512)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_21189_b200 import rand_nla  # noqa: E402

dev = torch.device("cuda", 0)
n, d = 4194304, 512
a = torch.randn(n, d, device=dev)
v = torch.randn(d, dtype=torch.float64, device=dev)
u = torch.randn(n, dtype=torch.float64, device=dev)


def t(name, fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    print(f"{name:30s} {ms:7.3f} ms  {n * d * 4 / ms / 1e6:7.0f} GB/s of A", flush=True)


t("fused step", lambda: rand_nla._lsqr_step(a, v, 0.5, u))
t("A v", lambda: rand_nla._matvec_blocks(a, v, 1 << 16))
t("A^T u", lambda: rand_nla._rmatvec_blocks(a, u, 1 << 16))
