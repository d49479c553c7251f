"""Mixed-precision matvecs of the LSQR loop at the config-4 shape (4194304 x 512 float32)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_21189_b200.rand_nla import _matvec_blocks, _rmatvec_blocks  # noqa: E402

dev = torch.device("cuda", 0)
a = torch.randn(4194304, 512, device=dev)
v = torch.randn(512, dtype=torch.float64, device=dev)
u = torch.randn(4194304, dtype=torch.float64, device=dev)


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


gb = a.numel() * 4 / 1e9
for name, fn in (("A v", lambda: _matvec_blocks(a, v, 0)), ("A^T u", lambda: _rmatvec_blocks(a, u, 0))):
    ms = timed(fn)
    print(f"{name:6s} {ms:.3f} ms  {gb / ms * 1e3:.0f} GB/s of A")
