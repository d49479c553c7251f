"""Time the fused one-pass two-sided sketch against two separate passes (generalized-Nystrom sketch stage)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_21189_b200 import rand_nla as rn  # noqa: E402
from paper_2508_21189_b200 import sketch as skb  # noqa: E402

dev = torch.device("cuda", 0)
n, d, k, p = 1 << 21, 512, 64, 96
a = torch.randn(n, d, device=dev)
om = skb.SparseRttTM(d, k, 1, "wht", seed=1)
ps = skb.SparseUniformTM(n, p, 8, seed=2)


def timed(fn, reps=5):
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
t_right = timed(lambda: om.apply_right(a))
t_adj = timed(lambda: ps.apply_adjoint(a))
print(f"A {n}x{d} f32 ({gb:.2f} GB): right {t_right:.3f} ms, adjoint {t_adj:.3f} ms, "
      f"two passes {t_right + t_adj:.3f} ms")
t = timed(lambda: rn.two_sided_sketch(a, om, ps, fused=True))
print(f"  fused one-pass kernel (sk_two_sided_sketch): {t:.3f} ms ({gb / t:.1f} TB/s of A, "
      f"{(t_right + t_adj) / t:.1f}x the two passes)")

for dbg in os.environ.get("TS_DBG", "").split(","):
    if dbg:
        os.environ["SKETCH_B200_TS_DBG"] = dbg
        t = timed(lambda: rn.two_sided_sketch(a, om, ps, fused=True))
        print(f"  SKETCH_B200_TS_DBG={dbg}: {t:.3f} ms")
        os.environ["SKETCH_B200_TS_DBG"] = "0"
