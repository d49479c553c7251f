"""Run the fused two-sided sketch a few times at the DESIGN §6 shape (for ncu)."""
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
for _ in range(3):
    rn.two_sided_sketch(a, om, ps, fused=True)
torch.cuda.synchronize()
print("ok")
