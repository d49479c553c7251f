"""One config-5 Khatri-Rao apply after warm-up (for ncu -k regex:dense_tc_pair -s 3 -c 1)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_21189_b200 import sketch as skb  # noqa: E402

tm = skb.KhatriRaoTM(256, 2, 512, "real_rademacher", seed=0)
a = torch.randn(16384, 65536, device="cuda")
for _ in range(4):
    tm.apply_right(a)
torch.cuda.synchronize()
