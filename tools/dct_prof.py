"""Run the fused DCT-III SRTT kernel a few times at the config-2 shape (for ncu).

    python tools/dct_prof.py [float32|float64]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_21189_b200 import sketch as skb  # noqa: E402

os.environ["SKETCH_B200_DCT"] = "fft"
dev = torch.device("cuda", 0)
dt = getattr(torch, sys.argv[1] if len(sys.argv) > 1 else "float32")
a = torch.randn(65536 if dt == torch.float32 else 32768, 8192, device=dev, dtype=dt)
tm = skb.SparseRttTM(8192, 512, 1, "dct", seed=0)
for _ in range(3):
    tm.apply_right(a)
torch.cuda.synchronize()
print("ok")
