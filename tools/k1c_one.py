import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2508_21189_b200 import sketch as skb
tm = skb.SparseUniformTM(4096, 256, 4, seed=0)
a = torch.randn(16384, 4096, dtype=torch.float64, device="cuda")
for _ in range(3): tm.apply_right(a)
torch.cuda.synchronize()
