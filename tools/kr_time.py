import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2508_21189_b200 import sketch as skb
tm = skb.KhatriRaoTM(256, 2, 512, "real_rademacher", seed=0)
a = torch.randn(16384, 65536, device="cuda")
for _ in range(3): tm.apply_right(a)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(10): tm.apply_right(a)
ev[1].record(); torch.cuda.synchronize()
print(f"cfg5 {ev[0].elapsed_time(ev[1]) / 10:.4f} ms")
