"""Generalized Nystrom SVD (the paper's headline application) at the DESIGN section-6 shape: wall time
and torch-profiler kernel breakdown of one warm call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_21189_b200 import rand_nla as rn  # noqa: E402
from paper_2508_21189_b200 import sketch as skb  # noqa: E402

n, d, k, p = 1 << 21, 512, 64, 96
a = torch.randn(n, d, device="cuda")
om = skb.SparseRttTM(d, k, 1, "wht", seed=1)
ps = skb.SparseUniformTM(n, p, 8, seed=2)
for _ in range(2):
    rn.gen_nystrom_svd(a, k, p, om, ps)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    rn.gen_nystrom_svd(a, k, p, om, ps)
    torch.cuda.synchronize()
    print(f"gen_nystrom_svd {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as prof:
    rn.gen_nystrom_svd(a, k, p, om, ps)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=18, max_name_column_width=60))
