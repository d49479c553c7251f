"""Config-3 rsvd: torch-profiler kernel breakdown of one warm call (top CUDA kernels by time)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_21189_b200 import rand_nla  # noqa: E402
from paper_2508_21189_b200.sketch import SparseUniformTM  # noqa: E402

dev = torch.device("cuda", 0)
n, d, k = 131072, 16384, 200
a = torch.randn(n, d, device=dev)
tm = SparseUniformTM(d, k, 8, seed=0)
for _ in range(2):
    rand_nla.rsvd(a, k, tm)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as prof:
    rand_nla.rsvd(a, k, tm)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))
