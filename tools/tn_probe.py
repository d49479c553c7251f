"""sk_dense_tn_tc at the config-3 rsvd shape: A 131072 x 16384 f32, Q 131072 x 200."""
import sys
import torch
sys.path.insert(0, "/root/repo")
from paper_2508_21189_b200.sketch.tensorcore import dense_tn_tc  # noqa: E402
dev = torch.device("cuda", 0)
a = torch.randn(131072, 16384, device=dev)
q = torch.randn(131072, 200, device=dev, dtype=torch.float64)
dense_tn_tc(a, q)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(5):
    dense_tn_tc(a, q)
e1.record()
torch.cuda.synchronize()
print("TN ms", e0.elapsed_time(e1) / 5)
