import os, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2508_21189_b200.sketch import SparseUniformTM
dev = torch.device("cuda", 0)
n, d, k = 4194304, 512, 2048
dt = torch.float64 if os.environ.get("ADJ_F64") == "1" else torch.float32
a = torch.randn(n, d, device=dev, dtype=dt)
tm = SparseUniformTM(n, k, 8, seed=0)
print("path", tm.adjoint_path(a))
y = tm.apply_adjoint(a); torch.cuda.synchronize()
for rep in range(2):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5): y = tm.apply_adjoint(a)
    e1.record(); torch.cuda.synchronize()
    print("SA ms", e0.elapsed_time(e1) / 5)
