import sys, torch, time
sys.path.insert(0, "/root/repo")
from paper_2508_21189_b200.sketch import SparseUniformTM
dev = torch.device("cuda", 0)
n, d, k = 4194304, 512, 2048
a = torch.randn(n, d, device=dev)
tm = SparseUniformTM(n, k, 8, seed=0)
y = tm.apply_adjoint(a); torch.cuda.synchronize()
for rep in range(2):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): y = tm.apply_adjoint(a)
    e1.record(); torch.cuda.synchronize()
    print("SA ms", e0.elapsed_time(e1) / 10)
