"""Config-4 S*A (K2g) timing: A 4194304 x 512 f32, k = 2048, zeta = 8."""
import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2508_21189_b200.sketch import SparseUniformTM
dev = torch.device("cuda", 0)
n, d, k = 4194304, 512, 2048
g = torch.Generator(device=dev).manual_seed(41)
a = torch.randn(n, d, device=dev, generator=g)
tm = SparseUniformTM(n, k, 8, seed=0)
y = tm.apply_adjoint(a)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
for _ in range(2):
    s.record()
    for _ in range(10): tm.apply_adjoint(a)
    e.record(); torch.cuda.synchronize()
    print(f"cfg4 S*A: {s.elapsed_time(e)/10:.3f} ms", flush=True)
torch.save(y.cpu(), "/tmp/sa_new.pt")
