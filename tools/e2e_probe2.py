import sys, time, torch
sys.path.insert(0, "/root/repo")
from paper_2508_21189_b200 import _device
from paper_2508_21189_b200.sketch import SparseRttTM
dev = torch.device("cuda", 0)
tm = SparseRttTM(8192, 512, 1, "wht", seed=0)
a = torch.randn(65536, 8192, device=dev)
a_host = torch.empty(a.shape, dtype=a.dtype, pin_memory=True)
a_host.copy_(a)
orig_empty = torch.empty
def timed_empty(*args, **kw):
    t0 = time.perf_counter(); r = orig_empty(*args, **kw); dt = time.perf_counter() - t0
    if dt > 0.005: print(f"   slow torch.empty {args} {kw.get('pin_memory')} {dt*1e3:.1f} ms", flush=True)
    return r
torch.empty = timed_empty
for i in range(12):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    y = tm.apply_right(a_host)
    t1 = time.perf_counter()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"step {i}: call {1e3*(t1-t0):7.2f} ms, sync {1e3*(t2-t1):7.2f} ms", flush=True)
