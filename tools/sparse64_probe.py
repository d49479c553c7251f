"""float64 sparse-sign right applies: K1r (row slabs when the lists exceed shared memory) vs the round-1 K1."""
import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2508_21189_b200.sketch import SparseUniformTM
dev = torch.device("cuda", 0)
def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
import os
for (n, d, k, z) in [(65536, 16384, 200, 8), (16384, 4096, 256, 4), (65536, 16384, 256, 4)]:
    a = torch.randn(n, d, device=dev, dtype=torch.float64)
    tm = SparseUniformTM(d, k, z, seed=0)
    r = tm._ring_on(dev)
    ms = timeit(lambda: tm.apply_right(a))
    os.environ["SKETCH_B200_K1"] = "classic"
    tm2 = SparseUniformTM(d, k, z, seed=0)
    ms2 = timeit(lambda: tm2.apply_right(a))
    del os.environ["SKETCH_B200_K1"]
    gb = (a.numel() + n * k) * 8 / 1e9
    print(f"n={n} d={d} k={k} zeta={z}: slabs {len(r[0]) if r else None}  ring {ms:.3f} ms ({gb/ms*1e3:.0f} GB/s)  classic {ms2:.3f} ms ({gb/ms2*1e3:.0f} GB/s)", flush=True)
    del a
