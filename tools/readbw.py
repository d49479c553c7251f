"""Read-bandwidth ceiling for the cfg2 shape: torch reductions over a 2 GiB f32 matrix (CUDA events)."""
import torch

a = torch.randn(65536, 8192, device="cuda")
out = torch.empty(65536, device="cuda")
for name, fn in [("sum(dim=1)", lambda: torch.sum(a, dim=1, out=out)), ("amax", lambda: a.amax()),
                 ("sum()", lambda: a.sum())]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    print(f"{name:12s} {ms:.4f} ms  {a.numel() * 4 / ms / 1e6:.0f} GB/s")
