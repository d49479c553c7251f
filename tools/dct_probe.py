"""SparseRttTM with the DCT transform (the reference's real-field default) at the config-2 shape:
the fused K3b row kernel against the tensor-core and cuFFT forms, float32 and float64."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_21189_b200 import sketch as skb  # noqa: E402

dev = torch.device("cuda", 0)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


for dt, n in ((torch.float32, 65536), (torch.float64, 32768)):
    a = torch.randn(n, 8192, device=dev, dtype=dt)
    gb = (a.numel() + n * 512) * a.element_size() / 1e9
    tm = skb.SparseRttTM(8192, 512, 1, "wht", seed=0)
    ms = timed(lambda: tm.apply_right(a))
    print(f"{dt} n={n} wht: {ms:.3f} ms  {gb / ms * 1e3:.0f} GB/s")
    tm = skb.SparseRttTM(8192, 512, 1, "dct", seed=0)
    for path in ("fft", "tc", "cufft"):
        os.environ["SKETCH_B200_DCT"] = path
        if tm.dct_path(dt) != path:
            continue
        ms = timed(lambda: tm.apply_right(a))
        print(f"{dt} n={n} dct[{path}]: {ms:.3f} ms  {gb / ms * 1e3:.0f} GB/s")
    os.environ.pop("SKETCH_B200_DCT")
    del a
    torch.cuda.empty_cache()
