"""The BASELINE configurations with float64 A (the reference's dtype): kernel path and time.

    python tools/f64_probe.py

Dense-shaped float64 applies (Khatri-Rao, Gaussian) run K4c on the CUDA cores; their FP64 rate is
printed next to cuBLAS DGEMM (torch.matmul) on the same shape as the yardstick.
"""
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_2508_21189_b200.sketch import GaussianTM, KhatriRaoTM, SparseRttTM, SparseUniformTM  # noqa: E402

dev = torch.device("cuda", 0)


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


cases = [("cfg2 SRTT f64", SparseRttTM(8192, 512, 1, "wht", seed=0), (65536, 8192), 0),
         ("cfg3 sparse f64", SparseUniformTM(16384, 200, 8, seed=0), (65536, 16384), 0),
         ("cfg5 KR f64", KhatriRaoTM(256, 2, 512, "real_rademacher", seed=0), (8192, 65536), 512),
         ("gauss f64", GaussianTM(16384, 200, seed=0), (32768, 16384), 200),
         ("gauss f64 k512", GaussianTM(4096, 512, seed=0), (65536, 4096), 512)]
only = sys.argv[1:]
if not only or any("adj" in o for o in only):
    tm = SparseUniformTM(1 << 20, 2048, 8, seed=0)
    a = torch.randn(1 << 20, 512, device=dev, dtype=torch.float64)
    ms = timeit(lambda: tm.apply_adjoint(a))
    gb = (a.numel() + 2048 * 512) * 8 / 1e9
    print(f"{'cfg4 adj f64':18s} A (1048576, 512) {a.numel() * 8 / 1e9:.1f} GB: {ms:8.2f} ms  {gb / ms * 1e3:7.0f} GB/s",
          flush=True)
    del a
    torch.cuda.empty_cache()
if not only or any("complex" in o for o in only):
    from paper_2508_21189_b200.sketch.kron import _device_contract_rows

    tm = KhatriRaoTM(256, 2, 512, seed=0)  # the reference's default base: complex_spherical
    for cplx in (False, True):
        a = torch.randn(4096, 65536, device=dev, dtype=torch.float64)
        if cplx:
            a = torch.complex(a, torch.randn_like(a))
        ms = timeit(lambda: tm.apply_right(a))
        f = tm._factors_on(dev, torch.complex128)
        ac = a.to(torch.complex128)
        ms_t = timeit(lambda: _device_contract_rows(f, ac, conjugate=False))
        print(f"{'KR complex':18s} A (4096, 65536) {'complex128' if cplx else 'float64'}: {ms:8.2f} ms (K5d planes)"
              f"  torch mode contraction {ms_t:8.2f} ms", flush=True)
        del a, ac
        torch.cuda.empty_cache()
for name, tm, shape, kflops in cases:
    if only and not any(o in name for o in only):
        continue
    a = torch.randn(*shape, device=dev, dtype=torch.float64)
    ms = timeit(lambda: tm.apply_right(a))
    gb = a.numel() * 8 / 1e9
    line = f"{name:18s} A {shape} {gb:.1f} GB: {ms:8.2f} ms  {gb / ms * 1e3:7.0f} GB/s"
    if kflops:
        fl = 2.0 * shape[0] * shape[1] * kflops
        om = torch.randn(shape[1], kflops, device=dev, dtype=torch.float64)
        ms_blas = timeit(lambda: a @ om)
        line += f"  {fl / ms / 1e9:6.1f} TFLOP/s   cuBLAS DGEMM same shape {ms_blas:8.2f} ms {fl / ms_blas / 1e9:6.1f} TFLOP/s"
        del om
    print(line, flush=True)
    del a
    torch.cuda.empty_cache()
