"""Concurrent applies from host threads (the reference runs its trials on a thread pool).

The library caches per-kernel launch state (dynamic shared-memory limits, co-resident cluster counts,
the tensor-map encoder).  Several host threads applying operators whose kernels need different
shared-memory sizes must give exactly the results of the same calls made one at a time.
"""

from concurrent.futures import ThreadPoolExecutor

import pytest

from paper_2508_21189_b200 import sketch as skb

pytestmark = pytest.mark.gpu


def _cases(cuda):
    import torch

    g = torch.Generator(device=cuda).manual_seed(77)
    out = []
    for d, k, dt in [(512, 64, torch.float64), (2048, 256, torch.float64), (4096, 128, torch.float32)]:
        out.append((skb.SparseUniformTM(d, k, 8, seed=d), torch.randn(3000, d, device=cuda, dtype=dt, generator=g)))
    for d, k in [(1024, 64), (8192, 512)]:
        out.append((skb.SparseRttTM(d, k, 1, "wht", seed=d),
                    torch.randn(1000, d, device=cuda, dtype=torch.float32, generator=g)))
    out.append((skb.KhatriRaoTM(64, 2, 1024, "real_gaussian", seed=1),
                torch.randn(2000, 4096, device=cuda, dtype=torch.float32, generator=g)))
    out.append((skb.GaussianTM(1024, 200, seed=2), torch.randn(1500, 1024, device=cuda, dtype=torch.float32,
                                                                generator=g)))
    # float64: the DMMA engine (K5d) and the fused DCT kernel (K3b); a complex Khatri-Rao (planes)
    out.append((skb.GaussianTM(2048, 96, seed=3), torch.randn(700, 2048, device=cuda, dtype=torch.float64,
                                                               generator=g)))
    out.append((skb.SparseRttTM(4096, 64, 2, "dct", seed=4), torch.randn(900, 4096, device=cuda,
                                                                         dtype=torch.float64, generator=g)))
    out.append((skb.KhatriRaoTM(32, 2, 80, seed=5), torch.randn(300, 1024, device=cuda, dtype=torch.float64,
                                                                 generator=g)))
    return out


def test_concurrent_applies_match_sequential(cuda):
    import torch

    cases = _cases(cuda)
    ref = [tm.apply_right(a) for tm, a in cases]  # also builds every device cache
    torch.cuda.synchronize()

    def run(i):
        tm, a = cases[i % len(cases)]
        y = tm.apply_right(a)
        torch.cuda.current_stream().synchronize()
        return i % len(cases), y

    with ThreadPoolExecutor(max_workers=6) as ex:
        results = list(ex.map(run, range(6 * len(cases))))
    for i, y in results:
        assert torch.equal(y, ref[i]), i


def test_concurrent_lsqr_solves(cuda):
    """Sketch-and-precondition LSQR from several host threads at once: the device loop's pinned scalar
    buffer is per thread, so every solve stops where it stops alone and returns the same x."""
    import numpy as np
    import torch

    from paper_2508_21189_b200 import rand_nla

    rng = np.random.default_rng(3)
    probs = []
    for i, (n, d) in enumerate([(60000, 128), (80000, 256), (50000, 384)]):
        a = torch.from_numpy((rng.standard_normal((n, d)) * (1.0 + rng.pareto(1.5, size=n))[:, None])
                             .astype(np.float32)).to(cuda)
        b = (a.double() @ torch.from_numpy(rng.standard_normal(d)).to(cuda)).float()
        probs.append((a, b, skb.SparseUniformTM(n, 4 * d, 8, seed=i)))
    ref = [rand_nla.sketch_precondition_lsqr(a, b, tm, atol=1e-8, btol=0.0) for a, b, tm in probs]
    torch.cuda.synchronize()

    def run(i):
        with torch.cuda.stream(torch.cuda.Stream()):
            a, b, tm = probs[i % len(probs)]
            r = rand_nla.sketch_precondition_lsqr(a, b, tm, atol=1e-8, btol=0.0)
            torch.cuda.current_stream().synchronize()
            return i % len(probs), r

    with ThreadPoolExecutor(max_workers=3) as ex:
        results = list(ex.map(run, range(6)))
    for i, r in results:
        assert (r.itn, r.istop) == (ref[i].itn, ref[i].istop)
        x, xr = r.x.cpu().numpy(), ref[i].x.cpu().numpy()
        assert np.linalg.norm(x - xr) <= 1e-10 * np.linalg.norm(xr)
