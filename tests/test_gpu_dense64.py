"""K5d — the float64 DMMA engine behind sk_kr_right_cc / sk_kr_adjoint_cc (csrc/dense64.cu).

Against a float64 reference of the same contraction (Y = scale * A * (W (x) F), the Khatri-Rao
block form; W = NULL is the dense one-block form): ragged M / N / K, K not a multiple of the 16-deep
stage, dl not a multiple of 16 (stages that straddle two leading indices P), both CTA tiles, the
transposed (adjoint) form, and a misaligned row stride that falls back to the CUDA-core kernel.
"""

import numpy as np
import pytest

from paper_2508_21189_b200 import _lib

pytestmark = pytest.mark.gpu


def _ref(a, f, w, P, dl, scale):
    import torch

    om = f.repeat(P, 1) if w is None else (w[:, None, :] * f[None, :, :]).reshape(P * dl, -1)
    return scale * (a @ om)


def _call(adjoint, x, rows, P, dl, f, w, k, scale, out):
    import torch

    lib = _lib.load()
    fn = lib.sk_kr_adjoint_cc if adjoint else lib.sk_kr_right_cc
    st = fn(_lib.SK_F64, x.data_ptr(), rows, P, dl, x.stride(0), f.data_ptr(), f.stride(0),
            None if w is None else w.data_ptr(), 0 if w is None else w.stride(0), k, scale, out.data_ptr(),
            out.stride(0), torch.cuda.current_stream().cuda_stream)
    _lib.check(st, "sk_kr_cc")


@pytest.mark.parametrize("n,P,dl,k", [(1000, 1, 777, 200), (4097, 1, 2048, 512), (300, 3, 40, 130),
                                      (129, 16, 16, 64), (777, 5, 33, 9), (64, 2, 100, 1000),
                                      (20000, 1, 512, 128)])
@pytest.mark.parametrize("kr", [False, True])
def test_gemm64_right(n, P, dl, k, kr, cuda):
    import torch

    g = torch.Generator(device=cuda).manual_seed(n + k)
    if not kr and P > 1:
        pytest.skip("dense form is one block")
    a = torch.randn(n, P * dl, device=cuda, dtype=torch.float64, generator=g)
    f = torch.randn(dl, k, device=cuda, dtype=torch.float64, generator=g)
    w = torch.randn(P, k, device=cuda, dtype=torch.float64, generator=g) if kr else None
    y = torch.empty(n, k, device=cuda, dtype=torch.float64)
    _call(False, a, n, P, dl, f, w, k, 0.75, y)
    ref = _ref(a, f, w, P, dl, 0.75)
    err = float(torch.linalg.norm(y - ref) / torch.linalg.norm(ref))
    assert err <= 1e-14, err


@pytest.mark.parametrize("m,P,dl,k", [(200, 1, 1000, 96), (1024, 4, 64, 300), (65, 3, 17, 8)])
@pytest.mark.parametrize("kr", [False, True])
def test_gemm64_adjoint(m, P, dl, k, kr, cuda):
    """X = Omega^T B with B (d x m) read in place (TA) and X written transposed (TC)."""
    import torch

    g = torch.Generator(device=cuda).manual_seed(m + k)
    if not kr and P > 1:
        pytest.skip("dense form is one block")
    b = torch.randn(P * dl, m, device=cuda, dtype=torch.float64, generator=g)
    f = torch.randn(dl, k, device=cuda, dtype=torch.float64, generator=g)
    w = torch.randn(P, k, device=cuda, dtype=torch.float64, generator=g) if kr else None
    x = torch.empty(k, m, device=cuda, dtype=torch.float64)
    _call(True, b, m, P, dl, f, w, k, -1.5, x)
    ref = _ref(b.T, f, w, P, dl, -1.5).T
    err = float(torch.linalg.norm(x - ref) / torch.linalg.norm(ref))
    assert err <= 1e-14, err


def test_gemm64_strided_and_misaligned(cuda):
    """Row strides: an even padded stride takes the DMMA engine, an odd one the CUDA-core kernel;
    both write only the n x k block of a wider output."""
    import torch

    g = torch.Generator(device=cuda).manual_seed(5)
    f = torch.randn(300, 70, device=cuda, dtype=torch.float64, generator=g)
    for lda in (302, 301):
        buf = torch.randn(500, lda, device=cuda, dtype=torch.float64, generator=g)
        a = buf[:, :300]
        out = torch.full((500, 75), 7.0, device=cuda, dtype=torch.float64)
        _call(False, a, 500, 1, 300, f, None, 70, 1.0, out)
        ref = a @ f
        assert float(torch.linalg.norm(out[:, :70] - ref) / torch.linalg.norm(ref)) <= 1e-14
        assert bool((out[:, 70:] == 7.0).all())


def test_gemm64_null_w_needs_one_block(cuda):
    import torch

    a = torch.zeros(100, 64, device=cuda, dtype=torch.float64)
    f = torch.zeros(32, 8, device=cuda, dtype=torch.float64)
    y = torch.empty(100, 8, device=cuda, dtype=torch.float64)
    with pytest.raises(ValueError):
        _call(False, a, 100, 2, 32, f, None, 8, 1.0, y)
