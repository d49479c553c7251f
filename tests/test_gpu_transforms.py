"""SRTT with the DCT transform (the reference's real-field default), SRTT and Khatri-Rao adjoints.

DCT rows run as DCT-III through the device FFT (O(d log d)); adjoints of the real SRTT / KR
operators run the row kernels on B^T (Omega^T B = (B^T Omega)^T). Oracles: oracle/ restatement
(src/sketch/rtt.py:129-154, khatri_rao.py:147-164) and the reference's materialised matrix.
"""

import numpy as np
import pytest

import oracle as orc
from _cases import rel_err
from paper_2508_21189_b200 import sketch as skb

pytestmark = pytest.mark.gpu

TOL = {np.float64: 1e-12, np.float32: 1e-5}


def _t(a, dev, dt):
    import torch

    return torch.as_tensor(np.asarray(a, dtype=dt)).to(dev)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("d,k,xi,n", [(8192, 512, 1, 40), (1000, 64, 3, 9), (4097, 100, 10, 5), (2, 1, 1, 3)])
def test_srtt_dct_right_vs_oracle(d, k, xi, n, dt, cuda):
    rng = np.random.default_rng(d + xi)
    a = (rng.standard_normal((n, d)) / np.arange(1, d + 1)).astype(dt)
    tm = skb.SparseRttTM(d, k, xi, seed=5)  # real field -> DCT (reference default)
    assert tm.transform == "dct"
    dv, samp = orc.srtt_parts(d, k, xi, 5)
    ref = orc.srtt_right(dv, samp, a, "dct")
    assert rel_err(tm.apply_right(_t(a, cuda, dt)).cpu().numpy(), ref) <= TOL[dt]
    if dt == np.float64:  # NumPy in / NumPy out, as the reference
        assert rel_err(tm.apply_right(a), ref) <= 1e-12


@pytest.mark.parametrize("transform", ["wht", "dct"])
@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_srtt_adjoint(transform, dt, cuda):
    d, k, xi, m = 2048, 96, 2, 7
    tm = skb.SparseRttTM(d, k, xi, transform, seed=3)
    b = np.random.default_rng(1).standard_normal((d, m)).astype(dt)
    ref = tm.materialize().T @ b.astype(np.float64)
    assert rel_err(tm.apply_adjoint(_t(b, cuda, dt)).cpu().numpy(), ref) <= TOL[dt]
    v = tm.apply_adjoint(b[:, 0].astype(np.float64))
    assert v.shape == (k,) and rel_err(v, ref[:, 0]) <= 1e-12


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_kr_adjoint(dt, cuda):
    tm = skb.KhatriRaoTM(32, 2, 200, "real_rademacher", seed=4)
    b = np.random.default_rng(2).standard_normal((tm.d, 11)).astype(dt)
    ref = tm.materialize().T @ b.astype(np.float64)
    assert rel_err(tm.apply_adjoint(_t(b, cuda, dt)).cpu().numpy(), ref) <= TOL[dt]


def test_dct3_rows_matches_scipy(cuda):
    import scipy.fft
    import torch

    for n in (1, 5, 64, 3000):
        x = np.random.default_rng(n).standard_normal((4, n))
        got = skb.dct3_rows(torch.as_tensor(x, device=cuda)).cpu().numpy()
        assert rel_err(got, scipy.fft.dct(x, type=3, norm="ortho", axis=1)) <= 1e-14


@pytest.mark.parametrize("d", [32, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384])
@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_srtt_dct_fused_kernel_every_pass_pattern(d, dt, cuda, monkeypatch):
    """K3b (sk_srtt_dct_right) for every power-of-two length it takes: log2(d/2) % 4 = 0..3 selects the
    radix-32/4/8 extra pass; float64 (the reference's dtype) at 1e-12, float32 at 1e-5; ragged k, xi > 1."""
    import torch

    if dt == "float64" and d > 8192:
        pytest.skip("float64 rows of d > 8192 take the cuFFT form")
    k, xi = 37, 3
    monkeypatch.setenv("SKETCH_B200_DCT", "fft")
    tm = skb.SparseRttTM(d, k, xi, "dct", seed=d)
    tdt = getattr(torch, dt)
    assert tm.dct_path(tdt) == "fft"
    rng = np.random.default_rng(d)
    a = rng.standard_normal((301, d)).astype(dt)
    y = tm.apply_right(torch.from_numpy(a).to(cuda)).double().cpu().numpy()
    dv, samp = orc.srtt_parts(d, k, xi, d)
    ref = orc.srtt_right(dv, samp, a, "dct")
    assert rel_err(y, ref) <= (1e-12 if dt == "float64" else 1e-5)


@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_srtt_dct_kernel_general_weights(dt, cuda):
    """K3b with weights that are not +-1 / s (the kernel's table path) against the same kernel on the
    +-1 path with the extra factors folded into A: sk_srtt_dct_right(A, w * v) == sk_srtt_dct_right(A * v, w)."""
    import torch

    from paper_2508_21189_b200 import _lib

    d, k, xi = 2048, 40, 2
    tm = skb.SparseRttTM(d, k, xi, "dct", seed=3)
    tdt = getattr(torch, dt)
    w, samp, scale = tm._dct_fft_tables(cuda, tdt)
    g = torch.Generator(device=cuda).manual_seed(2)
    a = torch.randn(300, d, device=cuda, dtype=tdt, generator=g)
    v = 0.5 + torch.rand(d, device=cuda, dtype=tdt, generator=g)
    lib = _lib.load()
    code = _lib.SK_F64 if dt == "float64" else _lib.SK_F32
    outs = []
    for x, ww in ((a, (w * v).contiguous()), ((a * v).contiguous(), w)):
        y = torch.empty(300, k, device=cuda, dtype=tdt)
        _lib.check(lib.sk_srtt_dct_right(code, x.data_ptr(), 300, d, x.stride(0), ww.data_ptr(), samp.data_ptr(), xi,
                                         k, scale, y.data_ptr(), y.stride(0), torch.cuda.current_stream().cuda_stream),
                   "sk_srtt_dct_right")
        outs.append(y.double())
    err = float(torch.linalg.norm(outs[0] - outs[1]) / torch.linalg.norm(outs[1]))
    assert err <= (1e-13 if dt == "float64" else 1e-6), err


def test_srtt_dct_paths_agree_config2_shape(cuda, monkeypatch):
    """Config-2 shape with the DCT transform (the reference default): the fused FFT kernel, the
    tensor-core form and the cuFFT form agree; a 64-row slab against the oracle."""
    import torch

    tm = skb.SparseRttTM(8192, 512, 1, "dct", seed=0)
    g = torch.Generator(device=cuda).manual_seed(5)
    a = torch.randn(4096, 8192, device=cuda, generator=g)
    outs = {}
    for path in ("fft", "tc", "cufft"):
        monkeypatch.setenv("SKETCH_B200_DCT", path)
        assert tm.dct_path(torch.float32) == path
        outs[path] = tm.apply_right(a).double()
    for path in ("tc", "cufft"):
        assert float((outs["fft"] - outs[path]).norm() / outs[path].norm()) <= 1e-5
    dv, samp = orc.srtt_parts(8192, 512, 1, 0)
    ref = orc.srtt_right(dv, samp, a[:64].cpu().numpy(), "dct")
    assert rel_err(outs["fft"][:64].cpu().numpy(), ref) <= 1e-5


@pytest.mark.parametrize("k,xi,n", [(512, 1, 301), (200, 3, 17), (1000, 2, 1)])
def test_srtt_float64_wide_d8192(k, xi, n, cuda, monkeypatch):
    """float64 SRTT-WHT at d = 8192 on the wide kernel (two register phases, bit 7 folded into the
    gather) against the oracle and against the 3-phase kernel (SKETCH_B200_SRTT64=3)."""
    import numpy as np
    import torch

    import oracle as orc
    from paper_2508_21189_b200 import sketch as skb

    rng = np.random.default_rng(k + xi)
    a = rng.standard_normal((n, 8192)) / np.arange(1, 8193)
    tm = skb.SparseRttTM(8192, k, xi, "wht", seed=7)
    at = torch.from_numpy(a).to(cuda)
    y = tm.apply_right(at).cpu().numpy()
    dv, samp = orc.srtt_parts(8192, k, xi, 7)
    ref = orc.srtt_right(dv, samp, a, "wht")
    assert np.linalg.norm(y - ref) <= 1e-12 * np.linalg.norm(ref)
    monkeypatch.setenv("SKETCH_B200_SRTT64", "3")
    y3 = tm.apply_right(at).cpu().numpy()
    assert np.linalg.norm(y - y3) <= 1e-14 * np.linalg.norm(y3)
