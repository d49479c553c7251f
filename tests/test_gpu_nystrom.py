"""Nystrom drivers (reference rand_nla.py:152-275) against outputs of the real reference
(tests/golden/make_golden.py), and the one-pass two-sided sketch against separate applies."""

import numpy as np
import pytest

from _cases import nystrom_inputs, rel_err
from paper_2508_21189_b200 import rand_nla as rn
from paper_2508_21189_b200 import sketch as skb

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,om,ps", [
    ("gn_su", lambda: skb.SparseUniformTM(300, 20, 4, seed=21), lambda: skb.SparseUniformTM(1024, 30, 4, seed=22)),
    ("gn_rtt", lambda: skb.SparseRttTM(300, 20, 2, "dct", seed=23), lambda: skb.SparseUniformTM(1024, 30, 8, seed=24)),
])
def test_gen_nystrom_golden(name, om, ps, golden, cuda):
    a, _, _, probe = nystrom_inputs()
    fo = rn.gen_nystrom_outer(a, 20, 30, om(), ps())
    assert isinstance(fo.f, np.ndarray) and fo.f.shape == (1024, fo.rank) and fo.g.shape == (300, fo.rank)
    assert rel_err(fo.matrix() @ probe[:300], golden[f"{name}_outer_probe"]) <= 1e-9
    fs = rn.gen_nystrom_svd(a, 20, 30, om(), ps())
    assert rel_err(fs.sigma, golden[f"{name}_svd_sigma"]) <= 1e-9
    assert rel_err((fs.u * fs.sigma) @ (fs.v.T @ probe[:300]), golden[f"{name}_svd_probe"]) <= 1e-9


def test_gen_nystrom_wide_golden(golden, cuda):
    _, a, _, probe = nystrom_inputs()
    fo = rn.gen_nystrom_outer(a, 20, 30, skb.SparseUniformTM(256, 20, 4, seed=25), skb.SparseUniformTM(300, 30, 4, seed=26))
    assert rel_err(fo.matrix() @ probe[:256], golden["gn_wide_outer_probe"]) <= 1e-9
    fs = rn.gen_nystrom_svd(a, 20, 30, skb.SparseUniformTM(256, 20, 4, seed=25), skb.SparseUniformTM(300, 30, 4, seed=26))
    assert rel_err((fs.u * fs.sigma) @ (fs.v.T @ probe[:256]), golden["gn_wide_outer_probe"]) <= 1e-9


@pytest.mark.parametrize("name,tm", [("nys_su", lambda: skb.SparseUniformTM(512, 30, 4, seed=27)),
                                     ("nys_gauss", lambda: skb.GaussianTM(512, 30, seed=28))])
def test_nystrom_psd_golden(name, tm, golden, cuda):
    _, _, apsd, probe = nystrom_inputs()
    fe = rn.nystrom_psd(apsd, 30, tm())
    assert rel_err(fe.lam, golden[f"{name}_lam"]) <= 1e-9
    assert rel_err(fe.matrix() @ probe, golden[f"{name}_probe"]) <= 1e-9


def test_validation_errors(cuda):
    a, _, apsd, _ = nystrom_inputs()
    with pytest.raises(ValueError, match="k <= p"):
        rn.gen_nystrom_outer(a, 31, 30, skb.SparseUniformTM(300, 31, 4), skb.SparseUniformTM(1024, 30, 4))
    with pytest.raises(ValueError, match="square"):
        rn.nystrom_psd(a, 5, skb.SparseUniformTM(300, 5, 4))
    with pytest.raises(ValueError, match="psd"):
        rn.nystrom_psd(-apsd, 30, skb.SparseUniformTM(512, 30, 4))


@pytest.mark.parametrize("n,d,k,p,omega", [(20000, 512, 64, 96, "srtt"), (1000, 100, 17, 128, "gauss"),
                                           (777, 300, 128, 5, "sparse"), (300001, 256, 32, 64, "srtt"),
                                           (129, 64, 1, 1, "sparse"), (5000, 448, 40, 96, "gauss"),
                                           (3000, 1024, 100, 33, "sparse")])
def test_two_sided_sketch_fused(n, d, k, p, omega, cuda):
    """The one-pass fused kernel (sk_two_sided_sketch) against the two separate applies and the oracle:
    ragged M-tiles and column groups (d = 100, 300, 448: an odd k-block count next to paired ones), one,
    two or four column groups, split Omega (Gaussian), 3-stage rings (k = 100, 128)."""
    import torch

    import oracle as orc

    g = torch.Generator(device=cuda).manual_seed(n)
    a = torch.randn(n, d, device=cuda, generator=g)
    om = {"srtt": lambda: skb.SparseRttTM(d, k, 1, "wht", seed=1), "gauss": lambda: skb.GaussianTM(d, k, seed=3),
          "sparse": lambda: skb.SparseUniformTM(d, k, min(4, k), seed=5)}[omega]()
    ps = skb.SparseUniformTM(n, p, min(8, p), seed=2)
    assert rn._psi_rows(ps) is not None
    y, x = rn.two_sided_sketch(a, om, ps, fused=True)
    assert y.shape == (n, k) and x.shape == (d, p)
    a64 = a.double().cpu().numpy()
    y_ref = a64 @ om.materialize()
    x_ref = orc.csr_adjoint(orc.sparse_uniform_csr(n, p, min(8, p), 2), a64).T
    assert rel_err(y.double().cpu().numpy(), y_ref) <= 1e-5
    assert rel_err(x.double().cpu().numpy(), x_ref) <= 1e-5
    y2, x2 = rn.two_sided_sketch(a, om, ps, fused=False)
    assert rel_err(y.double().cpu().numpy(), y2.double().cpu().numpy()) <= 1e-5


def test_gen_nystrom_float32_device_end_to_end(cuda):
    import torch

    n, d, k, p = 20000, 512, 64, 96
    a = torch.randn(n, d, device=cuda)
    om = skb.SparseRttTM(d, k, 1, "wht", seed=1)
    ps = skb.SparseUniformTM(n, p, 8, seed=2)
    fo = rn.gen_nystrom_outer(a, k, p, om, ps)  # float32 device path end to end (fused sketch)
    assert fo.f.shape[0] == n and fo.g.shape[0] == d
