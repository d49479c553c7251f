"""GPU parity of the tcgen05 dense engine (K-TC) and the families routed through it.

Tolerance: float32 inputs, relative Frobenius error <= 1e-5 against the float64 oracle (the
A hi+lo bf16 split alone contributes ~2e-6).
"""

import numpy as np
import pytest

import oracle as orc
from _cases import rel_err
from paper_2508_21189_b200 import sketch as skb
from paper_2508_21189_b200.sketch.tensorcore import bt_from_dense, bt_from_triplets, dense_right_tc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,d,k", [(1, 64, 16), (127, 100, 1), (128, 1024, 200), (300, 512, 256), (257, 256, 300),
                                   (64, 4096, 512), (130, 192, 700), (1000, 64, 48)])
def test_dense_tc_exact_b(n, d, k, cuda):
    import torch

    rng = np.random.default_rng(n + d + k)
    a = rng.standard_normal((n, d)).astype(np.float32)
    b = np.where(rng.random((d, k)) < 0.5, -1.0, 1.0) * (rng.random((d, k)) < 0.3)
    rows, cols = np.nonzero(b)
    hi, lo = bt_from_triplets(rows, cols, b[rows, cols] < 0, d, k, cuda)
    assert lo is None
    y = dense_right_tc(torch.from_numpy(a).to(cuda), hi, lo, k, 0.5).cpu().numpy()
    ref = 0.5 * (a.astype(np.float64) @ b)
    assert rel_err(y, ref) <= 1e-5


@pytest.mark.parametrize("n,d,k", [(200, 256, 64), (129, 1024, 512)])
def test_dense_tc_split_b(n, d, k, cuda):
    import torch

    rng = np.random.default_rng(7)
    a = rng.standard_normal((n, d)).astype(np.float32)
    b = rng.standard_normal((d, k)) / np.sqrt(k)
    hi, lo = bt_from_dense(b, cuda)
    assert lo is not None
    y = dense_right_tc(torch.from_numpy(a).to(cuda), hi, lo, k, 1.0).cpu().numpy()
    assert rel_err(y, a.astype(np.float64) @ b) <= 1e-5


def test_sparse_tc_and_gather_agree_config3_slab(cuda, monkeypatch):
    import torch

    tm = skb.SparseUniformTM(16384, 200, 8, seed=0)
    assert tm.right_path(torch.float32) == "tc"
    g = torch.Generator(device=cuda).manual_seed(3)
    a = torch.randn(512, 16384, dtype=torch.float32, device=cuda, generator=g)
    y_tc = tm.apply_right(a).double().cpu().numpy()
    monkeypatch.setenv("SKETCH_B200_SPARSE_RIGHT", "gather")
    y_g = tm.apply_right(a).double().cpu().numpy()
    ref = orc.csr_right(orc.sparse_uniform_csr(16384, 200, 8, 0), a.cpu().numpy())
    assert rel_err(y_tc, ref) <= 1e-5
    assert rel_err(y_g, ref) <= 1e-5


def test_khatri_rao_config5_rows(cuda):
    import torch

    tm = skb.KhatriRaoTM(256, 2, 512, "real_rademacher", seed=0)
    assert tm.right_path(torch.float32) == "tc"
    rng = np.random.default_rng(5)
    u = rng.standard_normal((48, 5, 256))
    v = rng.standard_normal((48, 5, 256))
    a = (np.einsum("nrp,nrq->npq", u, v) + 1e-2 * rng.standard_normal((48, 256, 256))).reshape(48, 65536)
    a = a.astype(np.float32)
    y = tm.apply_right(torch.from_numpy(a).to(cuda)).double().cpu().numpy()
    ref = orc.kr_right(orc.kr_factors(256, 2, 512, 0), a)
    assert rel_err(y, ref) <= 1e-5


@pytest.mark.parametrize("base,d0,ell,k", [("real_rademacher", 16, 2, 48), ("real_gaussian", 8, 3, 20),
                                           ("real_rademacher", 4, 4, 600)])
def test_khatri_rao_small(base, d0, ell, k, cuda):
    import torch

    tm = skb.KhatriRaoTM(d0, ell, k, base, seed=4)
    rng = np.random.default_rng(1)
    a = rng.standard_normal((37, d0**ell)).astype(np.float32)
    y = tm.apply_right(torch.from_numpy(a).to(cuda)).double().cpu().numpy()
    ref = orc.kr_right(orc.kr_factors(d0, ell, k, 4, base), a)
    assert rel_err(y, ref) <= 1e-5


def test_gaussian_f32(cuda):
    import torch

    tm = skb.GaussianTM(1024, 96, seed=9)
    rng = np.random.default_rng(2)
    a = rng.standard_normal((333, 1024)).astype(np.float32)
    y = tm.apply_right(torch.from_numpy(a).to(cuda)).double().cpu().numpy()
    assert rel_err(y, orc.dense_right(orc.gaussian_dense(1024, 96, 9), a)) <= 1e-5
