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


def _cfg5_rows(n, seed):
    """Config-5 input rows: vec(sum of 5 rank-one 256 x 256 outer products + 1e-2 noise), float32."""
    rng = np.random.default_rng(seed)
    u = rng.standard_normal((n, 5, 256))
    v = rng.standard_normal((n, 5, 256))
    a = np.einsum("nrp,nrq->npq", u, v) + 1e-2 * rng.standard_normal((n, 256, 256))
    return a.reshape(n, 65536).astype(np.float32)


def test_khatri_rao_config5_rows(cuda):
    """The production CTA-pair KR kernel (sk_kr_right: Omega never formed, F resident, split P
    range) on 256 config-5 rows at the full d = 65536, k = 512, against the oracle."""
    import torch

    tm = skb.KhatriRaoTM(256, 2, 512, "real_rademacher", seed=0)
    assert tm.right_path(torch.float32) == "tc"
    a = _cfg5_rows(256, 5)
    y = tm.apply_right(torch.from_numpy(a).to(cuda)).double().cpu().numpy()
    ref = orc.right_chunked(lambda x: orc.kr_right(orc.kr_factors(256, 2, 512, 0), x), a, rows=32, threads=8)
    assert rel_err(y, ref) <= 1e-5
    assert not any(k[0] == "dense" for k in tm._device_cache)  # no materialised Omega on the device


def test_khatri_rao_config5_full(cuda):
    """All 16384 config-5 rows (every pair tile, both N-block groups, the K splits): float64
    contraction on the device for the whole output + oracle rows from three separate tiles."""
    import torch

    tm = skb.KhatriRaoTM(256, 2, 512, "real_rademacher", seed=0)
    g = torch.Generator(device=cuda).manual_seed(11)
    n = 16384
    u = torch.randn(n, 5, 256, device=cuda, generator=g)
    v = torch.randn(n, 5, 256, device=cuda, generator=g)
    a = (torch.einsum("nrp,nrq->npq", u, v) + 1e-2 * torch.randn(n, 256, 256, device=cuda, generator=g))
    a = a.reshape(n, 65536).contiguous()
    del u, v
    y = tm.apply_right(a).double()
    f = torch.as_tensor(orc.kr_factors(256, 2, 512, 0), device=cuda)
    ref = torch.empty_like(y)
    for r0 in range(0, n, 1024):  # Y = sum_p f0[p] * (A[:, p, :] @ f1) in float64
        t = a[r0:r0 + 1024].double().reshape(-1, 256, 256) @ f[1]
        ref[r0:r0 + 1024] = torch.einsum("npj,pj->nj", t, f[0]) / np.sqrt(512)
    err = float(torch.linalg.norm(y - ref) / torch.linalg.norm(ref))
    assert err <= 1e-5, err
    rows = np.r_[0:8, 8000:8008, 16376:16384]
    ref_o = orc.kr_right(orc.kr_factors(256, 2, 512, 0), a[rows].cpu().numpy())
    assert rel_err(y[rows].cpu().numpy(), ref_o) <= 1e-5


@pytest.mark.parametrize("d0,ell,k", [(256, 2, 512), (16, 2, 48), (4, 4, 600), (5, 2, 70), (64, 2, 100)])
def test_khatri_rao_sign_bits_match_float_weights(d0, ell, k, cuda, monkeypatch):
    """sk_kr_right_signs (+-1 weights as sign bits) against sk_kr_right (float32 weights): the fold
    adds +-z either way, so the results agree bit for bit; both against the oracle."""
    import torch

    tm = skb.KhatriRaoTM(d0, ell, k, "real_rademacher", seed=3)
    if tm.right_path(torch.float32) != "tc":
        pytest.skip("not a tensor-core shape")
    assert tm._tc_operands(cuda)[5] is not None
    rng = np.random.default_rng(k)
    a = torch.from_numpy(rng.standard_normal((300, d0 ** ell)).astype(np.float32)).to(cuda)
    y = tm.apply_right(a)
    monkeypatch.setenv("SKETCH_B200_KR_SIGNS", "0")
    y0 = tm.apply_right(a)
    assert torch.equal(y, y0)
    ref = orc.kr_right(orc.kr_factors(d0, ell, k, 3), a.cpu().numpy())
    assert rel_err(y.double().cpu().numpy(), ref) <= 1e-5


def test_khatri_rao_config5_adjoint_in_place(cuda):
    """Omega^T B for a tall B (65536 x 40) read in place by the transposing KR kernel."""
    import torch

    tm = skb.KhatriRaoTM(256, 2, 512, "real_rademacher", seed=0)
    rng = np.random.default_rng(8)
    b = rng.standard_normal((65536, 40)).astype(np.float32)
    x = tm.apply_adjoint(torch.from_numpy(b).to(cuda)).double().cpu().numpy()
    ref = orc.kr_right(orc.kr_factors(256, 2, 512, 0), b.T).T
    assert x.shape == (512, 40)
    assert rel_err(x, ref) <= 1e-5
    xv = tm.apply_adjoint(torch.from_numpy(b[:, 3].copy()).to(cuda)).double().cpu().numpy()
    assert xv.shape == (512,)
    assert rel_err(xv, ref[:, 3]) <= 1e-5


@pytest.mark.parametrize("base,d0,ell,k", [("real_rademacher", 16, 2, 48), ("real_gaussian", 8, 3, 20),
                                           ("real_rademacher", 4, 4, 600), ("real_gaussian", 100, 2, 300),
                                           ("real_rademacher", 5, 2, 70), ("real_spherical", 12, 2, 33),
                                           ("real_rademacher", 2, 5, 9)])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_khatri_rao_small(base, d0, ell, k, dtype, cuda):
    """Every real KR shape class: tcgen05 with grouped trailing factors (d0 = 16, 8, 4), padded
    q blocks (d0 = 100), split F (Gaussian/spherical), the CUDA-core form (d0 = 5, 2; float64)."""
    import torch

    tm = skb.KhatriRaoTM(d0, ell, k, base, seed=4)
    rng = np.random.default_rng(1)
    a = rng.standard_normal((333, d0**ell))
    b = rng.standard_normal((d0**ell, 7))
    tdt = getattr(torch, dtype)
    tol = 1e-5 if dtype == "float32" else 1e-12
    fac = orc.kr_factors(d0, ell, k, 4, base)
    y = tm.apply_right(torch.from_numpy(a).to(cuda, tdt)).double().cpu().numpy()
    assert rel_err(y, orc.kr_right(fac, a.astype(dtype))) <= tol
    x = tm.apply_adjoint(torch.from_numpy(b).to(cuda, tdt)).double().cpu().numpy()
    assert rel_err(x, orc.kr_right(fac, b.astype(dtype).T).T) <= tol


def test_khatri_rao_numpy_float64_dropin(cuda):
    """A NumPy float64 caller (the reference's dtype) gets float64 through the CUDA-core kernel."""
    tm = skb.KhatriRaoTM(64, 2, 96, "real_rademacher", seed=2)
    rng = np.random.default_rng(3)
    a = rng.standard_normal((500, 4096))
    y = tm.apply_right(a)
    assert y.dtype == np.float64
    assert rel_err(y, orc.kr_right(orc.kr_factors(64, 2, 96, 2), a)) <= 1e-12


def test_gaussian_f32(cuda):
    import torch

    tm = skb.GaussianTM(1024, 96, seed=9)
    rng = np.random.default_rng(2)
    a = rng.standard_normal((333, 1024)).astype(np.float32)
    y = tm.apply_right(torch.from_numpy(a).to(cuda)).double().cpu().numpy()
    assert rel_err(y, orc.dense_right(orc.gaussian_dense(1024, 96, 9), a)) <= 1e-5


@pytest.mark.parametrize("dt", ["float64", "float32"])
def test_gaussian_dense_families_own_kernel(dt, cuda):
    """float64 Gaussian (the reference's dtype) and every real adjoint of a materialised family run the
    library's CUDA-core contraction kernel (float64 accumulation), not cuBLAS."""
    import torch

    tm = skb.GaussianTM(3000, 70, seed=11)
    rng = np.random.default_rng(4)
    a = rng.standard_normal((257, 3000))
    b = rng.standard_normal((3000, 9))
    tdt = getattr(torch, dt)
    tol = 1e-12 if dt == "float64" else 1e-5
    om = orc.gaussian_dense(3000, 70, 11)
    y = tm.apply_right(torch.from_numpy(a).to(cuda, tdt)).double().cpu().numpy()
    x = tm.apply_adjoint(torch.from_numpy(b).to(cuda, tdt)).double().cpu().numpy()
    assert rel_err(y, a.astype(dt).astype(np.float64) @ om) <= tol
    assert rel_err(x, om.T @ b.astype(dt).astype(np.float64)) <= tol
    assert any(k[0] == "dense_cc" for k in tm._device_cache)


def test_khatri_rao_wide_k_slabs(cuda):
    """k > 2048 runs the KR kernel in column slabs (N-block groups per launch): k = 2100 = 2048 + 52."""
    import torch

    tm = skb.KhatriRaoTM(16, 2, 2100, "real_rademacher", seed=6)
    rng = np.random.default_rng(2)
    a = rng.standard_normal((200, 256)).astype(np.float32)
    b = rng.standard_normal((256, 5)).astype(np.float32)
    fac = orc.kr_factors(16, 2, 2100, 6)
    y = tm.apply_right(torch.from_numpy(a).to(cuda)).double().cpu().numpy()
    x = tm.apply_adjoint(torch.from_numpy(b).to(cuda)).double().cpu().numpy()
    assert rel_err(y, orc.kr_right(fac, a)) <= 1e-5
    assert rel_err(x, orc.kr_right(fac, b.T).T) <= 1e-5
