"""World-size-2 runs of the row-sharded drivers with the PRODUCT operators and kernels on CUDA
tensors (both ranks on cuda:0, gloo collectives): the sharded S A with device-sliced row blocks,
the distributed LSQR and rSVD, against the single-process product result and the oracle.

The CPU-only twins in test_dist_gloo.py check the partition/reduction logic with an oracle
operator; these check that the kernels themselves run under torch.distributed.
"""

import os

import numpy as np
import pytest

import oracle as orc

pytestmark = pytest.mark.gpu


def _problem():
    rng = np.random.default_rng(0)
    n, d, k = 300001, 64, 512
    a = (rng.standard_normal((n, d)) * (1.0 + rng.pareto(1.5, size=n))[:, None]).astype(np.float32)
    b = (a.astype(np.float64) @ rng.standard_normal(d) + 1e-3 * rng.standard_normal(n)).astype(np.float32)
    return a, b, k


def _sa_job(rank, world):
    import torch

    from paper_2508_21189_b200 import dist as skd
    from paper_2508_21189_b200.sketch import SparseUniformTM

    a, b, k = _problem()
    r0, r1 = skd.row_range(a.shape[0], world, rank)
    dev = torch.device("cuda", 0)
    tm = SparseUniformTM(a.shape[0], k, 8, seed=0)
    sa = skd.sharded_adjoint(tm, torch.from_numpy(a[r0:r1]).to(dev), r0)
    res = skd.sharded_lsqr(torch.from_numpy(a[r0:r1]).to(dev), torch.from_numpy(b[r0:r1]).to(dev), tm, r0,
                           atol=1e-10, btol=0.0)
    return sa.cpu().numpy(), res.x.double().cpu().numpy(), res.itn


def _rsvd_job(rank, world):
    import torch

    from paper_2508_21189_b200 import dist as skd
    from paper_2508_21189_b200.sketch import SparseUniformTM

    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(5)
    n, d, k = 20000, 1024, 64
    u, _ = torch.linalg.qr(torch.randn(n, k * 2, device=dev, dtype=torch.float64, generator=g))
    v, _ = torch.linalg.qr(torch.randn(d, k * 2, device=dev, dtype=torch.float64, generator=g))
    a = ((u * torch.arange(1, 2 * k + 1, device=dev, dtype=torch.float64) ** -2.0) @ v.T).float()
    r0, r1 = skd.row_range(n, world, rank)
    tm = SparseUniformTM(d, k, 8, seed=3)
    f = skd.sharded_rsvd(a[r0:r1], k, tm)
    err = skd.sharded_residual(a[r0:r1], f)
    return f.sigma.cpu().numpy(), err


def test_sharded_sa_and_lsqr_product_kernels():
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_dist_gloo import _run

    out = _run(_sa_job)
    a, b, k = _problem()
    ref = orc.csr_adjoint(orc.sparse_uniform_csr(a.shape[0], k, 8, 0), a)
    for r, (sa, x, itn) in out.items():
        assert np.linalg.norm(sa - ref) / np.linalg.norm(ref) <= 1e-5
    assert np.array_equal(out[0][1], out[1][1])  # every rank holds the same x
    # same x as a single-process solve (same sketch, same iterations up to reduction order)
    import torch

    from paper_2508_21189_b200 import rand_nla
    from paper_2508_21189_b200.sketch import SparseUniformTM

    dev = torch.device("cuda", 0)
    x1 = rand_nla.sketch_precondition_lsqr(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev),
                                           SparseUniformTM(a.shape[0], k, 8, seed=0), atol=1e-10, btol=0.0).x
    x1 = x1.double().cpu().numpy()
    assert np.linalg.norm(out[0][1] - x1) / np.linalg.norm(x1) <= 1e-6


def test_sharded_rsvd_product_kernels():
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_dist_gloo import _run

    out = _run(_rsvd_job)
    (s0, e0), (s1, e1) = out[0], out[1]
    assert np.array_equal(s0, s1) and e0 == e1
    s_one, e_one = _rsvd_job(0, 1)  # the same job in one process (no torch.distributed)
    assert np.allclose(s0, s_one, rtol=1e-6)
    assert abs(e0 - e_one) <= 1e-4 * e_one
