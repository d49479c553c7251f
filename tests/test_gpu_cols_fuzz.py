"""Randomised shapes through the default sparse-sign right apply (K1c with its K1r / K1 fall-backs)
against the oracle: d, k, zeta, n, dtype and row strides drawn from a fixed seed."""

import numpy as np
import pytest

import oracle as orc
from _cases import rel_err
from paper_2508_21189_b200 import sketch as skb

pytestmark = pytest.mark.gpu

_rng = np.random.default_rng(2024)
CASES = []
for _ in range(24):
    d = int(_rng.choice([8, 64, 130, 512, 1000, 2048, 3000, 4096, 6144]))
    k = int(_rng.integers(1, 700))
    zeta = int(min(k, _rng.integers(1, 9)))
    n = int(_rng.choice([1, 7, 129, 1000]))
    dt = np.float64 if _rng.random() < 0.6 else np.float32
    pad = int(_rng.choice([0, 0, 1, 4]))
    CASES.append((d, k, zeta, n, dt, pad))


@pytest.mark.parametrize("d,k,zeta,n,dt,pad", CASES)
def test_sparse_right_fuzz(d, k, zeta, n, dt, pad, cuda):
    import torch

    rng = np.random.default_rng(d * 31 + k * 7 + n)
    a = rng.standard_normal((n, d)).astype(dt)
    tm = skb.SparseUniformTM(d, k, zeta, seed=d + k)
    base = torch.zeros((n, d + pad), dtype=torch.float64 if dt == np.float64 else torch.float32, device=cuda)
    base[:, :d] = torch.as_tensor(a).to(cuda)
    at = base[:, :d]  # row stride d + pad
    y = tm.apply_right(at).cpu().numpy()
    ref = orc.csr_right(orc.sparse_uniform_csr(d, k, zeta, d + k), a)
    assert rel_err(y, ref) <= (1e-12 if dt == np.float64 else 1e-5)
