"""K1c (csrc/sparse_right_cols.cu, lanes = output columns) against the oracle and the older kernels.

The sparse-sign right applies (`_SparseTM.apply_right`, reference src/sketch/sparse.py:63-66) take
K1c by default; these tests pin the slab path (lists longer than 128 or rows longer than the ring),
groups of 256 columns, ragged k, the fall-back for rows that are not 16-byte aligned, and agreement
with K1r / K1 (SKETCH_B200_K1=ring / classic).
"""

import numpy as np
import pytest

import oracle as orc
from _cases import rel_err
from paper_2508_21189_b200 import sketch as skb

pytestmark = pytest.mark.gpu

TOL = {np.float64: 1e-12, np.float32: 1e-5}


def _dt(dt):
    import torch

    return torch.float64 if dt == np.float64 else torch.float32


def _plan(tm, a):
    from paper_2508_21189_b200 import _lib

    code = _lib.SK_F64 if a.dtype.itemsize == 8 else _lib.SK_F32
    return tm._cols_on(a.device, code)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("d,k,zeta,n,nslab", [(4096, 256, 4, 777, 1), (1000, 300, 5, 33, 1), (8192, 256, 8, 70, 2),
                                              (16000, 64, 1, 9, 4), (512, 1000, 40, 129, 1)])
def test_cols_vs_oracle(d, k, zeta, n, nslab, dt, cuda):
    import torch

    rng = np.random.default_rng(d * 7 + k)
    a = rng.standard_normal((n, d)).astype(dt)
    tm = skb.SparseUniformTM(d, k, zeta, seed=5)
    at = torch.as_tensor(a).to(cuda)
    if dt == np.float32 and tm.right_path(_dt(dt)) == "tc":
        pytest.skip("float32 operator with many nonzeros per row takes the tensor-core form")
    plan = _plan(tm, at)
    assert plan is not None and (len(plan[0]) == 1) == (nslab == 1) and len(plan[0]) >= nslab
    y = tm.apply_right(at).cpu().numpy()
    ref = orc.csr_right(orc.sparse_uniform_csr(d, k, zeta, 5), a)
    assert rel_err(y, ref) <= TOL[dt]


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_cols_matches_ring_and_classic(dt, cuda, monkeypatch):
    import torch

    tm_args = (4096, 256, 4)
    g = torch.Generator(device=cuda).manual_seed(1)
    a = torch.randn(5000, 4096, dtype=_dt(dt), device=cuda, generator=g)
    y = skb.SparseUniformTM(*tm_args, seed=2).apply_right(a)
    for mode in (["ring", "classic"] if dt == np.float64 else ["classic"]):
        monkeypatch.setenv("SKETCH_B200_K1", mode)
        y2 = skb.SparseUniformTM(*tm_args, seed=2).apply_right(a)
        assert float((y - y2).norm() / y2.norm()) <= (1e-14 if dt == np.float64 else 1e-6)


def test_cols_long_lists_take_the_ring(cuda):
    """Lists beyond 4 slabs (here ~650 entries per column) go to K1r; same result as the oracle."""
    import torch

    d, k, zeta, n = 16384, 200, 8, 40
    tm = skb.SparseUniformTM(d, k, zeta, seed=6)
    a = torch.randn(n, d, dtype=torch.float64, device=cuda)
    assert _plan(tm, a) is None
    ref = orc.csr_right(orc.sparse_uniform_csr(d, k, zeta, 6), a.cpu().numpy())
    assert rel_err(tm.apply_right(a).cpu().numpy(), ref) <= 1e-12


def test_cols_unaligned_rows_fall_back(cuda):
    """A view whose rows are not 16-byte aligned cannot be bulk-copied: the apply takes K1r."""
    import torch

    d, k = 1002, 40
    base = torch.randn(300, d + 1, dtype=torch.float64, device=cuda)
    a = base[:, 1:]  # 8-byte offset rows, stride d + 1 (odd)
    tm = skb.SparseUniformTM(d, k, 3, seed=4)
    y = tm.apply_right(a).cpu().numpy()
    ref = orc.csr_right(orc.sparse_uniform_csr(d, k, 3, 4), a.cpu().numpy())
    assert rel_err(y, ref) <= 1e-12


def test_cols_config1_full_size(cuda):
    """BASELINE config 1 at full size: every row against the oracle (float64, 1e-12)."""
    import torch

    d, k, zeta, n = 4096, 256, 4, 16384
    tm = skb.SparseUniformTM(d, k, zeta, seed=0)
    g = torch.Generator(device=cuda).manual_seed(11)
    a = torch.randn(n, d, dtype=torch.float64, device=cuda, generator=g)
    plan = _plan(tm, a)
    assert plan is not None and len(plan[0]) == 1 and plan[0][0][5] == 96
    y = tm.apply_right(a).cpu().numpy()
    ref = orc.csr_right(orc.sparse_uniform_csr(d, k, zeta, 0), a.cpu().numpy())
    assert rel_err(y, ref) <= 1e-12


def test_cols_empty_and_single_row(cuda):
    import torch

    tm = skb.SparseUniformTM(256, 40, 2, seed=1)
    a0 = torch.zeros(0, 256, dtype=torch.float64, device=cuda)
    assert tm.apply_right(a0).shape == (0, 40)
    a1 = torch.randn(1, 256, dtype=torch.float64, device=cuda)
    ref = orc.csr_right(orc.sparse_uniform_csr(256, 40, 2, 1), a1.cpu().numpy())
    assert rel_err(tm.apply_right(a1).cpu().numpy(), ref) <= 1e-12


@pytest.mark.parametrize("d,k,zeta,dt", [(2, 1, 1, np.float64), (6, 3, 2, np.float64), (8, 40, 3, np.float32),
                                         (1001, 33, 4, np.float64), (1002, 257, 9, np.float32),
                                         (4100, 512, 4, np.float64)])
def test_cols_odd_shapes(d, k, zeta, dt, cuda):
    """Tiny / odd d (odd d or d * 4 % 16 != 0 cannot bulk-copy rows and falls back), k of one lane,
    ragged groups of 256 columns; every case against the oracle."""
    import torch

    rng = np.random.default_rng(d + 3 * k)
    a = rng.standard_normal((77, d)).astype(dt)
    tm = skb.SparseUniformTM(d, k, min(zeta, k), seed=9)
    at = torch.as_tensor(a).to(cuda)
    y = tm.apply_right(at).cpu().numpy()
    ref = orc.csr_right(orc.sparse_uniform_csr(d, k, min(zeta, k), 9), a)
    assert rel_err(y, ref) <= TOL[dt]


def test_cols_stack_and_iid_families(cuda):
    """SparseStack (zeta blocks) and SparseIID (variable nonzeros per row) take K1c as well."""
    import torch

    a = torch.randn(500, 2048, dtype=torch.float64, device=cuda)
    for tm in (skb.SparseStackTM(2048, 4, 24, seed=1), skb.SparseIIDTM(2048, 96, 4.0, seed=2)):
        plan = _plan(tm, a)
        assert plan is not None
        y = tm.apply_right(a).cpu().numpy()
        ref = a.cpu().numpy() @ tm.materialize()
        assert rel_err(y, ref) <= 1e-12
