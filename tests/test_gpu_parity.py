"""GPU parity: the CUDA kernels (through the C ABI) against the CPU oracle and golden vectors.

Tolerances (BASELINE north_star): relative Frobenius error <= 1e-12 for float64 inputs and
<= 1e-5 for float32 inputs, always measured in float64 against the float64 oracle.
"""

import numpy as np
import pytest

import oracle as orc
from _cases import CASES, oracle_right, product, rel_err
from paper_2508_21189_b200 import sketch as skb

pytestmark = pytest.mark.gpu

TOL = {np.float64: 1e-12, np.float32: 1e-5}


def _t(a, dev, dt):
    import torch

    return torch.as_tensor(np.asarray(a, dtype=dt)).to(dev)


@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_right_numpy(name, golden, cuda):
    """Drop-in call with NumPy in, NumPy float64 out, against the reference's own outputs."""
    tm = product(name)
    a = golden[f"{name}__A"]
    y = tm.apply_right(a)
    assert isinstance(y, np.ndarray) and y.dtype == np.float64
    assert rel_err(y, golden[f"{name}__right"]) <= 1e-12


@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_adjoint_numpy(name, golden, cuda):
    tm = product(name)
    b = golden[f"{name}__B"]
    assert rel_err(tm.apply_adjoint(b), golden[f"{name}__adjoint"]) <= 1e-12
    v = tm.apply_adjoint(b[:, 0])
    assert v.shape == (tm.k,)
    assert rel_err(v, golden[f"{name}__adjoint_vec"]) <= 1e-12


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("d,k,zeta,n", [(4096, 256, 4, 100), (16384, 200, 8, 64), (1000, 300, 5, 33), (700, 64, 1, 5),
                                        (513, 17, 3, 1), (64, 600, 4, 40)])
def test_sparse_right_vs_oracle(d, k, zeta, n, dt, cuda):
    rng = np.random.default_rng(d + k)
    a = rng.standard_normal((n, d)).astype(dt)
    tm = skb.SparseUniformTM(d, k, zeta, seed=3)
    y = tm.apply_right(_t(a, cuda, dt)).cpu().numpy()
    ref = orc.csr_right(orc.sparse_uniform_csr(d, k, zeta, 3), a)
    assert rel_err(y, ref) <= TOL[dt]


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("d,k,zeta,n", [(4096, 256, 4, 10007), (2048, 200, 8, 4900), (1536, 72, 2, 6001)])
def test_sparse_right_many_row_tiles(d, k, zeta, n, dt, cuda, monkeypatch):
    """Several row tiles per persistent CTA (chunk stream across tile boundaries, ragged last tile,
    k not a multiple of the column block), and the persistent form equal to the classic one."""
    import torch

    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, d)).astype(dt)
    tm = skb.SparseUniformTM(d, k, zeta, seed=11)
    at = _t(a, cuda, dt)
    y = tm.apply_right(at).cpu().numpy()
    ref = orc.csr_right(orc.sparse_uniform_csr(d, k, zeta, 11), a)
    assert rel_err(y, ref) <= TOL[dt]
    monkeypatch.setenv("SKETCH_B200_K1_CLASSIC", "1")
    y2 = tm.apply_right(at)
    torch.cuda.synchronize()
    assert rel_err(y2.cpu().numpy(), y) <= (1e-15 if dt == np.float64 else 1e-6)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("d,k,zeta,m", [(4096, 2048, 8, 40), (20000, 256, 8, 512), (1000, 300, 5, 1), (777, 64, 3, 33)])
def test_sparse_adjoint_vs_oracle(d, k, zeta, m, dt, cuda):
    rng = np.random.default_rng(d + m)
    b = rng.standard_normal((d, m)).astype(dt)
    tm = skb.SparseUniformTM(d, k, zeta, seed=5)
    y = tm.apply_adjoint(_t(b, cuda, dt)).cpu().numpy()
    ref = orc.csr_adjoint(orc.sparse_uniform_csr(d, k, zeta, 5), b)
    assert rel_err(y, ref) <= TOL[dt]


def test_sparse_misaligned_and_strided(cuda):
    import torch

    d, k = 1000, 48
    tm = skb.SparseStackTM(d, 4, 12, seed=9)
    big = torch.randn(37, d + 3, dtype=torch.float32, device=cuda)
    a = big[:, 1:d + 1]  # row stride d+3, base not 16-byte aligned -> scalar loader
    y = tm.apply_right(a).cpu().numpy()
    ref = orc.csr_right(orc.sparse_stack_csr(d, 4, 12, 9), a.cpu().numpy())
    assert rel_err(y, ref) <= 1e-5


def test_zero_and_empty_inputs(cuda):
    tm = skb.SparseUniformTM(300, 40, 4, seed=1)
    assert np.all(tm.apply_right(np.zeros((5, 300))) == 0)
    assert tm.apply_right(np.zeros((0, 300))).shape == (0, 40)
    assert np.all(tm.apply_adjoint(np.zeros((300, 3))) == 0)
    assert np.array_equal(tm.apply_right(np.eye(300)), tm.materialize())


def test_identity_input_equals_materialize(cuda):
    for tm in (skb.SparseStackTM(64, 2, 8, seed=1), skb.SparseRttTM(256, 32, 2, "wht", seed=2),
               skb.SparseColTM(50, 9, 3, seed=4)):
        assert rel_err(tm.apply_right(np.eye(tm.d)), tm.materialize()) <= 1e-13


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("d,k,xi,n", [(8192, 512, 1, 70), (1024, 100, 3, 9), (2048, 64, 2, 5), (4096, 256, 1, 3),
                                      (16384, 128, 2, 4), (256, 64, 1, 7), (32, 12, 4, 2), (512, 64, 2, 301),
                                      (64, 16, 3, 9), (128, 128, 1, 33), (16, 8, 2, 5), (32768, 300, 2, 5),
                                      (65536, 64, 1, 3)])
def test_srtt_wht_vs_oracle(d, k, xi, n, dt, cuda):
    rng = np.random.default_rng(d * 3 + xi)
    a = (rng.standard_normal((n, d)) / np.arange(1, d + 1)).astype(dt)
    tm = skb.SparseRttTM(d, k, xi, "wht", seed=11)
    y = tm.apply_right(_t(a, cuda, dt)).cpu().numpy()
    dv, samp = orc.srtt_parts(d, k, xi, 11)
    ref = orc.srtt_right(dv, samp, a, "wht")
    assert rel_err(y, ref) <= TOL[dt]


@pytest.mark.parametrize("d", [8192, 512, 64])
def test_srtt_uniform_diagonal(d, cuda):
    k, xi = 64, 2
    rng = np.random.default_rng(1)
    a = rng.standard_normal((6, d))
    tm = skb.SparseRttTM(d, k, xi, "wht", diagonal="uniform_symmetric", seed=4)
    dv, samp = orc.srtt_parts(d, k, xi, 4, "uniform_symmetric")
    assert rel_err(tm.apply_right(a), orc.srtt_right(dv, samp, a, "wht")) <= 1e-12


@pytest.mark.parametrize("d", [16, 8192, 32768])
def test_wht_function(d, cuda):
    x = np.random.default_rng(0).standard_normal((d, 3))
    y = skb.wht(x)
    assert rel_err(np.asarray(y), orc.wht_rows(x.T).T) <= 1e-13
    assert rel_err(np.asarray(skb.wht(np.asarray(y))), x) <= 1e-13


def test_linearity_at_config_sizes(cuda):
    """Size-independent property at full config-1 size: Y(aA + bB) = aY(A) + bY(B)."""
    import torch

    tm = skb.SparseUniformTM(4096, 256, 4, seed=0)
    g = torch.Generator(device=cuda).manual_seed(0)
    a = torch.randn(16384, 4096, dtype=torch.float64, device=cuda, generator=g)
    b = torch.randn(16384, 4096, dtype=torch.float64, device=cuda, generator=g)
    lhs = tm.apply_right(2.0 * a - 3.0 * b)
    rhs = 2.0 * tm.apply_right(a) - 3.0 * tm.apply_right(b)
    assert float((lhs - rhs).norm() / rhs.norm()) <= 1e-13
    # spot-check 256 rows against the oracle
    rows = torch.arange(0, 16384, 64, device=cuda)
    ref = orc.csr_right(orc.sparse_uniform_csr(4096, 256, 4, 0), a[rows].cpu().numpy())
    assert rel_err(tm.apply_right(a)[rows].cpu().numpy(), ref) <= 1e-12


def test_config2_rows_vs_oracle(cuda):
    """BASELINE config 2 operator on a 256-row slab of the config's input distribution."""
    import torch

    tm = skb.SparseRttTM(8192, 512, 1, "wht", seed=0)
    g = torch.Generator(device=cuda).manual_seed(1)
    a = torch.randn(256, 8192, dtype=torch.float32, device=cuda, generator=g)
    a /= torch.arange(1, 8193, device=cuda, dtype=torch.float32)
    y = tm.apply_right(a).cpu().numpy()
    dv, samp = orc.srtt_parts(8192, 512, 1, 0)
    assert rel_err(y, orc.srtt_right(dv, samp, a.cpu().numpy(), "wht")) <= 1e-5


def test_pipelined_host_path_matches_device(cuda):
    """Host operands >= 256 MB stream through the device in chunks (H2D / kernel / D2H overlap)."""
    import torch

    tm = skb.SparseRttTM(8192, 512, 1, "wht", seed=0)
    g = torch.Generator().manual_seed(0)
    a_host = torch.randn(9000, 8192, generator=g)  # 295 MB, not a multiple of the chunk
    ref = tm.apply_right(a_host.to(cuda)).cpu()
    y_pageable = tm.apply_right(a_host)
    assert y_pageable.dtype == torch.float32 and not y_pageable.is_cuda
    assert torch.equal(y_pageable, ref)
    y_pinned = tm.apply_right(a_host.pin_memory())
    assert torch.equal(y_pinned, ref)
    y_np = tm.apply_right(a_host.numpy())
    assert isinstance(y_np, np.ndarray) and y_np.dtype == np.float64
    assert np.array_equal(y_np, ref.double().numpy())


@pytest.mark.parametrize("n", [0, 1, 2, 3, 149, 297])
def test_srtt_tc_row_counts_and_strides(n, cuda):
    """The tcgen05 SRTT kernel (d = 8192, float32): odd row counts, fewer rows than SMs, padded lda."""
    import torch

    d, k = 8192, 512
    tm = skb.SparseRttTM(d, k, 1, "wht", seed=2)
    g = torch.Generator(device=cuda).manual_seed(n)
    big = torch.randn(max(n, 1), d + 12, device=cuda, generator=g)[:n]
    a = big[:, 4:d + 4]  # lda = d + 12, rows start 16 bytes in: bulk copies stay 16-byte aligned
    y = tm.apply_right(a)
    assert y.shape == (n, k)
    if n:
        dv, samp = orc.srtt_parts(d, k, 1, 2)
        assert rel_err(y.cpu().numpy(), orc.srtt_right(dv, samp, a.cpu().numpy(), "wht")) <= 1e-5
        # strided and contiguous launches agree
        assert rel_err(y.cpu().numpy(), tm.apply_right(a.contiguous()).cpu().numpy()) <= 1e-5


@pytest.mark.parametrize("d", [2048, 4096, 8192])
def test_srtt_tc_matches_cuda_core_kernel(d, cuda, monkeypatch):
    import torch

    tm = skb.SparseRttTM(d, 512, 3, "wht", seed=9)
    a = torch.randn(1000, d, device=cuda)
    y_tc = tm.apply_right(a).double()
    monkeypatch.setenv("SKETCH_B200_SRTT", "regs")
    y_cc = tm.apply_right(a).double()
    assert float((y_tc - y_cc).norm() / y_cc.norm()) <= 1e-5


def _families():
    return [skb.SparseUniformTM(512, 48, 4, seed=1), skb.SparseStackTM(512, 4, 12, seed=2),
            skb.SparseIIDTM(512, 40, 3.0, seed=3), skb.SparseColTM(512, 30, 2, seed=4),
            skb.SparseRttTM(512, 32, 2, "wht", seed=5), skb.SparseRttTM(512, 32, 2, "dct", seed=6),
            skb.KhatriRaoTM(8, 3, 24, "real_rademacher", seed=7), skb.GaussianTM(512, 20, seed=8)]


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_edge_shapes_every_family(dt, cuda):
    """Empty, single-row, 1-D and strided (non-contiguous) operands on every family, host and
    device, against the materialized Omega."""
    import torch

    rng = np.random.default_rng(0)
    for tm in _families():
        om = tm.materialize()
        tol = 1e-12 if dt == np.float64 else 1e-5
        # empty operands keep their shapes
        assert tm.apply_right(np.zeros((0, tm.d), dt)).shape == (0, tm.k)
        assert tm.apply_adjoint(np.zeros((tm.d, 0), dt)).shape == (tm.k, 0)
        z = tm.apply_right(torch.zeros((0, tm.d), dtype=torch.float64 if dt == np.float64 else torch.float32,
                                       device=cuda))
        assert tuple(z.shape) == (0, tm.k)
        # one row, and a 1-D adjoint operand (squeezed like the reference, base.py:86-91)
        a1 = rng.standard_normal((1, tm.d)).astype(dt)
        assert rel_err(tm.apply_right(a1), a1.astype(np.float64) @ om) <= tol
        v = rng.standard_normal(tm.d).astype(dt)
        got = tm.apply_adjoint(v)
        assert got.shape == (tm.k,) and rel_err(got, om.T @ v.astype(np.float64)) <= tol
        # strided device operands (a column slice and a transposed view)
        big = torch.as_tensor(rng.standard_normal((9, 2 * tm.d)).astype(dt)).to(cuda)
        sl = big[:, ::2]
        assert rel_err(tm.apply_right(sl).cpu().numpy(), sl.cpu().double().numpy() @ om) <= tol
        bt = torch.as_tensor(rng.standard_normal((7, tm.d)).astype(dt)).to(cuda).T
        assert rel_err(tm.apply_adjoint(bt).cpu().numpy(), om.T @ bt.cpu().double().numpy()) <= tol


def test_right_paths_randomized(cuda):
    """Random shapes, families and dtypes through the default right-apply paths (K1 persistent /
    classic, tensor-core dense form, SRTT, Khatri-Rao) against the materialized Omega."""
    import torch

    rng = np.random.default_rng(7)
    for trial in range(20):
        n = int(rng.integers(1, 3000))
        dt = torch.float32 if trial % 2 else torch.float64
        fam = trial % 5
        if fam == 0:
            d, k = int(rng.integers(1, 9000)), int(rng.integers(1, 700))
            tm = skb.SparseUniformTM(d, k, int(rng.integers(1, min(k, 8) + 1)), seed=trial)
        elif fam == 1:
            d = int(rng.integers(1, 9000))
            z = int(rng.integers(1, 5))
            tm = skb.SparseStackTM(d, z, int(rng.integers(1, 150)), seed=trial)
        elif fam == 2:
            d = 2 ** int(rng.integers(3, 14))
            tm = skb.SparseRttTM(d, int(rng.integers(1, min(d, 600) + 1)), int(rng.integers(1, 3)), "wht", seed=trial)
        elif fam == 3:
            d0 = int(rng.integers(2, 40))
            tm = skb.KhatriRaoTM(d0, 2, int(rng.integers(1, 300)), "real_rademacher", seed=trial)
        else:
            tm = skb.SparseColTM(int(rng.integers(2, 5000)), int(rng.integers(1, 400)), 2, seed=trial)
        a = torch.randn(n, tm.d, device=cuda, dtype=dt)
        y = tm.apply_right(a).double().cpu().numpy()
        ref = a.double().cpu().numpy() @ tm.materialize()
        tol = 1e-5 if dt == torch.float32 else 1e-12
        assert rel_err(y, ref) <= tol, (trial, type(tm).__name__, n, tm.d, tm.k)


def test_adjoint_and_dense_paths_randomized(cuda):
    """Random shapes / families / dtypes through the adjoint paths (K2g / K2w / K2 / narrow, SRTT TN,
    Khatri-Rao in place, K5d) and the float64 dense families on the DMMA engine (K5d, both tile sizes,
    Khatri-Rao tile synthesis), against the materialized Omega."""
    import torch

    rng = np.random.default_rng(11)
    for trial in range(24):
        dt = torch.float32 if trial % 2 else torch.float64
        fam = trial % 6
        if fam == 0:
            d, k = int(rng.integers(1, 20000)), int(rng.integers(1, 600))
            tm = skb.SparseUniformTM(d, k, int(rng.integers(1, min(k, 8) + 1)), seed=trial)
        elif fam == 1:
            d = 2 ** int(rng.integers(3, 14))
            tm = skb.SparseRttTM(d, int(rng.integers(1, min(d, 400) + 1)), int(rng.integers(1, 3)),
                                 "wht" if trial % 4 < 2 else "dct", seed=trial)
        elif fam == 2:
            d0 = int(rng.integers(2, 60))
            tm = skb.KhatriRaoTM(d0, 2, int(rng.integers(1, 300)), "real_rademacher", seed=trial)
        elif fam == 3:
            tm = skb.GaussianTM(int(rng.integers(1, 3000)), int(rng.integers(1, 300)), seed=trial)
        elif fam == 4:
            tm = skb.KhatriRaoTM(int(rng.integers(2, 12)), 3, int(rng.integers(1, 200)), "real_gaussian", seed=trial)
        else:
            tm = skb.SparseStackTM(int(rng.integers(1, 9000)), int(rng.integers(1, 5)), int(rng.integers(1, 90)),
                                   seed=trial)
        m = int(rng.integers(1, 400))
        b = torch.randn(tm.d, m, device=cuda, dtype=dt)
        x = tm.apply_adjoint(b).double().cpu().numpy()
        om = tm.materialize()
        tol = 1e-5 if dt == torch.float32 else 1e-12
        assert rel_err(x, om.T @ b.double().cpu().numpy()) <= tol, (trial, type(tm).__name__, tm.d, tm.k, m)
        if fam in (2, 3, 4):  # dense-shaped families: the right apply too (float64: K5d)
            n = int(rng.integers(1, 2000))
            a = torch.randn(n, tm.d, device=cuda, dtype=dt)
            y = tm.apply_right(a).double().cpu().numpy()
            assert rel_err(y, a.double().cpu().numpy() @ om) <= tol, (trial, type(tm).__name__, n, tm.d, tm.k)


def test_k1_ring_config1_full_vs_oracle(cuda):
    """BASELINE config 1 in full on the ring kernel (K1r, stream-K over 148 SMs): every one of the
    16384 rows against the oracle (csr_right, 1.3 s on the host), float64 bar 1e-12; and equal to
    the round-1 kernel (SKETCH_B200_K1=classic) to rounding."""
    import os

    import torch

    tm = skb.SparseUniformTM(4096, 256, 4, seed=0)
    assert tm._ring_on(cuda) is not None
    g = torch.Generator(device=cuda).manual_seed(21)
    a = torch.randn(16384, 4096, dtype=torch.float64, device=cuda, generator=g)
    y = tm.apply_right(a).cpu().numpy()
    ref = orc.csr_right(orc.sparse_uniform_csr(4096, 256, 4, 0), a.cpu().numpy())
    assert rel_err(y, ref) <= 1e-12
    os.environ["SKETCH_B200_K1"] = "classic"
    try:
        tm2 = skb.SparseUniformTM(4096, 256, 4, seed=0)
        assert tm2._ring_on(cuda) is None
        y2 = tm2.apply_right(a).cpu().numpy()
    finally:
        del os.environ["SKETCH_B200_K1"]
    assert rel_err(y, y2) <= 1e-14


@pytest.mark.parametrize("n,d,k,zeta", [(1, 64, 256, 4), (63, 100, 17, 3), (65, 4097, 200, 4), (1000, 64, 1, 1),
                                        (3000, 640, 256, 8), (130, 7, 5, 2), (20000, 1000, 64, 4)])
def test_k1_ring_edge_shapes(n, d, k, zeta, cuda):
    """Ragged tiles (n % 64), ragged chunks (d % 64), k < 256, a single CTA, tiles cut between CTAs."""
    import torch

    tm = skb.SparseUniformTM(d, k, zeta, seed=n)
    assert tm._ring_on(cuda) is not None
    rng = np.random.default_rng(n + d)
    a = rng.standard_normal((n, d))
    y = tm.apply_right(torch.from_numpy(a).to(cuda)).cpu().numpy()
    assert rel_err(y, orc.csr_right(orc.sparse_uniform_csr(d, k, zeta, n), a)) <= 1e-12


@pytest.mark.parametrize("n,d,k,zeta", [(700, 16384, 200, 8), (129, 30000, 256, 4), (3000, 9000, 33, 16)])
def test_k1_ring_slabs(n, d, k, zeta, cuda):
    """Omega whose ring lists exceed shared memory runs as a fixed sequence of row slabs (Y =, then Y +=
    per slab): against the oracle at 1e-12, slab count > 1, and a strided A (padded rows)."""
    import torch

    tm = skb.SparseUniformTM(d, k, zeta, seed=d)
    ring = tm._ring_on(cuda)
    assert ring is not None and len(ring[0]) > 1
    widths = [w for _, w, _, _, _ in ring[0]]
    assert sum(widths) == d
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, d))
    ref = orc.csr_right(orc.sparse_uniform_csr(d, k, zeta, d), a)
    y = tm.apply_right(torch.from_numpy(a).to(cuda)).cpu().numpy()
    assert rel_err(y, ref) <= 1e-12
    buf = torch.zeros((n, d + 6), dtype=torch.float64, device=cuda)
    buf[:, 3:3 + d] = torch.from_numpy(a).to(cuda)
    y2 = tm.apply_right(buf[:, 3:3 + d]).cpu().numpy()
    assert rel_err(y2, ref) <= 1e-12


def test_k1_ring_stack_family(cuda):
    import torch

    tm = skb.SparseStackTM(3000, 4, 50, seed=3)
    rng = np.random.default_rng(9)
    a = rng.standard_normal((777, 3000))
    y = tm.apply_right(torch.from_numpy(a).to(cuda)).cpu().numpy()
    assert rel_err(y, orc.csr_right(orc.sparse_stack_csr(3000, 4, 50, 3), a)) <= 1e-12
