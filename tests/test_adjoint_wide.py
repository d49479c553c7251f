"""K2w (register-accumulator float32 adjoint): host encoder layout (CPU) and GPU parity."""

import ctypes

import numpy as np
import pytest

import oracle as orc
from _cases import rel_err
from paper_2508_21189_b200 import _lib
from paper_2508_21189_b200 import sketch as skb

R, CG, CPW, WARPS, HDR = 128, 256, 16, 16, 24


def _encode(d, k, rows, cols, neg):
    lib = _lib.load()
    rows = np.ascontiguousarray(rows, np.int64)
    cols = np.ascontiguousarray(cols, np.int64)
    neg = np.ascontiguousarray(neg, np.uint8)
    nseg1 = lib.sk_sparse_adjoint_wide_segments(d, k)
    seg = np.zeros(nseg1, np.int64)
    cap = ctypes.c_int32(0)
    args = (d, k, rows.size, rows.ctypes.data, cols.ctypes.data, neg.ctypes.data)
    total = lib.sk_sparse_adjoint_wide_encode(*args, None, 0, seg.ctypes.data, ctypes.byref(cap))
    enc = np.zeros(total, np.uint16)
    assert lib.sk_sparse_adjoint_wide_encode(*args, enc.ctypes.data, enc.size, seg.ctypes.data,
                                             ctypes.byref(cap)) == total
    return enc, seg, cap.value


@pytest.mark.parametrize("d,k,zeta", [(1000, 300, 5), (300, 1100, 3), (129, 64, 1)])
def test_encoder_roundtrip(d, k, zeta):
    """Decoding every segment gives back exactly the (row, col, sign) triplets of Omega."""
    tm = skb.SparseUniformTM(d, k, zeta, seed=2)
    rows, cols, neg, _ = tm._sign_form()
    enc, seg, cap = _encode(d, k, rows, cols, neg)
    ngroups = -(-k // CG)
    got = []
    for sg in range(seg.size - 1):
        s = enc[seg[sg]:seg[sg + 1]]
        assert s.size % 8 == 0 and s.size <= cap
        h = s[:WARPS + 1]
        assert np.all(h % 4 == 0) and np.all(np.diff(h.astype(int)) >= 0)
        chunk, g = divmod(sg, ngroups)
        for w in range(WARPS):
            for u in s[HDR + h[w]:HDR + h[w + 1]]:
                u = int(u)
                if u == 32:  # padding no-op
                    continue
                got.append((chunk * R + (u >> 9), g * CG + w * CPW + (u & 15), (u >> 4) & 1))
    want = sorted(zip(rows.tolist(), cols.tolist(), neg.astype(int).tolist()))
    assert sorted(got) == want


def test_encoder_rejects_bad_indices():
    lib = _lib.load()
    rows = np.array([0, 5], np.int64)
    cols = np.array([0, 70], np.int64)
    neg = np.zeros(2, np.uint8)
    seg = np.zeros(lib.sk_sparse_adjoint_wide_segments(4, 64), np.int64)
    cap = ctypes.c_int32(0)
    st = lib.sk_sparse_adjoint_wide_encode(4, 64, 2, rows.ctypes.data, cols.ctypes.data, neg.ctypes.data, None, 0,
                                           seg.ctypes.data, ctypes.byref(cap))
    assert st == _lib.SK_EINVAL


@pytest.mark.gpu
@pytest.mark.parametrize("d,k,zeta,m", [(4096, 2048, 8, 512), (20000, 1300, 8, 100), (1000, 300, 5, 4),
                                        (129, 513, 3, 64), (70000, 2048, 8, 68)])
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_wide_vs_oracle(d, k, zeta, m, dt, cuda, monkeypatch):
    import torch

    monkeypatch.setenv("SKETCH_B200_SPARSE_ADJOINT", "wide")
    tm = skb.SparseUniformTM(d, k, zeta, seed=7)
    rng = np.random.default_rng(d + m)
    b = rng.standard_normal((d, m)).astype(dt)
    bt = torch.as_tensor(b).to(cuda)
    if m % 2 == 0 or dt == np.float32:
        assert tm.adjoint_path(bt) == "wide"
    y = tm.apply_adjoint(bt).cpu().numpy()
    ref = orc.csr_adjoint(orc.sparse_uniform_csr(d, k, zeta, 7), b)
    assert rel_err(y, ref) <= (1e-5 if dt == np.float32 else 1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("path", ["wide", "rowgather"])
def test_wide_variable_row_counts(path, cuda, monkeypatch):
    """SparseIID: rows carry 0..many nonzeros (K2w pads each warp list independently; K2g lists
    have any length per target row)."""
    import torch

    monkeypatch.setenv("SKETCH_B200_SPARSE_ADJOINT", path)
    tm = skb.SparseIIDTM(3000, 700, 6.0, seed=3)
    b = torch.randn(3000, 96, device=cuda)
    assert tm.adjoint_path(b) == path
    ref = tm.materialize().T @ b.cpu().double().numpy()
    assert rel_err(tm.apply_adjoint(b).cpu().numpy(), ref) <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_wide_matches_gather_path(dtype, cuda, monkeypatch):
    import torch

    tm = skb.SparseStackTM(8192, 8, 64, seed=1)
    b = torch.randn(8192, 256, device=cuda, dtype=getattr(torch, dtype))
    assert tm.adjoint_path(b) == "rowgather"
    rowg = tm.apply_adjoint(b).double()
    monkeypatch.setenv("SKETCH_B200_SPARSE_ADJOINT", "wide")
    assert tm.adjoint_path(b) == "wide"
    wide = tm.apply_adjoint(b).double()
    assert float((wide - rowg).norm() / rowg.norm()) <= (1e-6 if dtype == "float32" else 1e-14)
    monkeypatch.setenv("SKETCH_B200_SPARSE_ADJOINT", "gather")
    assert tm.adjoint_path(b) == "gather"
    gather = tm.apply_adjoint(b).double()
    assert float((wide - gather).norm() / gather.norm()) <= (1e-6 if dtype == "float32" else 1e-14)


@pytest.mark.parametrize("d,k,zeta", [(1000, 300, 5), (300, 1100, 3), (129, 64, 1), (5000, 2048, 8)])
def test_device_encoder_matches_host(d, k, zeta):
    """wide_encode_device (torch ops; run here on CPU tensors) produces the host encoder's bytes."""
    import torch

    from paper_2508_21189_b200.sketch.encode import wide_encode_device

    tm = skb.SparseUniformTM(d, k, zeta, seed=4)
    rows, cols, neg, _ = tm._sign_form()
    assert np.array_equal(rows, np.repeat(np.arange(d), zeta))
    enc, seg, cap = _encode(d, k, rows, cols, neg)
    e2, s2, c2 = wide_encode_device(torch.from_numpy(cols.reshape(d, zeta)), torch.from_numpy(neg.reshape(d, zeta)),
                                    zeta, d, k)
    assert c2 == cap
    assert np.array_equal(s2.numpy(), seg)
    assert np.array_equal(e2.numpy().view(np.uint16), enc)


@pytest.mark.gpu
def test_device_encoding_on_gpu(cuda, monkeypatch):
    """Device-drawn operator: the adjoint builds its K2w encoding on the GPU without a host copy
    of the draws, byte-identical to the host encoder, and matches the oracle."""
    import torch

    monkeypatch.setenv("SKETCH_B200_SPARSE_ADJOINT", "wide")
    d, k, zeta, m = 200003, 2048, 8, 40
    tm = skb.SparseUniformTM(d, k, zeta, seed=12)
    b = torch.randn(d, m, device=cuda)
    y = tm.apply_adjoint(b)
    assert tm._coo is None  # draws stayed on the device
    enc_dev, seg_dev, cap_dev, _ = tm._adjoint_wide_on(b.device)
    rows, cols, neg, _ = tm._sign_form()
    enc, seg, cap = _encode(d, k, rows, cols, neg)
    assert cap_dev == cap and np.array_equal(seg_dev.cpu().numpy(), seg)
    assert np.array_equal(enc_dev.cpu().numpy().view(np.uint16), enc)
    ref = orc.csr_adjoint(orc.sparse_uniform_csr(d, k, zeta, 12), b.cpu().double().numpy())
    assert rel_err(y.cpu().numpy(), ref) <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("d,k,zeta,m", [(70000, 2048, 8, 68), (1000, 300, 5, 512), (129, 513, 3, 260),
                                        (40000, 64, 2, 1000)])
def test_rowgather_vs_oracle(d, k, zeta, m, dt, cuda, monkeypatch):
    """K2g (TMA row gathers, one warp per target row / column block / row piece) against the oracle."""
    import torch

    monkeypatch.setenv("SKETCH_B200_SPARSE_ADJOINT", "rowgather")
    tm = skb.SparseUniformTM(d, k, zeta, seed=7)
    rng = np.random.default_rng(d + m)
    b = rng.standard_normal((d, m)).astype(dt)
    bt = torch.as_tensor(b).to(cuda)
    assert tm.adjoint_path(bt) == "rowgather"
    y = tm.apply_adjoint(bt).cpu().numpy()
    ref = orc.csr_adjoint(orc.sparse_uniform_csr(d, k, zeta, 7), b)
    assert rel_err(y, ref) <= (1e-5 if dt == np.float32 else 1e-12)


@pytest.mark.gpu
def test_adjoint_paths_randomized(cuda):
    """Random shapes, families and dtypes through the default adjoint path (K2g when aligned,
    K2 otherwise) against the materialized Omega."""
    import torch

    rng = np.random.default_rng(2024)
    for trial in range(24):
        d = int(rng.integers(1, 60000))
        k = int(rng.integers(1, 2600))
        m = int(rng.integers(1, 700))
        dt = torch.float32 if trial % 2 else torch.float64
        fam = trial % 4
        if fam == 0:
            tm = skb.SparseUniformTM(d, k, int(rng.integers(1, min(k, 8) + 1)), seed=trial)
        elif fam == 1:
            z = int(rng.integers(1, 5))
            tm = skb.SparseStackTM(d, z, max(1, k // z), seed=trial)
        elif fam == 2:
            tm = skb.SparseIIDTM(d, k, float(rng.uniform(0.5, min(k, 6))), seed=trial)
        else:
            tm = skb.SparseColTM(d, k, int(rng.integers(1, min(d, 4) + 1)), seed=trial)
        b = torch.randn(d, m, device=cuda, dtype=dt)
        y = tm.apply_adjoint(b).double().cpu().numpy()
        om = tm.materialize()
        ref = om.T @ b.double().cpu().numpy()
        tol = 1e-5 if dt == torch.float32 else 1e-12
        assert rel_err(y, ref) <= tol, (trial, type(tm).__name__, d, tm.k, m, tm.adjoint_path(b))


@pytest.mark.gpu
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_narrow_adjoint(dt, cuda):
    """m <= 8 columns (right-hand sides): warp per target row over the K2g encoding."""
    import torch

    tm = skb.SparseUniformTM(50003, 700, 5, seed=9)
    om = orc.sparse_uniform_csr(50003, 700, 5, 9)
    rng = np.random.default_rng(1)
    tol = 1e-5 if dt == np.float32 else 1e-12
    for m in (1, 3, 8):
        b = rng.standard_normal((50003, m)).astype(dt)
        bt = torch.as_tensor(b).to(cuda)
        assert tm.adjoint_path(bt) == "narrow"
        assert rel_err(tm.apply_adjoint(bt).cpu().numpy(), orc.csr_adjoint(om, b)) <= tol
    # 1-D vector (squeezed back), and a strided row view
    v = rng.standard_normal(50003).astype(dt)
    got = tm.apply_adjoint(torch.as_tensor(v).to(cuda))
    assert tuple(got.shape) == (700,)
    assert rel_err(got.cpu().numpy(), orc.csr_adjoint(om, v[:, None])[:, 0]) <= tol
    big = torch.as_tensor(rng.standard_normal((50003, 10)).astype(dt)).to(cuda)
    sl = big[:, 2:6]
    assert tm.adjoint_path(sl) == "narrow"
    assert rel_err(tm.apply_adjoint(sl).cpu().numpy(), orc.csr_adjoint(om, sl.cpu().numpy())) <= tol
