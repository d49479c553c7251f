"""CPU tests of the product's host logic: bit-exact test matrices, encodings, RNG, no-CPU-fallback."""

import hashlib

import numpy as np
import pytest

import oracle as orc
from _cases import CASES, product, rel_err
from paper_2508_21189_b200 import RngStream, derive_seed
from paper_2508_21189_b200 import sketch as skb
from paper_2508_21189_b200.rng import entropy_of
from paper_2508_21189_b200.sketch.encode import bcsc_decode, bcsc_encode, sign_bits, srtt_sampler_encode


def sha1(a):
    return hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", [n for n, (f, _) in CASES.items() if f in ("su", "ss", "sc")])
def test_product_csr_bit_exact(name, golden):
    m = product(name).matrix
    assert np.array_equal(m.indptr.astype(np.int64), golden[f"{name}__indptr"])
    assert np.array_equal(m.indices.astype(np.int64), golden[f"{name}__indices"])
    assert np.array_equal(m.data, golden[f"{name}__data"])


@pytest.mark.parametrize("name", sorted(CASES))
def test_product_materialize_matches_reference(name, golden):
    key = f"{name}__dense"
    if key not in golden:
        pytest.skip("no dense fixture")
    assert rel_err(product(name).materialize(), golden[key]) <= 1e-13


@pytest.mark.parametrize("name", [n for n, (f, _) in CASES.items() if f == "rtt"])
def test_product_srtt_parts_bit_exact(name, golden):
    dv, samp = product(name)._parts()
    assert np.array_equal(dv, golden[f"{name}__dvals"])
    assert np.array_equal(samp.matrix.indices.astype(np.int64), golden[f"{name}__s_indices"])
    assert np.array_equal(samp.matrix.data, golden[f"{name}__s_data"])


@pytest.mark.parametrize("name", [n for n, (f, _) in CASES.items() if f == "kr"])
def test_product_kr_factors_bit_exact(name, golden):
    assert np.array_equal(product(name).factors, golden[f"{name}__factors"])


def test_config_test_matrices_bit_exact(golden_hashes):
    h = golden_hashes["cfg1_sparseuniform_4096_256_4_s0"]
    m = skb.SparseUniformTM(4096, 256, 4, seed=0).matrix
    assert (sha1(m.indices.astype(np.int64)), sha1(m.data), sha1(m.indptr.astype(np.int64))) == (
        h["indices"], h["data"], h["indptr"])
    h = golden_hashes["cfg2_srtt_wht_8192_512_1_s0"]
    tm = skb.SparseRttTM(8192, 512, 1, "wht", seed=0)
    dv, samp = tm._parts()
    assert sha1(dv) == h["dvals"]
    assert sha1(samp.matrix.indices.astype(np.int64)) == h["sampler"]["indices"]
    assert sha1(samp.matrix.data) == h["sampler"]["data"]
    h = golden_hashes["cfg3_sparseuniform_16384_200_8_s0"]
    m = skb.SparseUniformTM(16384, 200, 8, seed=0).matrix
    assert sha1(m.indices.astype(np.int64)) == h["indices"]
    assert sha1(m.data) == h["data"]
    h = golden_hashes["cfg5_khatrirao_256_2_512_rad_s0"]
    assert sha1(skb.KhatriRaoTM(256, 2, 512, "real_rademacher", seed=0).factors) == h["factors"]


@pytest.mark.slow
def test_config4_test_matrix_bit_exact(golden_hashes):
    h = golden_hashes["cfg4_sparseuniform_4194304_2048_8_s0"]
    rows, cols, vals = skb.SparseUniformTM(4194304, 2048, 8, seed=0)._triplets()
    assert sha1(cols) == h["indices"]
    assert sha1(vals) == h["data"]


def test_countsketch_fixture_structure():
    tm = skb.SparseStackTM.from_assignments([[1.0], [-1.0], [1.0]], [[0], [1], [0]], 2)
    assert np.allclose(tm.materialize(), [[1, 0], [0, -1], [1, 0]])


def test_stack_structure_forced():
    # reference pkg/tests/test_sketch.py:39-48
    tm = skb.SparseStackTM(30, zeta=4, block_size=5, seed=3)
    m = tm.matrix
    assert np.all(np.diff(m.indptr) == 4)
    assert np.all(m.indices.reshape(30, 4) // 5 == np.arange(4))
    assert np.allclose(np.abs(m.data), 0.5)


def test_constructor_errors():
    with pytest.raises(ValueError, match="divisible"):
        skb.SparseStackTM(10, zeta=3, k=10)
    with pytest.raises(ValueError, match="power-of-two"):
        skb.SparseRttTM(48, 8, 3, "wht")
    with pytest.raises(ValueError, match="complex"):
        skb.SparseRttTM(16, 8, 3, "dft", field="real")
    assert skb.SparseRttTM(256, 64, seed=0).xi == int(np.ceil(1.5 * np.log(64)))
    assert skb.SparseRttTM(20, 8, 3, seed=0).transform == "dct"


def test_rng_stream_contract():
    a = RngStream(7).substream("x", 3).generator().standard_normal(8)
    b = RngStream(7).substream("x", 3).generator().standard_normal(8)
    c = RngStream(7).substream("x", 4).generator().standard_normal(8)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert derive_seed(3, "a", 5) == derive_seed(3, "a", 5) != derive_seed(3, "a", 6)
    # entropy for seed 0, path (SparseUniformTM, entries)
    ent = entropy_of(0, ("SparseUniformTM", "entries"))
    assert ent[:2] == [0, 0] and ent[3:5] == [15, 2] and ent[6:] == [7, 2]
    assert ent[2] == int.from_bytes(b"SparseUniformTM", "little")
    g1 = RngStream(0, ("SparseUniformTM", "entries")).generator()
    g2 = orc.stream(0, "SparseUniformTM", "entries")
    assert np.array_equal(g1.integers(0, 100, 50), g2.integers(0, 100, 50))


@pytest.mark.parametrize("d,k,zeta,r", [(40, 12, 3, 32), (1000, 200, 8, 256), (4096, 256, 4, 512), (70, 5, 5, 64)])
def test_bcsc_roundtrip(d, k, zeta, r):
    tm = skb.SparseUniformTM(d, k, zeta, seed=d)
    rows, cols, neg, mag = tm._sign_form()
    ptr, ent = bcsc_encode(rows, cols, neg, d, k, r)
    assert ptr[-1] == rows.size and ptr.dtype == np.int32 and ent.dtype == np.uint16
    r2, c2, n2 = bcsc_decode(ptr, ent, d, k, r)
    want = sorted(zip(rows.tolist(), cols.tolist(), neg.tolist()))
    assert sorted(zip(r2.tolist(), c2.tolist(), n2.tolist())) == want
    # within each (chunk, column) list rows ascend
    keys = (r2 // r) * k + c2
    same = keys[1:] == keys[:-1]
    assert np.all(r2[1:][same] > r2[:-1][same])
    dense = np.zeros((d, k))
    np.add.at(dense, (r2, c2), np.where(n2, -mag, mag))
    assert np.array_equal(dense, tm.materialize())


def test_srtt_sampler_and_sign_bits():
    rows = np.array([[5], [0], [7]])
    neg = np.array([[True], [False], [True]])
    e = srtt_sampler_encode(rows, neg).view(np.uint32)
    assert list(e & 0x7FFFFFFF) == [5, 0, 7] and list(e >> 31) == [1, 0, 1]
    bits = sign_bits(np.arange(70) % 3 == 0)
    assert bits.size == 3 and all(((bits[i // 32] >> (i % 32)) & 1) == (i % 3 == 0) for i in range(70))


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2508_21189_b200._device import NoDeviceError

    tm = skb.SparseUniformTM(40, 12, 3, seed=0)
    with pytest.raises(NoDeviceError):
        tm.apply_right(np.ones((2, 40)))
    with pytest.raises(NoDeviceError):
        tm.apply_adjoint(np.ones(40))


def test_shape_errors_precede_device():
    # reference pkg/tests/test_sketch.py:260-265 (error texts mention the method)
    tm = skb.GaussianTM(10, 4, seed=0)
    with pytest.raises(ValueError, match="apply_right"):
        tm.apply_right(np.ones((3, 9)))
    with pytest.raises(ValueError, match="apply_adjoint"):
        tm.apply_adjoint(np.ones((9, 2)))


def test_bcsc_segments():
    from paper_2508_21189_b200.sketch.encode import bcsc_segments

    d, k, r = 3000, 2100, 512
    tm = skb.SparseUniformTM(d, k, 8, seed=2)
    rows, cols, neg, _ = tm._sign_form()
    ptr, ent = bcsc_encode(rows, cols, neg, d, k, r)
    seg, cap = bcsc_segments(ptr, d, k, r, group=1024)
    seg = seg.reshape(-1, 3, 2)
    for h in range(seg.shape[0]):
        for g in range(3):
            e0, cnt = seg[h, g]
            lo, hi = ptr[h * k + g * 1024], ptr[h * k + min(k, (g + 1) * 1024)]
            assert e0 % 8 == 0 and cnt % 8 == 0 and e0 <= lo and e0 + cnt >= hi and cnt <= cap


def test_redraw_determinism():
    """redraw(seed) is the same operator as a fresh construction with that seed, every family
    (reference pkg/tests/test_sketch.py:82-85 checks the same contract)."""
    fams = [skb.SparseUniformTM(64, 12, 3, seed=1), skb.SparseStackTM(64, 3, 5, seed=1),
            skb.SparseIIDTM(64, 12, 2.0, seed=1), skb.SparseColTM(64, 12, 2, seed=1),
            skb.SparseRttTM(64, 12, 2, "wht", seed=1), skb.SparseRttTM(64, 12, 2, "dct", seed=1),
            skb.KhatriRaoTM(4, 3, 12, "real_rademacher", seed=1), skb.GaussianTM(64, 12, seed=1)]
    for tm in fams:
        a, b = tm.redraw(7), tm.redraw(7)
        assert type(a) is type(tm) and (a.d, a.k) == (tm.d, tm.k) and a.seed == 7
        assert np.array_equal(a.materialize(), b.materialize())
        assert not np.array_equal(a.materialize(), tm.materialize())
        assert np.array_equal(tm.materialize(), tm.materialize())


def test_row_blocks_cached_and_partition_rows():
    """Row blocks of a sparse operator (multi-GPU shards) are cached per parent and their rows
    concatenate to the parent's matrix exactly."""
    tm = skb.SparseUniformTM(300, 40, 5, seed=3)
    blocks = [tm.row_block(0, 128), tm.row_block(128, 300)]
    assert tm.row_block(0, 128) is blocks[0] and tm.row_block(128, 300) is blocks[1]
    assert blocks[0].row_offset == 0 and blocks[1].row_offset == 128
    full = tm.materialize()
    assert np.array_equal(np.vstack([b.materialize() for b in blocks]), full)
    assert tm.redraw(3).row_block(0, 128) is not blocks[0]


@pytest.mark.parametrize("d0,ell,k,base", [(256, 2, 512, "real_rademacher"), (16, 2, 48, "real_rademacher"),
                                           (8, 3, 20, "real_gaussian"), (4, 4, 60, "real_rademacher"),
                                           (5, 2, 7, "real_spherical"), (2, 5, 9, "real_rademacher")])
def test_kr_factor_split_reproduces_omega(d0, ell, k, base):
    """The device operands of the Khatri-Rao kernels: Omega[P*dl + q, j] = W[P, j] F[q, j] exactly
    (W, F = Khatri-Rao products of the leading / trailing factors; Omega itself is never formed)."""
    tm = skb.KhatriRaoTM(d0, ell, k, base, seed=3)
    om = tm.materialize()
    for tensor_cores in (True, False):
        g = tm._kr_group(tensor_cores) or 1
        w, f = tm._kr_split_arrays(g)
        assert w.shape == (d0 ** (ell - g), k) and f.shape == (d0 ** g, k)
        np.testing.assert_allclose((w[:, None, :] * f[None, :, :]).reshape(-1, k) / np.sqrt(k), om, rtol=1e-15,
                                   atol=0)  # products regrouped: exact for +-1, 1 ulp otherwise
    if (d0, ell) == (256, 2):
        assert tm._kr_group(True) == 1  # config 5: F = factor 1, W = factor 0 (no Kronecker columns formed)


@pytest.mark.parametrize("d,k,zeta", [(4096, 256, 4), (100, 17, 3), (4097, 200, 8), (7, 5, 2)])
def test_ring_encode_roundtrip(d, k, zeta):
    """K1r's per-(chunk, warp) segments decode back to exactly Omega's (row, column, sign) triplets."""
    from paper_2508_21189_b200.sketch.encode import ring_decode, ring_encode

    coo = orc.sparse_uniform_csr(d, k, zeta, 5).tocoo()
    lists, seg = ring_encode(coo.row, coo.col, coo.data < 0, d, k)
    assert lists.size == int(seg[-1]) * 16 and seg.size == ((d + 127) // 128) * 16 + 1
    r, c, n = ring_decode(lists, seg, d, k)
    assert sorted(zip(coo.row.tolist(), coo.col.tolist(), (coo.data < 0).tolist())) == \
        sorted(zip(r.tolist(), c.tolist(), n.tolist()))


@pytest.mark.parametrize("d,k,zeta", [(16384, 200, 8), (30000, 256, 4), (4096, 256, 4)])
def test_ring_slabs_partition_omega(d, k, zeta):
    """K1r row slabs (wide Omega): widths tile [0, d) on 128-row unit boundaries, every slab's lists
    fit shared memory (the library's own check, no device needed), and the slabs' lists, decoded with
    slab-local rows, are exactly Omega's triplets."""
    from paper_2508_21189_b200 import _lib
    from paper_2508_21189_b200.sketch.encode import ring_decode

    tm = skb.SparseUniformTM(d, k, zeta, seed=d)
    rows, cols, neg, _ = tm._sign_form()
    from paper_2508_21189_b200.sketch.encode import ring_encode

    lists, seg = ring_encode(rows, cols, neg, d, k)
    slabs = tm._ring_slabs(lists, seg, "cpu")
    assert slabs is not None
    lib = _lib.load()
    got = []
    s_expect = 0
    for s0, width, sl, sg, nbytes in slabs:
        assert s0 == s_expect and s0 % 128 == 0 and width > 0
        s_expect = s0 + width
        assert lib.sk_sparse_right_ring_supported(_lib.SK_F64, width, k, nbytes)
        r, c, n = ring_decode(sl.numpy(), sg.numpy().view(np.uint32), width, k)
        got += list(zip((r + s0).tolist(), c.tolist(), n.tolist()))
    assert s_expect == d
    assert (len(slabs) > 1) == (d > 4096)
    assert sorted(got) == sorted(zip(rows.tolist(), cols.tolist(), neg.astype(bool).tolist()))


@pytest.mark.parametrize("name,make", [
    ("kr_16_2_48_csph_s4", lambda: skb.KhatriRaoTM(16, 2, 48, seed=4)),
    ("kr_8_3_20_cgauss_s3", lambda: skb.KhatriRaoTM(8, 3, 20, "complex_gaussian", seed=3)),
    ("kr_6_2_70_stein_s8", lambda: skb.KhatriRaoTM(6, 2, 70, "steinhaus", seed=8)),
    ("gauss_c_128_32_s9", lambda: skb.GaussianTM(128, 32, "complex", 9))])
def test_complex_fields_match_reference(name, make, golden):
    """Complex-field constructors (the reference's default Khatri-Rao base is complex_spherical):
    factors bit-exact and Omega equal to the reference's; the planes the DMMA engine reads rebuild it."""
    from paper_2508_21189_b200.sketch.zplanes import z_operands

    tm = make()
    if f"{name}__factors" in golden:
        assert np.array_equal(tm.factors, golden[f"{name}__factors"])
    assert rel_err(tm.materialize(), golden[f"{name}__dense"]) <= 1e-13
    if isinstance(tm, skb.KhatriRaoTM):
        w, f = tm._kr_split_arrays(tm._kr_group(False))
        ops = z_operands(None if w.shape[0] == 1 else w, f, "cpu")
        fz = ops.fr[:, :tm.k].numpy() + 1j * ops.fi[:, :tm.k].numpy()
        wz = np.ones((1, tm.k)) if ops.wr is None else ops.wr[:, :tm.k].numpy() + 1j * ops.wi[:, :tm.k].numpy()
        om = (wz[:, None, :] * fz[None, :, :]).reshape(-1, tm.k) / np.sqrt(tm.k)
        assert rel_err(om, golden[f"{name}__dense"]) <= 1e-13
