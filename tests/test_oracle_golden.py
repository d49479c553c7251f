"""Pin the CPU oracle (oracle/) against golden vectors produced by the REAL reference.

Golden data: tests/golden/make_golden.py imported /root/reference/pkg/src/sketchkit and recorded
small test matrices, their applies on seeded inputs, the known-answer fixtures of the reference
tests, and sha1 digests of the full-size BASELINE config test matrices.
"""

import hashlib

import numpy as np
import pytest

import oracle as orc
from _cases import CASES, oracle_dense, oracle_right, rel_err


def sha1(a):
    return hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_right_matches_reference(name, golden):
    a = golden[f"{name}__A"]
    assert rel_err(oracle_right(name, a), golden[f"{name}__right"]) <= 1e-13


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_dense_matches_reference(name, golden):
    key = f"{name}__dense"
    if key not in golden:
        pytest.skip("no dense fixture at this size")
    assert rel_err(oracle_dense(name), golden[key]) <= 1e-13


@pytest.mark.parametrize("name", [n for n, (f, _) in CASES.items() if f in ("su", "ss", "sc")])
def test_oracle_csr_bit_exact(name, golden):
    fam, p = CASES[name]
    m = {"su": lambda: orc.sparse_uniform_csr(p["d"], p["k"], p["zeta"], p["seed"]),
         "ss": lambda: orc.sparse_stack_csr(p["d"], p["zeta"], p["block"], p["seed"]),
         "sc": lambda: orc.sparse_col_csr(p["d"], p["k"], p["xi"], p["seed"])}[fam]()
    assert np.array_equal(m.indptr.astype(np.int64), golden[f"{name}__indptr"])
    assert np.array_equal(m.indices.astype(np.int64), golden[f"{name}__indices"])
    assert np.array_equal(m.data, golden[f"{name}__data"])


def test_oracle_known_answers(golden):
    # reference pkg/tests/test_sketch.py:56-63 (CountSketch worked example)
    m = orc.stack_from_assignments([[1.0], [-1.0], [1.0]], [[0], [1], [0]], 2)
    assert np.allclose(orc.csr_right(m, np.array([[1.0, 2.0, 3.0]])), golden["kat_countsketch"])
    assert np.allclose(golden["kat_countsketch"], [[4.0, -2.0]])
    # reference pkg/tests/test_transforms.py:18-21 (WHT == H8 / sqrt 8)
    assert np.allclose(orc.wht_rows(np.eye(8)).T, golden["kat_wht_eye8"])
    # reference pkg/tests/test_sketch.py:172-176 (explicit Kronecker column)
    f = np.array([[[1.0], [1.0]], [[1.0], [-1.0]]])
    col = orc.kr_right(f, np.eye(4))[:, 0] * np.sqrt(1)
    assert np.allclose(col, golden["kat_kr_column"])


def test_oracle_config_hashes_small(golden_hashes):
    h = golden_hashes["cfg1_sparseuniform_4096_256_4_s0"]
    m = orc.sparse_uniform_csr(4096, 256, 4, 0)
    assert sha1(m.indices.astype(np.int64)) == h["indices"]
    assert sha1(m.data) == h["data"]
    h = golden_hashes["cfg2_srtt_wht_8192_512_1_s0"]
    dv, samp = orc.srtt_parts(8192, 512, 1, 0)
    assert sha1(dv) == h["dvals"]
    assert sha1(samp.indices.astype(np.int64)) == h["sampler"]["indices"]
    assert sha1(samp.data) == h["sampler"]["data"]
    assert np.unique(samp.tocoo().row).size == h["distinct_rows"] == 490
    h = golden_hashes["cfg3_sparseuniform_16384_200_8_s0"]
    m = orc.sparse_uniform_csr(16384, 200, 8, 0)
    assert sha1(m.indices.astype(np.int64)) == h["indices"]
    h = golden_hashes["cfg5_khatrirao_256_2_512_rad_s0"]
    assert sha1(orc.kr_factors(256, 2, 512, 0)) == h["factors"]


@pytest.mark.slow
def test_oracle_config4_hash(golden_hashes):
    h = golden_hashes["cfg4_sparseuniform_4194304_2048_8_s0"]
    m = orc.sparse_uniform_csr(4194304, 2048, 8, 0)
    assert sha1(m.indices.astype(np.int64)) == h["indices"]
    assert sha1(m.data) == h["data"]


def test_oracle_drivers_match_reference(golden):
    a = golden["rsvd_A"]
    for name, om in (("rsvd_su", lambda x: orc.csr_right(orc.sparse_uniform_csr(256, 40, 8, 5), x)),
                     ("rsvd_rtt", lambda x: orc.srtt_right(*orc.srtt_parts(256, 40, 1, 6), x, "wht"))):
        u, s, v = orc.rsvd(a, om, 40)
        assert np.allclose(s, golden[f"{name}_sigma"], rtol=1e-10, atol=1e-15)
        assert rel_err((u * s) @ v.T, golden[f"{name}_recon"]) <= 1e-10
    om = orc.sparse_uniform_csr(3000, 200, 8, 9)
    x = orc.sketch_and_solve(golden["sas_A"], golden["sas_b"], lambda b: orc.csr_adjoint(om, b))
    assert rel_err(x, golden["sas_x"]) <= 1e-10
