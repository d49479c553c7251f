"""Generate golden fixtures by importing the REAL reference package (build container only).

Run from the repo root:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden_small.npz (small Omega arrays + apply outputs) and
tests/golden/golden_hashes.json (sha1 digests of the full-size BASELINE config
test matrices).  /root/reference is not present on the GPU box, so the tests
only ever read these committed outputs.
"""

from __future__ import annotations

import hashlib
import json
import zlib
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from sketchkit.sketch import (  # noqa: E402
    GaussianTM,
    KhatriRaoTM,
    SparseColTM,
    SparseRttTM,
    SparseStackTM,
    SparseUniformTM,
    wht,
)

HERE = os.path.dirname(os.path.abspath(__file__))


def sha1(arr) -> str:
    return hashlib.sha1(np.ascontiguousarray(arr).tobytes()).hexdigest()


def csr_digest(m) -> dict:
    return {
        "indptr": sha1(m.indptr.astype(np.int64)),
        "indices": sha1(m.indices.astype(np.int64)),
        "data": sha1(m.data.astype(np.float64)),
        "nnz": int(m.nnz),
        "shape": list(m.shape),
    }


# small cases: name -> constructor; each records Omega + right/adjoint applies
SMALL = {
    "su_40_12_3_s26": lambda: SparseUniformTM(40, 12, 3, seed=26),
    "su_300_64_4_s1": lambda: SparseUniformTM(300, 64, 4, seed=1),
    "su_1000_200_8_s5": lambda: SparseUniformTM(1000, 200, 8, seed=5),
    "su_4096_256_4_s0_small": lambda: SparseUniformTM(512, 256, 4, seed=0),
    "su_full_row": lambda: SparseUniformTM(6, 4, 4, seed=1),
    "su_perm_path": lambda: SparseUniformTM(50, 10, 9, seed=3),  # acceptance < 5% -> permutation path
    "ss_40_3_4_s23": lambda: SparseStackTM(40, 3, 4, seed=23),
    "ss_500_8_25_s2": lambda: SparseStackTM(500, 8, 25, seed=2),
    "sc_40_12_5_s29": lambda: SparseColTM(40, 12, 5, seed=29),
    "rtt_wht_32_12_4_unif_s31": lambda: SparseRttTM(32, 12, 4, "wht", diagonal="uniform_symmetric", seed=31),
    "rtt_wht_256_64_1_s0": lambda: SparseRttTM(256, 64, 1, "wht", seed=0),
    "rtt_wht_8192_512_1_s0": lambda: SparseRttTM(8192, 512, 1, "wht", seed=0),
    "rtt_dct_40_12_4_s30": lambda: SparseRttTM(40, 12, 4, "dct", seed=30),
    "rtt_dct_512_64_3_s7": lambda: SparseRttTM(512, 64, 3, "dct", seed=7),
    "kr_2_5_9_rad_s33": lambda: KhatriRaoTM(2, 5, 9, "real_rademacher", seed=33),
    "kr_16_2_48_rad_s4": lambda: KhatriRaoTM(16, 2, 48, "real_rademacher", seed=4),
    "kr_8_3_20_gauss_s3": lambda: KhatriRaoTM(8, 3, 20, "real_gaussian", seed=3),
    "gauss_40_12_s21": lambda: GaussianTM(40, 12, "real", 21),
    "gauss_128_32_s9": lambda: GaussianTM(128, 32, "real", 9),
    # complex fields (the reference's default Khatri-Rao base is complex_spherical)
    "kr_16_2_48_csph_s4": lambda: KhatriRaoTM(16, 2, 48, seed=4),
    "kr_8_3_20_cgauss_s3": lambda: KhatriRaoTM(8, 3, 20, "complex_gaussian", seed=3),
    "kr_6_2_70_stein_s8": lambda: KhatriRaoTM(6, 2, 70, "steinhaus", seed=8),
    "gauss_c_128_32_s9": lambda: GaussianTM(128, 32, "complex", 9),
}


def small_fixtures() -> dict:
    out = {}
    for name, make in SMALL.items():
        tm = make()
        rng = np.random.default_rng(zlib.crc32(name.encode()))
        n_rows = 5
        a = rng.standard_normal((n_rows, tm.d))
        b = rng.standard_normal((tm.d, 3))
        out[f"{name}__A"] = a
        out[f"{name}__B"] = b
        out[f"{name}__right"] = tm.apply_right(a)
        out[f"{name}__adjoint"] = tm.apply_adjoint(b)
        out[f"{name}__adjoint_vec"] = tm.apply_adjoint(b[:, 0])
        if tm.d * tm.k <= 100_000:
            out[f"{name}__dense"] = tm.materialize()
        if tm.field == "complex":  # complex inputs too (drawn after the real ones: those stay unchanged)
            ac = a + 1j * rng.standard_normal((n_rows, tm.d))
            bc = b + 1j * rng.standard_normal((tm.d, 3))
            out[f"{name}__Ac"] = ac
            out[f"{name}__Bc"] = bc
            out[f"{name}__right_c"] = tm.apply_right(ac)
            out[f"{name}__adjoint_c"] = tm.apply_adjoint(bc)
        if isinstance(tm, (SparseUniformTM, SparseStackTM, SparseColTM)):
            m = tm.matrix
            out[f"{name}__indptr"] = m.indptr.astype(np.int64)
            out[f"{name}__indices"] = m.indices.astype(np.int64)
            out[f"{name}__data"] = m.data.astype(np.float64)
        if isinstance(tm, SparseRttTM):
            dv, samp = tm._parts()
            out[f"{name}__dvals"] = dv
            out[f"{name}__s_indptr"] = samp.matrix.indptr.astype(np.int64)
            out[f"{name}__s_indices"] = samp.matrix.indices.astype(np.int64)
            out[f"{name}__s_data"] = samp.matrix.data.astype(np.float64)
        if isinstance(tm, KhatriRaoTM):
            out[f"{name}__factors"] = tm.factors
    # known-answer fixtures from the reference tests
    cs = SparseStackTM.from_assignments(signs=[[1.0], [-1.0], [1.0]], buckets=[[0], [1], [0]], block_size=2)
    out["kat_countsketch"] = cs.apply_right(np.array([[1.0, 2.0, 3.0]]))  # test_sketch.py:56-63
    out["kat_kr_column"] = KhatriRaoTM.from_factors(np.array([[[1.0], [1.0]], [[1.0], [-1.0]]])).materialize()[:, 0]
    out["kat_wht_eye8"] = wht(np.eye(8))  # test_transforms.py:18-21
    # downstream drivers: rsvd (rand_nla.py:84-109) and sketch_and_solve (rand_nla.py:278-297)
    from sketchkit.rand_nla import rsvd, sketch_and_solve

    rng = np.random.default_rng(123)
    u0, _ = np.linalg.qr(rng.standard_normal((600, 60)))
    v0, _ = np.linalg.qr(rng.standard_normal((256, 60)))
    a = (u0 * (np.arange(1, 61) ** -2.0)) @ v0.T
    out["rsvd_A"] = a
    for name, tm in (("rsvd_su", SparseUniformTM(256, 40, 8, seed=5)), ("rsvd_rtt", SparseRttTM(256, 40, 1, "wht", seed=6))):
        f = rsvd(a, 40, tm)
        out[f"{name}_sigma"] = f.sigma
        out[f"{name}_recon"] = (f.u * f.sigma) @ f.v.conj().T
    al = rng.standard_normal((3000, 20))
    bl = al @ rng.standard_normal(20) + 1e-3 * rng.standard_normal(3000)
    out["sas_A"] = al
    out["sas_b"] = bl
    out["sas_x"] = sketch_and_solve(al, bl, SparseUniformTM(3000, 200, 8, seed=9))
    # generalized Nystrom (rand_nla.py:191-275) and psd Nystrom (rand_nla.py:152-188); inputs are
    # rebuilt by nystrom_inputs() in the tests, approximations stored as products with probes
    from sketchkit.rand_nla import gen_nystrom_outer, gen_nystrom_svd, nystrom_psd
    from sketchkit.sketch import GaussianTM

    sys.path[:0] = [os.path.dirname(HERE), os.path.dirname(os.path.dirname(HERE))]  # tests/, repo root
    from _cases import nystrom_inputs

    agn, aw, apsd, probe = nystrom_inputs()
    for name, (om, ps) in {
        "gn_su": (SparseUniformTM(300, 20, 4, seed=21), SparseUniformTM(1024, 30, 4, seed=22)),
        "gn_rtt": (SparseRttTM(300, 20, 2, "dct", seed=23), SparseUniformTM(1024, 30, 8, seed=24)),
    }.items():
        fo = gen_nystrom_outer(agn, 20, 30, om, ps)
        out[f"{name}_outer_probe"] = fo.f @ (fo.g.conj().T @ probe[:300])
        fs = gen_nystrom_svd(agn, 20, 30, om, ps)
        out[f"{name}_svd_sigma"] = fs.sigma
        out[f"{name}_svd_probe"] = (fs.u * fs.sigma) @ (fs.v.conj().T @ probe[:300])
    # wide input: processed through the adjoint (rand_nla.py:222-226, 271-273)
    fo = gen_nystrom_outer(aw, 20, 30, SparseUniformTM(256, 20, 4, seed=25), SparseUniformTM(300, 30, 4, seed=26))
    out["gn_wide_outer_probe"] = fo.f @ (fo.g.conj().T @ probe[:256])
    for name, tm in (("nys_su", SparseUniformTM(512, 30, 4, seed=27)), ("nys_gauss", GaussianTM(512, 30, seed=28))):
        fe = nystrom_psd(apsd, 30, tm)
        out[f"{name}_lam"] = fe.lam
        out[f"{name}_probe"] = (fe.u * fe.lam) @ (fe.u.conj().T @ probe)
    return out


def config_hashes() -> dict:
    res = {}
    tm = SparseUniformTM(4096, 256, 4, seed=0)
    res["cfg1_sparseuniform_4096_256_4_s0"] = csr_digest(tm.matrix)
    tm = SparseRttTM(8192, 512, 1, "wht", seed=0)
    dv, samp = tm._parts()
    res["cfg2_srtt_wht_8192_512_1_s0"] = {"dvals": sha1(dv.astype(np.float64)), "sampler": csr_digest(samp.matrix),
                                          "distinct_rows": int(np.unique(samp.matrix.tocoo().row).size)}
    tm = SparseUniformTM(16384, 200, 8, seed=0)
    res["cfg3_sparseuniform_16384_200_8_s0"] = csr_digest(tm.matrix)
    tm = SparseUniformTM(4194304, 2048, 8, seed=0)
    res["cfg4_sparseuniform_4194304_2048_8_s0"] = csr_digest(tm.matrix)
    tm = KhatriRaoTM(256, 2, 512, "real_rademacher", seed=0)
    res["cfg5_khatrirao_256_2_512_rad_s0"] = {"factors": sha1(tm.factors.astype(np.float64))}
    return res


if __name__ == "__main__":
    small = small_fixtures()
    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **small)
    hashes = config_hashes()
    hashes["_generator"] = "tests/golden/make_golden.py against /root/reference sketchkit 0.1.0, numpy " + np.__version__
    with open(os.path.join(HERE, "golden_hashes.json"), "w") as f:
        json.dump(hashes, f, indent=1, sort_keys=True)
    print("wrote", len(small), "small arrays and", len(hashes) - 1, "config digests")
