"""Shared case table: golden fixture name -> oracle construction and product construction."""

from __future__ import annotations

import numpy as np

import oracle as orc  # noqa: E402
from paper_2508_21189_b200 import sketch as skb

# name -> (family, params); keep in sync with tests/golden/make_golden.py SMALL
CASES = {
    "su_40_12_3_s26": ("su", dict(d=40, k=12, zeta=3, seed=26)),
    "su_300_64_4_s1": ("su", dict(d=300, k=64, zeta=4, seed=1)),
    "su_1000_200_8_s5": ("su", dict(d=1000, k=200, zeta=8, seed=5)),
    "su_4096_256_4_s0_small": ("su", dict(d=512, k=256, zeta=4, seed=0)),
    "su_full_row": ("su", dict(d=6, k=4, zeta=4, seed=1)),
    "su_perm_path": ("su", dict(d=50, k=10, zeta=9, seed=3)),
    "ss_40_3_4_s23": ("ss", dict(d=40, zeta=3, block=4, seed=23)),
    "ss_500_8_25_s2": ("ss", dict(d=500, zeta=8, block=25, seed=2)),
    "sc_40_12_5_s29": ("sc", dict(d=40, k=12, xi=5, seed=29)),
    "rtt_wht_32_12_4_unif_s31": ("rtt", dict(d=32, k=12, xi=4, transform="wht", diagonal="uniform_symmetric", seed=31)),
    "rtt_wht_256_64_1_s0": ("rtt", dict(d=256, k=64, xi=1, transform="wht", diagonal="real_rademacher", seed=0)),
    "rtt_wht_8192_512_1_s0": ("rtt", dict(d=8192, k=512, xi=1, transform="wht", diagonal="real_rademacher", seed=0)),
    "rtt_dct_40_12_4_s30": ("rtt", dict(d=40, k=12, xi=4, transform="dct", diagonal="real_rademacher", seed=30)),
    "rtt_dct_512_64_3_s7": ("rtt", dict(d=512, k=64, xi=3, transform="dct", diagonal="real_rademacher", seed=7)),
    "kr_2_5_9_rad_s33": ("kr", dict(d0=2, ell=5, k=9, base="real_rademacher", seed=33)),
    "kr_16_2_48_rad_s4": ("kr", dict(d0=16, ell=2, k=48, base="real_rademacher", seed=4)),
    "kr_8_3_20_gauss_s3": ("kr", dict(d0=8, ell=3, k=20, base="real_gaussian", seed=3)),
    "gauss_40_12_s21": ("gauss", dict(d=40, k=12, seed=21)),
    "gauss_128_32_s9": ("gauss", dict(d=128, k=32, seed=9)),
}


def oracle_right(name, a):
    fam, p = CASES[name]
    if fam == "su":
        return orc.csr_right(orc.sparse_uniform_csr(p["d"], p["k"], p["zeta"], p["seed"]), a)
    if fam == "ss":
        return orc.csr_right(orc.sparse_stack_csr(p["d"], p["zeta"], p["block"], p["seed"]), a)
    if fam == "sc":
        return orc.csr_right(orc.sparse_col_csr(p["d"], p["k"], p["xi"], p["seed"]), a)
    if fam == "rtt":
        dv, samp = orc.srtt_parts(p["d"], p["k"], p["xi"], p["seed"], p["diagonal"])
        return orc.srtt_right(dv, samp, a, p["transform"])
    if fam == "kr":
        return orc.kr_right(orc.kr_factors(p["d0"], p["ell"], p["k"], p["seed"], p["base"]), a)
    if fam == "gauss":
        return orc.dense_right(orc.gaussian_dense(p["d"], p["k"], p["seed"]), a)
    raise KeyError(fam)


def oracle_dense(name):
    """Omega as a dense float64 matrix, from the oracle."""
    fam, p = CASES[name]
    if fam == "su":
        return orc.sparse_uniform_csr(p["d"], p["k"], p["zeta"], p["seed"]).toarray()
    if fam == "ss":
        return orc.sparse_stack_csr(p["d"], p["zeta"], p["block"], p["seed"]).toarray()
    if fam == "sc":
        return orc.sparse_col_csr(p["d"], p["k"], p["xi"], p["seed"]).toarray()
    if fam == "gauss":
        return orc.gaussian_dense(p["d"], p["k"], p["seed"])
    d = p["d"] if fam == "rtt" else p["d0"] ** p["ell"]
    return oracle_right(name, np.eye(d))


def product(name):
    fam, p = CASES[name]
    if fam == "su":
        return skb.SparseUniformTM(p["d"], p["k"], p["zeta"], seed=p["seed"])
    if fam == "ss":
        return skb.SparseStackTM(p["d"], p["zeta"], p["block"], seed=p["seed"])
    if fam == "sc":
        return skb.SparseColTM(p["d"], p["k"], p["xi"], seed=p["seed"])
    if fam == "rtt":
        return skb.SparseRttTM(p["d"], p["k"], p["xi"], p["transform"], diagonal=p["diagonal"], seed=p["seed"])
    if fam == "kr":
        return skb.KhatriRaoTM(p["d0"], p["ell"], p["k"], p["base"], seed=p["seed"])
    if fam == "gauss":
        return skb.GaussianTM(p["d"], p["k"], seed=p["seed"])
    raise KeyError(fam)


def rel_err(x, ref) -> float:
    """Relative Frobenius error; complex arrays compare in complex128 (both parts)."""
    cplx = np.iscomplexobj(x) or np.iscomplexobj(ref)
    x = np.asarray(x, dtype=np.complex128 if cplx else np.float64)
    ref = np.asarray(ref, dtype=np.complex128 if cplx else np.float64)
    return float(np.linalg.norm(x - ref) / max(np.linalg.norm(ref), 1e-300))


def nystrom_inputs():
    """(tall 1024x300, wide 300x256, psd 512x512, probe 512x3) for the Nystrom golden fixtures."""
    rng = np.random.default_rng(2508)
    u1, _ = np.linalg.qr(rng.standard_normal((1024, 40)))
    v1, _ = np.linalg.qr(rng.standard_normal((300, 40)))
    agn = (u1 * (0.7 ** np.arange(40))) @ v1.T
    aw = agn[:256].T.copy()
    q, _ = np.linalg.qr(rng.standard_normal((512, 512)))
    apsd = (q * (0.8 ** np.arange(512))) @ q.T
    apsd = (apsd + apsd.T) / 2
    probe = rng.standard_normal((512, 3))
    return agn, aw, apsd, probe
