"""Complex fields on the FP64 DMMA engine (K5d over planes, sketch/zplanes.py): the reference's
default Khatri-Rao base (complex_spherical), complex Gaussian and Steinhaus Khatri-Rao, with real and
complex operands, right applies and adjoints (matrix and vector), against outputs of the real
reference stored in tests/golden (float64 / complex128, 1e-12)."""

import numpy as np
import pytest

from _cases import rel_err
from paper_2508_21189_b200 import sketch as skb

pytestmark = pytest.mark.gpu

ZCASES = {
    "kr_16_2_48_csph_s4": lambda: skb.KhatriRaoTM(16, 2, 48, seed=4),
    "kr_8_3_20_cgauss_s3": lambda: skb.KhatriRaoTM(8, 3, 20, "complex_gaussian", seed=3),
    "kr_6_2_70_stein_s8": lambda: skb.KhatriRaoTM(6, 2, 70, "steinhaus", seed=8),
    "gauss_c_128_32_s9": lambda: skb.GaussianTM(128, 32, "complex", 9),
}


@pytest.mark.parametrize("name", sorted(ZCASES))
def test_complex_field_applies_vs_reference(name, golden, cuda):
    tm = ZCASES[name]()
    g = {k[len(name) + 2:]: v for k, v in golden.items() if k.startswith(name + "__")}
    assert rel_err(tm.apply_right(g["A"]), g["right"]) <= 1e-12
    assert rel_err(tm.apply_right(g["Ac"]), g["right_c"]) <= 1e-12
    assert rel_err(tm.apply_adjoint(g["B"]), g["adjoint"]) <= 1e-12
    assert rel_err(tm.apply_adjoint(g["Bc"]), g["adjoint_c"]) <= 1e-12
    assert rel_err(tm.apply_adjoint(g["B"][:, 0]), g["adjoint_vec"]) <= 1e-12
    assert any(k[0] in ("kr_z", "dense_z") for k in tm._device_cache)  # the DMMA planes ran


@pytest.mark.parametrize("d0,ell,k", [(64, 2, 96), (5, 3, 33), (256, 2, 64)])
def test_complex_kr_config_scale(d0, ell, k, cuda):
    """Larger complex Khatri-Rao (several leading blocks P > 1, ragged k) against the dense product."""
    import torch

    tm = skb.KhatriRaoTM(d0, ell, k, seed=k)
    rng = np.random.default_rng(k)
    a = rng.standard_normal((700, d0 ** ell)) + 1j * rng.standard_normal((700, d0 ** ell))
    b = rng.standard_normal((d0 ** ell, 130)) + 1j * rng.standard_normal((d0 ** ell, 130))
    om = tm.materialize()
    y = tm.apply_right(torch.from_numpy(a).to(cuda)).cpu().numpy()
    x = tm.apply_adjoint(torch.from_numpy(b).to(cuda)).cpu().numpy()
    assert rel_err(y, a @ om) <= 1e-12
    assert rel_err(x, om.conj().T @ b) <= 1e-12
