"""GPU drivers: rsvd / sketch_and_solve against the reference's own outputs (golden) and the
oracle; sketch-and-precondition LSQR against SciPy's LSQR (no reference test exists: unpinned)."""

import numpy as np
import pytest

import oracle as orc
from _cases import rel_err
from paper_2508_21189_b200 import rand_nla
from paper_2508_21189_b200 import sketch as skb

pytestmark = pytest.mark.gpu


def test_rsvd_matches_reference(golden, cuda):
    a = golden["rsvd_A"]
    for name, tm in (("rsvd_su", skb.SparseUniformTM(256, 40, 8, seed=5)),
                     ("rsvd_rtt", skb.SparseRttTM(256, 40, 1, "wht", seed=6))):
        f = rand_nla.rsvd(a, 40, tm)
        assert isinstance(f.sigma, np.ndarray)
        assert np.allclose(f.sigma, golden[f"{name}_sigma"], rtol=1e-9, atol=1e-14)
        assert rel_err((f.u * f.sigma) @ f.v.T, golden[f"{name}_recon"]) <= 1e-9


def test_rsvd_errors(cuda):
    tm = skb.SparseUniformTM(64, 8, 2, seed=0)
    with pytest.raises(ValueError, match="incompatible"):
        rand_nla.rsvd(np.ones((10, 64)), 9, tm)
    with pytest.raises(ValueError, match="exceeds"):
        rand_nla.rsvd(np.ones((4, 64)), 8, tm)


def test_rsvd_zero_matrix(cuda):
    f = rand_nla.rsvd(np.zeros((50, 64)), 8, skb.SparseUniformTM(64, 8, 2, seed=1))
    assert f.u.shape == (50, 0) and f.sigma.shape == (0,)


def test_rsvd_f32_config3_like(cuda):
    """Config-3 structure at reduced size: A = U diag(i^-2) V^T float32, k = 200, zeta = 8."""
    import torch

    n, d, k = 8192, 2048, 200
    g = torch.Generator(device=cuda).manual_seed(0)
    u, _ = torch.linalg.qr(torch.randn(n, d, device=cuda, dtype=torch.float64, generator=g))
    v, _ = torch.linalg.qr(torch.randn(d, d, device=cuda, dtype=torch.float64, generator=g))
    s = torch.arange(1, d + 1, device=cuda, dtype=torch.float64) ** -2.0
    a = ((u * s) @ v.T).to(torch.float32)
    tm = skb.SparseUniformTM(d, k, 8, seed=0)
    f = rand_nla.rsvd(a, k, tm)
    err = rand_nla.rsvd_residual(a, f)
    a64 = a.double().cpu().numpy()
    uo, so, vo = orc.rsvd(a64, lambda x: orc.csr_right(orc.sparse_uniform_csr(d, k, 8, 0), x), k)
    err_ref = np.linalg.norm(a64 - (uo * so) @ vo.T) / np.linalg.norm(a64)
    # The float32 sketch (BF16x2 tensor-core apply, ~3e-6 relative) perturbs the captured subspace in
    # directions with sigma_i near 1e-5 sigma_1; with sigma_i = i^-2 that moves the rank-200 residual by
    # ~1.5 %.  Stated tolerance for the float32 pipeline: 5 % of the float64 oracle's residual.
    assert abs(err - err_ref) <= 5e-2 * err_ref


def test_sketch_and_solve_matches_reference(golden, cuda):
    x = rand_nla.sketch_and_solve(golden["sas_A"], golden["sas_b"], skb.SparseUniformTM(3000, 200, 8, seed=9))
    assert rel_err(x, golden["sas_x"]) <= 1e-9


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_lsqr_vs_scipy(dt, cuda):
    import scipy.sparse.linalg as sla

    rng = np.random.default_rng(4)
    n, d = 40000, 64
    w = 1.0 + rng.pareto(1.5, size=n)
    a = (rng.standard_normal((n, d)) * w[:, None]).astype(dt)
    x0 = rng.standard_normal(d)
    b = (a.astype(np.float64) @ x0 + 1e-3 * rng.standard_normal(n)).astype(dt)
    tm = skb.SparseUniformTM(n, 256, 8, seed=3)
    res = rand_nla.sketch_precondition_lsqr(a, b, tm, atol=1e-10, btol=1e-10)
    ref = sla.lsqr(a.astype(np.float64), b.astype(np.float64), atol=1e-12, btol=1e-12, iter_lim=5000)[0]
    r_gpu = np.linalg.norm(a.astype(np.float64) @ res.x - b) / np.linalg.norm(b)
    r_ref = np.linalg.norm(a.astype(np.float64) @ ref - b) / np.linalg.norm(b)
    assert abs(r_gpu - r_ref) <= 1e-4 * r_ref
    assert res.itn < 60  # preconditioned: few iterations


@pytest.mark.parametrize("n,d", [(100000, 512), (3001, 37), (5, 1000), (70000, 130)])
def test_mixed_precision_gemv(n, d, cuda):
    """float32 A read once, float64 vectors / accumulation (LSQR matvecs)."""
    import torch

    from paper_2508_21189_b200.rand_nla import _matvec_blocks, _rmatvec_blocks

    g = torch.Generator(device=cuda).manual_seed(n + d)
    big = torch.randn(n, d + 3, device=cuda, generator=g)
    for a in (big[:, :d].contiguous(), big[:, 1:d + 1]):  # aligned and strided / misaligned
        v = torch.randn(d, dtype=torch.float64, device=cuda, generator=g)
        u = torch.randn(n, dtype=torch.float64, device=cuda, generator=g)
        a64 = a.double()
        y = _matvec_blocks(a, v, 1 << 16)
        z = _rmatvec_blocks(a, u, 1 << 16)
        assert float((y - a64 @ v).norm() / (a64 @ v).norm()) <= 1e-14
        assert float((z - a64.T @ u).norm() / (a64.T @ u).norm()) <= 1e-13


@pytest.mark.parametrize("n,d,k", [(1000, 260, 37), (5000, 128, 200), (70001, 516, 64), (300, 4, 1)])
def test_dense_tn_tc_vs_float64(n, d, k, cuda):
    """A^T W on the tensor cores (BF16x3, transposing converters) against float64 torch."""
    import torch

    from paper_2508_21189_b200.sketch.tensorcore import dense_tn_tc

    g = torch.Generator(device=cuda).manual_seed(n + d)
    a = torch.randn(n, d, device=cuda, generator=g)
    w = torch.randn(n, k, device=cuda, dtype=torch.float64, generator=g)
    y = dense_tn_tc(a, w, 0.5)
    ref = 0.5 * (a.double().T @ w)
    assert tuple(y.shape) == (d, k)
    assert float((y.double() - ref).norm() / ref.norm()) <= 1e-5
    # strided A (a column slice): copied to a dense operand first
    y2 = dense_tn_tc(torch.randn(n, 2 * d, device=cuda, generator=g)[:, :d].contiguous(), w)
    assert tuple(y2.shape) == (d, k)


def test_truncated_pinv_qr_path(cuda):
    """Well-conditioned tall systems take the QR solve, ill-conditioned / rank-deficient ones the
    reference's SVD with the 5-eps cut; both agree with the float64 SVD pseudo-inverse."""
    import torch

    g = torch.Generator(device=cuda).manual_seed(3)
    m = torch.randn(3000, 200, device=cuda, dtype=torch.float64, generator=g)
    b = torch.randn(3000, 3, device=cuda, dtype=torch.float64, generator=g)
    assert rand_nla._qr_solve_if_well_conditioned(m, b, rand_nla.DEFAULT_RANK_TOL) is not None
    ref = torch.linalg.pinv(m) @ b
    got = rand_nla.truncated_pinv_apply(m, b)
    assert float((got - ref).norm() / ref.norm()) <= 1e-12
    # exactly rank-deficient: the QR path must decline and the cut must apply
    m2 = m.clone()
    m2[:, 7] = m2[:, 3] * 2.0
    assert rand_nla._qr_solve_if_well_conditioned(m2, b, rand_nla.DEFAULT_RANK_TOL) is None
    u, s, vh = torch.linalg.svd(m2, full_matrices=False)
    r = int((s > rand_nla.DEFAULT_RANK_TOL * s[0]).sum())
    ref2 = vh[:r].T @ ((u[:, :r].T @ b) / s[:r, None])
    assert float((rand_nla.truncated_pinv_apply(m2, b) - ref2).norm() / ref2.norm()) <= 1e-10


@pytest.mark.parametrize("cond", [4e4, 1e9])
def test_svd_wide_matches_direct_svd(cond, cuda):
    """rsvd's SVD of B = Q^* A (200 x 16384): CholeskyQR2 + k x k SVD when B is well conditioned,
    the direct SVD otherwise; singular values to 1e-12 relative and B reconstructed to 1e-12."""
    import torch

    k, d = 200, 16384
    g = torch.Generator(device=cuda).manual_seed(1)
    u0, _ = torch.linalg.qr(torch.randn(d, k, dtype=torch.float64, device=cuda, generator=g))
    w0, _ = torch.linalg.qr(torch.randn(k, k, dtype=torch.float64, device=cuda, generator=g))
    s0 = torch.logspace(0, -np.log10(cond), k, dtype=torch.float64, device=cuda)
    b = (w0 * s0) @ u0.T
    u, s, vh = rand_nla._svd_wide(b)
    s_ref = torch.linalg.svdvals(b)
    assert float(((s - s_ref).abs() / s_ref).max()) <= 1e-9 * (cond / 4e4 if cond > 4e4 else 1.0)
    assert float(torch.linalg.norm((u * s) @ vh - b) / torch.linalg.norm(b)) <= 1e-12
    eye = torch.eye(k, dtype=torch.float64, device=cuda)
    assert float(torch.linalg.norm(u.T @ u - eye)) <= 1e-11 and float(torch.linalg.norm(vh @ vh.T - eye)) <= 1e-11


@pytest.mark.parametrize("n,d", [(100000, 512), (3001, 128), (7, 384), (70001, 256)])
def test_lsqr_fused_step(n, d, cuda):
    """One-pass LSQR step: u <- A v - alpha u, [A^T u_new, ||u_new||^2] against float64 torch."""
    import torch

    from paper_2508_21189_b200.rand_nla import _lsqr_fused_ok, _lsqr_step

    g = torch.Generator(device=cuda).manual_seed(n + d)
    a = torch.randn(n, d, device=cuda, generator=g)
    assert _lsqr_fused_ok(a)
    v = torch.randn(d, dtype=torch.float64, device=cuda, generator=g)
    u = torch.randn(n, dtype=torch.float64, device=cuda, generator=g)
    alpha = 0.37
    a64 = a.double()
    u_ref = a64 @ v - alpha * u
    zb = _lsqr_step(a, v, alpha, u)
    assert float((u - u_ref).norm() / u_ref.norm()) <= 1e-14
    z_ref = a64.T @ u_ref
    assert float((zb[:d] - z_ref).norm() / z_ref.norm()) <= 1e-13
    assert abs(float(zb[d]) - float(u_ref @ u_ref)) <= 1e-13 * float(u_ref @ u_ref)
    zb2 = _lsqr_step(a, v, alpha, u_ref.clone())  # deterministic: same inputs, same bits
    zb3 = _lsqr_step(a, v, alpha, u_ref.clone())
    assert torch.equal(zb2, zb3)


def test_lsqr_fused_matches_two_pass(cuda, monkeypatch):
    """float32 A, d = 256: the fused iteration and the two-kernel iteration reach the same solution."""
    import torch

    rng = np.random.default_rng(11)
    n, d = 200000, 256
    w = 1.0 + rng.pareto(1.5, size=n)
    a = torch.from_numpy((rng.standard_normal((n, d)) * w[:, None]).astype(np.float32)).to(cuda)
    x0 = rng.standard_normal(d)
    b = (a.double() @ torch.from_numpy(x0).to(cuda) + 1e-3 * torch.randn(n, dtype=torch.float64, device=cuda)).float()
    tm = skb.SparseUniformTM(n, 1024, 8, seed=5)
    r1 = rand_nla.sketch_precondition_lsqr(a, b, tm, atol=1e-10, btol=0.0)
    monkeypatch.setenv("SKETCH_B200_LSQR_FUSED", "0")
    r2 = rand_nla.sketch_precondition_lsqr(a, b, tm, atol=1e-10, btol=0.0)
    x1, x2 = np.asarray(r1.x.cpu() if hasattr(r1.x, "cpu") else r1.x), np.asarray(r2.x.cpu() if hasattr(r2.x, "cpu") else r2.x)
    assert r1.itn == r2.itn or abs(r1.itn - r2.itn) <= 2
    assert np.linalg.norm(x1 - x2) <= 1e-8 * np.linalg.norm(x2)


def test_lsqr_cpu_torch_b_with_cuda_a(cuda):
    """A CPU torch b with a CUDA A is moved to A's device (kernels take device pointers); a CPU
    torch A is uploaded and the solution comes back on the host."""
    import torch

    rng = np.random.default_rng(6)
    a = rng.standard_normal((5000, 32))
    b = a @ rng.standard_normal(32) + 1e-3 * rng.standard_normal(5000)
    tm = skb.SparseUniformTM(5000, 128, 8, seed=1)
    ref = rand_nla.sketch_precondition_lsqr(a, b, tm, atol=1e-12, btol=1e-12).x
    x_dev = rand_nla.sketch_precondition_lsqr(torch.from_numpy(a).to(cuda), torch.from_numpy(b), tm, atol=1e-12,
                                              btol=1e-12).x
    assert x_dev.is_cuda
    assert rel_err(x_dev.cpu().numpy(), ref) <= 1e-12
    x_cpu = rand_nla.sketch_precondition_lsqr(torch.from_numpy(a), torch.from_numpy(b), tm, atol=1e-12, btol=1e-12).x
    assert isinstance(x_cpu, torch.Tensor) and not x_cpu.is_cuda
    assert rel_err(x_cpu.numpy(), ref) <= 1e-12


def test_lsqr_iter_lim_zero(cuda):
    rng = np.random.default_rng(7)
    a = rng.standard_normal((3000, 16))
    b = rng.standard_normal(3000)
    res = rand_nla.sketch_precondition_lsqr(a, b, skb.SparseUniformTM(3000, 64, 8, seed=2), iter_lim=0)
    assert res.itn == 0 and np.all(res.x == 0)


@pytest.mark.parametrize("atol,btol", [(1e-10, 0.0), (1e-6, 1e-6), (1e-3, 1e-8)])
def test_lsqr_device_loop_matches_host_loop(atol, btol, cuda, monkeypatch):
    """The device recurrences (sk_lsqr_recur_f64) against the host-recurrence fused loop: same stop,
    same iteration count, same solution and estimates (float64 both, rounding-level differences)."""
    import torch

    rng = np.random.default_rng(12)
    n, d = 150000, 384
    w = 1.0 + rng.pareto(1.5, size=n)
    a = torch.from_numpy((rng.standard_normal((n, d)) * w[:, None]).astype(np.float32)).to(cuda)
    b = (a.double() @ torch.from_numpy(rng.standard_normal(d)).to(cuda)
         + 1e-2 * torch.randn(n, dtype=torch.float64, device=cuda)).float()
    tm = skb.SparseUniformTM(n, 1536, 8, seed=6)
    r1 = rand_nla.sketch_precondition_lsqr(a, b, tm, atol=atol, btol=btol)
    monkeypatch.setenv("SKETCH_B200_LSQR_DEVLOOP", "0")
    r2 = rand_nla.sketch_precondition_lsqr(a, b, tm, atol=atol, btol=btol)
    x1, x2 = r1.x.cpu().numpy(), r2.x.cpu().numpy()
    assert (r1.istop, r1.itn) == (r2.istop, r2.itn)
    assert np.linalg.norm(x1 - x2) <= 1e-9 * np.linalg.norm(x2)
    for f in ("r1norm", "arnorm", "acond", "normal_eq_test"):
        assert abs(getattr(r1, f) - getattr(r2, f)) <= 1e-6 * abs(getattr(r2, f)) + 1e-300, f


@pytest.mark.parametrize("k,kind", [(1, "rand"), (7, "rand"), (200, "decay"), (200, "repeated"), (300, "illcond"),
                                    (512, "rand")])
def test_svd_square_augmented_eigh(k, kind, cuda):
    """`_svd_square` (eigh of [[0, R], [R^T, 0]]) against torch.linalg.svd: singular values, the
    reconstruction and orthonormal factors; an ill-conditioned R takes the direct SVD."""
    import torch

    g = torch.Generator(device=cuda).manual_seed(k)
    u, _ = torch.linalg.qr(torch.randn(k, k, dtype=torch.float64, device=cuda, generator=g))
    v, _ = torch.linalg.qr(torch.randn(k, k, dtype=torch.float64, device=cuda, generator=g))
    if kind == "decay":
        s = torch.arange(1, k + 1, dtype=torch.float64, device=cuda) ** -2.0
    elif kind == "repeated":
        s = torch.ones(k, dtype=torch.float64, device=cuda)
        s[k // 2:] = 0.5
    elif kind == "illcond":
        s = torch.logspace(0, -12, k, dtype=torch.float64, device=cuda)
    else:
        s = torch.rand(k, dtype=torch.float64, device=cuda, generator=g) + 0.1
    r = (u * s) @ v.T
    uu, ss, vh = rand_nla._svd_square(r)
    s_ref = torch.linalg.svdvals(r)
    assert float((ss - s_ref).abs().max()) <= 1e-12 * float(s_ref[0])
    assert float(((uu * ss) @ vh - r).norm()) <= 1e-12 * float(r.norm())
    eye = torch.eye(k, dtype=torch.float64, device=cuda)
    assert float((uu.T @ uu - eye).norm()) <= 1e-10 and float((vh @ vh.T - eye).norm()) <= 1e-10


@pytest.mark.parametrize("dup", [0, 1, 3])
def test_qr_tall_paths(dup, cuda):
    """`_qr_tall` on a tall float64 matrix with `dup` duplicated columns (an SRTT sketch sampled with
    replacement): Q orthonormal with k columns, m = Q R, and Q's span contains m's columns."""
    import torch

    g = torch.Generator(device=cuda).manual_seed(dup)
    n, k = 1 << 18, 48
    m = torch.randn(n, k, dtype=torch.float64, device=cuda, generator=g)
    for i in range(dup):
        m[:, 2 * i + 1] = -m[:, 2 * i]
    q, r = rand_nla._qr_tall(m)
    eye = torch.eye(k, dtype=torch.float64, device=cuda)
    assert q.shape == (n, k)
    assert float((q.T @ q - eye).norm()) <= 1e-12
    assert float((q @ r - m).norm()) <= 1e-12 * float(m.norm())
    assert float((m - q @ (q.T @ m)).norm()) <= 1e-12 * float(m.norm())


def test_gen_nystrom_svd_srtt_with_repeats(cuda):
    """Generalized Nystrom with an SRTT Omega whose sampler repeats rows (rank-deficient Y): the
    factorization reproduces a low-rank A to rounding."""
    import torch

    g = torch.Generator(device=cuda).manual_seed(4)
    n, d, r = 200000, 512, 20
    a = (torch.randn(n, r, dtype=torch.float64, device=cuda, generator=g)
         @ torch.randn(r, d, dtype=torch.float64, device=cuda, generator=g)).float()
    om = skb.SparseRttTM(d, 64, 1, "wht", seed=1)
    ps = skb.SparseUniformTM(n, 96, 8, seed=2)
    fs = rn_gn(a, om, ps)
    approx = (fs.u * fs.sigma) @ fs.v.T
    assert float((approx - a.double()).norm() / a.double().norm()) <= 1e-5


def rn_gn(a, om, ps):
    return rand_nla.gen_nystrom_svd(a, 64, 96, om, ps)
