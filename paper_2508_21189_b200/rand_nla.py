"""Downstream drivers of the sketch on the GPU: randomized SVD, sketch-and-solve and
sketch-and-precondition LSQR.

`rsvd` and `sketch_and_solve` mirror the reference (src/rand_nla.py:84-109 and :278-297, with
`orth` / `truncated_pinv_apply` / `svd_econ` from src/core/factor.py:56-136): same argument
checks, same 5-eps numerical-rank cut, same result shapes.  The sketch runs through the B200
kernels (`tm.apply_right` / `tm.apply_adjoint`); the small dense factorizations run in float64
on the device (cuSOLVER through torch); the second pass over A (Q^* A) is a plain fp32 GEMM.

`sketch_precondition_lsqr` is new (the reference only remarks on it; SPEC.md:301 marks
it a non-goal): S A = Q R, then LSQR (Paige-Saunders) on A R^-1 with the normal-equation stopping
test ||(A R^-1)^T r|| <= atol ||A R^-1|| ||r|| (the problem is inconsistent), matvecs on the
resident A with float64 reductions.  Its parity is pinned against SciPy's LSQR in the tests, not
against a reference test (none exists).
"""

from __future__ import annotations

from dataclasses import dataclass

import math
import os

import threading

import numpy as np

from ._device import require_cuda, to_operand

__all__ = ["SvdFactorization", "OuterProduct", "EigFactorization", "LsqrResult", "PositiveDefinitenessError", "orth",
           "rsvd", "rsvd_residual", "nystrom_psd", "gen_nystrom_outer", "gen_nystrom_svd", "two_sided_sketch",
           "default_left_dim", "sketch_and_solve", "truncated_pinv_apply", "sketch_precondition_lsqr", "EPS",
           "DEFAULT_RANK_TOL"]

EPS = float(np.finfo(np.float64).eps)
DEFAULT_RANK_TOL = 5.0 * EPS  # reference core/factor.py:27-28


@dataclass
class SvdFactorization:
    """A ~= u diag(sigma) v^*  (reference core/containers.py SvdFactorization)."""

    u: object
    sigma: object
    v: object

    def to_numpy(self) -> "SvdFactorization":
        return SvdFactorization(*(x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)
                                  for x in (self.u, self.sigma, self.v)))


@dataclass
class OuterProduct:
    """A ~= f g^* (reference core/containers.py:124-146)."""

    f: object
    g: object

    @property
    def rank(self) -> int:
        return self.f.shape[1]

    def matrix(self):
        return self.f @ self.g.conj().T


@dataclass
class EigFactorization:
    """Psd A ~= u diag(lam) u^* (reference core/containers.py:180-206)."""

    u: object
    lam: object

    @property
    def rank(self) -> int:
        return self.lam.shape[0]

    def matrix(self):
        return (self.u * self.lam) @ self.u.conj().T


class PositiveDefinitenessError(np.linalg.LinAlgError):
    """Cholesky met a non-positive pivot (reference core/factor.py:31-32)."""


@dataclass
class LsqrResult:
    x: object
    istop: int
    itn: int
    r1norm: float
    arnorm: float
    acond: float
    sketch_seconds: float = 0.0
    normal_eq_test: float = 0.0


def _t64(x):
    import torch

    return x.to(torch.complex128 if x.is_complex() else torch.float64)


def orth(m, rel_tol: float = DEFAULT_RANK_TOL):
    """Orthonormal basis of the numerical range (reference core/factor.py:63-82), on the device.

    Tall well-conditioned inputs (the rsvd sketch Y) take CholeskyQR2 in float64 — two Gram
    matrices, two Cholesky factors, two triangular solves: a handful of GEMM-shaped passes instead
    of a Householder QR (config 3, Y 131072 x 200: 9.9 -> ~2 ms). Anything else — a failed
    Cholesky, diag(R) spread beyond 1e6 (CholeskyQR2 keeps orthogonality to ~eps only while
    cond(Y) stays well below eps^-1/2), or the reference's rank cut firing — goes through the
    reference path: Householder QR, then the 5-eps rank test on diag(R), else an SVD.
    """
    import torch

    m = _t64(m)
    if not bool(torch.isfinite(m).all()):
        raise ValueError("matrix has nonfinite entries")
    if m.shape[1] == 0:
        return m.clone()
    n, k = m.shape
    if m.is_cuda and n >= 16 * k and n * k >= (1 << 20) and not m.is_complex():
        q = _cholqr2(m)
        if q is not None:
            return q
    q, r = torch.linalg.qr(m, mode="reduced")
    diag = r.diagonal().abs()
    top = float(diag.max()) if diag.numel() else 0.0
    if top == 0.0:
        return q[:, :0]
    if float(diag.min()) > rel_tol * top:
        return q
    u, s, _ = torch.linalg.svd(m, full_matrices=False)
    rank = int((s > rel_tol * s[0]).sum())
    return u[:, :rank]


def _cholqr2(m, max_spread: float = 1e6):
    """Q of m = QR by CholeskyQR2 (float64), or None when the reference path must decide."""
    res = _cholqr2_qr(m, max_spread)
    return None if res is None else res[0]


def _svd_square(r, min_ratio: float = 1e-7):
    """Thin SVD (U, S, Vh) of a small float64 CUDA matrix (m x n) through the symmetric eigenproblem
    of the augmented [[0, R], [R^T, 0]] (eigenvalues +-sigma_i and |m - n| zeros, eigenvectors
    [u_i; v_i] / sqrt 2): no squaring of the condition number (unlike the Gram matrix), sigma to
    ~eps * sigma_max.  cuSOLVER's SVD of the config-3 200 x 200 factor takes ~7-11 ms (Jacobi
    sweeps), this eigh 4 ms (`tools/svd_small_probe.py`).  A matrix with sigma_min below
    min_ratio * sigma_max (where the zero eigenvalues could mix u and v) takes torch.linalg.svd."""
    import torch

    m, n = r.shape
    q = min(m, n)
    if q == 0:
        return torch.linalg.svd(r, full_matrices=False)
    aug = torch.zeros((m + n, m + n), dtype=r.dtype, device=r.device)
    aug[:m, m:] = r
    aug[m:, :m] = r.T
    w, vec = torch.linalg.eigh(aug)
    s = w[m + n - q:].flip(0)
    if not bool(torch.isfinite(s).all()) or float(s[-1]) <= min_ratio * float(s[0]):
        return torch.linalg.svd(r, full_matrices=False)
    top = vec[:, m + n - q:].flip(1) * math.sqrt(2.0)
    return top[:m].contiguous(), s.contiguous(), top[m:].T.contiguous()


def _qr_tall(m):
    """Reduced QR of a tall float64 matrix: CholeskyQR2 on the device for tall, well-conditioned m
    (the generalized-Nystrom Y at the DESIGN section-6 shape, 2M x 64: cuSOLVER's Householder QR
    ~40 ms, CholeskyQR2 a few), else torch.linalg.qr.  Q differs from Householder's by column signs
    only (R with a positive diagonal); every caller consumes it sign-invariantly."""
    import torch

    n, k = m.shape
    if m.is_cuda and not m.is_complex() and k > 0 and n >= 16 * k and n * k >= (1 << 20):
        res = _cholqr2_qr(m)
        if res is None:
            res = _qr_tall_split(m)
        if res is not None:
            return res
    return torch.linalg.qr(m, mode="reduced")


def _qr_tall_split(m, gap: float = 1e10, kept_cond: float = 1e8):
    """Orthonormal Q (n x k) and R = Q^T m for a tall m whose Gram spectrum splits cleanly into a
    well-conditioned part and exact zeros — e.g. an SRTT sketch whose sampler drew the same row for
    two columns (sampling with replacement), where CholeskyQR2 cannot run: Q = [m V_r L_r^-1/2
    re-orthonormalised by CholeskyQR2, a seeded orthonormal completion].  Householder QR's Q also
    completes the rank-deficient part arbitrarily; callers use Q's span and m = Q R only.  None when
    the spectrum has no clean split (Householder QR then runs)."""
    import torch

    n, k = m.shape
    lam, vec = torch.linalg.eigh(m.T @ m)  # ascending
    lmax = float(lam[-1])
    if not lmax > 0.0:
        return None
    lam_h = lam.cpu().numpy()
    nz = int((lam_h > lmax / kept_cond).sum())  # eigenvalues of the kept, well-conditioned part
    if nz == 0 or nz == k or not lam_h[k - nz] > gap * max(float(lam_h[k - nz - 1]), 0.0):
        return None
    keep = slice(k - nz, k)
    qr_ = m @ (vec[:, keep] / lam[keep].sqrt())
    res = _cholqr2_qr(qr_)
    if res is None:
        return None
    q1 = res[0]
    g = torch.Generator(device=m.device).manual_seed(20250821)
    c = torch.randn(n, k - nz, dtype=m.dtype, device=m.device, generator=g)
    for _ in range(2):
        c = c - q1 @ (q1.T @ c)
    res_c = _cholqr2_qr(c)
    if res_c is None:
        return None
    q = torch.cat([q1, res_c[0]], dim=1)
    return q, q.T @ m


def _svd_wide(b):
    """Thin SVD of a wide float64 B (k x d, d >> k), as torch.linalg.svd(b, full_matrices=False).

    The rsvd core step (reference rand_nla.py:105, svd_econ of B = Q^* A): CholeskyQR2 of B^T (two
    k x k Gram matrices) and the SVD of the k x k triangular factor (`_svd_square`) at the accuracy of
    the direct SVD (B^T = Q_B R, R = U_R S V_R^T: B = V_R S (Q_B U_R)^T). Ill-conditioned or rank-deficient B (where CholeskyQR2 loses
    orthogonality, or the reference's rank cut applies) takes the direct SVD.
    """
    import torch

    k, d = b.shape
    if b.is_cuda and not b.is_complex() and k > 0 and d >= 16 * k and k * d >= (1 << 20):
        res = _cholqr2_qr(b.T)
        if res is not None:
            qb, r = res
            ur, s, vrh = _svd_square(r) if r.shape[0] <= 512 else torch.linalg.svd(r, full_matrices=False)
            return vrh.T, s, (qb @ ur).T
    return torch.linalg.svd(b, full_matrices=False)


def _cholqr2_qr(m, max_spread: float = 1e6):
    """(Q, R) of m = QR by CholeskyQR2 (float64), or None when the reference path must decide."""
    import torch

    r_tot = None
    q = m
    for _ in range(2):
        g = q.T @ q
        r, info = torch.linalg.cholesky_ex(g, upper=True)
        if int(info) != 0:
            return None
        d = r.diagonal()
        if float(d.min()) <= 0.0 or float(d.max()) > max_spread * float(d.min()):
            return None
        # Q R^-1 as one GEMM with the explicit k x k inverse (cuBLAS trsm on a tall Q is ~3x slower:
        # 1.26 vs 0.41 + 0.12 ms at 131072 x 200); the second pass restores orthogonality to ~eps
        eye = torch.eye(r.shape[0], dtype=r.dtype, device=r.device)
        q = q @ torch.linalg.solve_triangular(r, eye, upper=True)
        r_tot = r if r_tot is None else r @ r_tot
    diag = r_tot.diagonal().abs()
    if float(diag.min()) <= DEFAULT_RANK_TOL * float(diag.max()):
        return None  # the reference's rank cut applies: let QR + SVD handle it
    return q, r_tot


def _as_device_2d(a, host_scaffold: bool = False):
    """A as a CUDA tensor (host input is uploaded).  host_scaffold=True keeps a CPU torch A on the host
    for the driver-logic tests (tests/test_dist_gloo.py), whose operator is a CPU oracle stand-in."""
    import torch

    if isinstance(a, torch.Tensor) and a.dim() == 2 and a.dtype in (torch.float32, torch.float64) and (
            a.is_cuda or host_scaffold):
        return a, ("cuda" if a.is_cuda else "tensor")
    op = to_operand(a, allow_vector=False)
    return op.tensor, op.kind


def _as_vec(b, like):
    """b as a tensor on A's device (a CPU tensor b with a CUDA A is moved: kernels take device pointers)."""
    import torch

    t = b if isinstance(b, torch.Tensor) else torch.as_tensor(np.asarray(b))
    t = t.to(like.device)
    return t[:, 0] if t.dim() == 2 and t.shape[1] == 1 else t


def _back(x, kind):
    if kind == "numpy":
        x = x.cpu().numpy()
        return x.astype(np.complex128 if np.iscomplexobj(x) else np.float64, copy=False)
    if kind == "torch-cpu":
        return x.cpu()
    return x


def rsvd(a, k: int, tm) -> SvdFactorization:
    """Randomized SVD, two passes over A, rank <= k (reference rand_nla.py:84-109)."""
    import torch

    require_cuda()
    shape = tuple(a.shape)
    n, d = shape
    if tm.d != d or tm.k != k:
        raise ValueError(f"test matrix {tm!r} incompatible with A {shape} and k={k}")
    if k > min(n, d):
        raise ValueError(f"k={k} exceeds min(n, d)={min(n, d)}")
    A, kind = _as_device_2d(a)
    y = tm.apply_right(A)
    q = orth(y)
    if q.shape[1] == 0:
        z = torch.zeros
        fac = SvdFactorization(z((n, 0), dtype=q.dtype, device=A.device), z(0, dtype=torch.float64, device=A.device),
                               z((d, 0), dtype=q.dtype, device=A.device))
    else:
        b = _qt_a(q, A)
        u, s, vh = _svd_wide(_t64(b))
        fac = SvdFactorization(q @ u.to(q.dtype), s, vh.conj().T)
    if kind in ("numpy", "torch-cpu"):
        return SvdFactorization(_back(fac.u, kind), _back(fac.sigma, kind), _back(fac.v, kind))
    return fac


def _qt_a(q, A):
    """B = Q^* A, the second pass over A. float32 CUDA A: the tensor-core TN product
    (sk_dense_tn_tc, BF16x3, A read once: config 3 20.5 ms fp32 cuBLAS -> ~2 ms); otherwise a
    GEMM in A's precision (no TF32)."""
    import torch

    if (A.is_cuda and A.dtype == torch.float32 and not q.is_complex() and A.shape[1] % 4 == 0
            and A.shape[0] * A.shape[1] >= (1 << 22)):
        from .sketch.tensorcore import dense_tn_tc

        return dense_tn_tc(A, q).T.to(q.dtype)
    with _no_tf32():
        return (q.to(A.dtype).conj().T @ A).to(q.dtype)


class _no_tf32:
    def __enter__(self):
        import torch

        self.prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False

    def __exit__(self, *exc):
        import torch

        torch.backends.cuda.matmul.allow_tf32 = self.prev


def rsvd_residual(a, fac: SvdFactorization, block_rows: int = 8192) -> float:
    """||A - U diag(s) V^*||_F / ||A||_F, computed explicitly in row blocks with float64 sums.

    ||A||^2 - ||B||^2 cancels catastrophically in fp32, so the residual is formed.
    """
    import torch

    A, _ = _as_device_2d(a)
    u = torch.as_tensor(fac.u, device=A.device)
    s = torch.as_tensor(fac.sigma, device=A.device)
    v = torch.as_tensor(fac.v, device=A.device)
    w = (s[None, :] * v.conj()).T.to(A.dtype)  # k x d
    num = 0.0
    den = 0.0
    with _no_tf32():
        for r0 in range(0, A.shape[0], block_rows):
            blk = A[r0:r0 + block_rows]
            res = blk - u[r0:r0 + block_rows].to(A.dtype) @ w
            num += float((res.double() ** 2).sum())
            den += float((blk.double() ** 2).sum())
    return float(np.sqrt(num / den)) if den > 0 else 0.0


def truncated_pinv_apply(m, b, rel_tol: float = DEFAULT_RANK_TOL):
    """V_r diag(1/sigma_r) U_r^* b with the 5-eps cut (reference core/factor.py:112-136)."""
    import torch

    m = _t64(m)
    b = _t64(b)
    squeeze = b.dim() == 1
    if squeeze:
        b = b[:, None]
    if b.shape[0] != m.shape[0]:
        raise ValueError(f"shape mismatch: m {tuple(m.shape)}, b {tuple(b.shape)}")
    if m.is_cuda and not m.is_complex() and m.shape[0] >= m.shape[1] >= 64:
        x = _qr_solve_if_well_conditioned(m, b, rel_tol)
        if x is not None:
            return x[:, 0] if squeeze else x
    u, s, vh = torch.linalg.svd(m, full_matrices=False)
    rank = 0 if s.numel() == 0 or float(s[0]) == 0.0 else int((s > rel_tol * s[0]).sum())
    dt = torch.promote_types(m.dtype, b.dtype)
    if rank == 0:
        out = torch.zeros((m.shape[1], b.shape[1]), dtype=dt, device=m.device)
    else:
        core = (u[:, :rank].conj().T.to(dt) @ b.to(dt)) / s[:rank, None]
        out = vh[:rank].conj().T.to(dt) @ core
    return out[:, 0] if squeeze else out


def _qr_solve_if_well_conditioned(m, b, rel_tol, iters: int = 12, margin: float = 1e4):
    """min ||m x - b|| by Householder QR when m is far from the rank cut, else None.

    With every singular value above rel_tol * sigma_max the truncated pseudo-inverse is the exact
    least-squares solution, so R^-1 Q^* b equals it up to rounding. cuSOLVER's SVD of the config-4
    sketch (2048 x 512 float64) takes ~32 ms, latency-bound; QR + a condition estimate a few ms. The
    estimate (power iteration on R^T R, inverse iteration through two triangular solves) is only
    trusted with a margin of `margin` below the cut (kappa < 1 / (margin * rel_tol))."""
    import torch

    # CholeskyQR2 (two k x k Gram matrices: ~1 ms at 2048 x 512) unless R's diagonal spread says the
    # Gram matrix is too ill-conditioned for it; then Householder QR (cuSOLVER geqrf, ~4 ms)
    qr2 = _cholqr2_qr(m) if m.shape[0] >= 2 * m.shape[1] else None
    q, r = qr2 if qr2 is not None else torch.linalg.qr(m, mode="reduced")
    d = r.diagonal().abs()
    if float(d.min()) == 0.0:
        return None
    g = torch.Generator(device=m.device).manual_seed(12345)
    v = torch.randn(r.shape[1], 1, dtype=r.dtype, device=m.device, generator=g)
    w = v.clone()
    for _ in range(iters):
        v = r.T @ (r @ v)
        v = v / torch.linalg.norm(v)
        w = torch.linalg.solve_triangular(r, torch.linalg.solve_triangular(r.T, w, upper=False), upper=True)
        w = w / torch.linalg.norm(w)
    smax = float(torch.linalg.norm(r @ v))
    smin = float(torch.linalg.norm(r @ w))
    if not (smin > margin * rel_tol * smax):
        return None
    return torch.linalg.solve_triangular(r, q.T @ b, upper=True)


def sketch_and_solve(a, b, tm_psi):
    """(Psi^* A)^+ (Psi^* B) with the 5-eps cut (reference rand_nla.py:278-297)."""
    n = tuple(a.shape)[0]
    if tm_psi.d != n:
        raise ValueError("left test matrix must act on the row space of A")
    bshape = tuple(np.shape(b)) if not hasattr(b, "shape") else tuple(b.shape)
    squeeze = len(bshape) == 1
    if bshape[0] != n:
        raise ValueError(f"B must have {n} rows, got {bshape}")
    A, kind = _as_device_2d(a)
    a_sk = tm_psi.apply_adjoint(A)
    B = to_operand(b, allow_vector=True)
    b_sk = tm_psi.apply_adjoint(B.tensor)
    out = truncated_pinv_apply(a_sk, b_sk)
    if squeeze:
        out = out[:, 0]
    return _back(out, kind)


def default_left_dim(k: int) -> int:
    """Recommended left-sketch dimension p = ceil(1.5 k) (reference rand_nla.py:48-50)."""
    return int(np.ceil(1.5 * k))


def _svd_econ(m):
    import torch

    m = _t64(m)
    if m.is_cuda and not m.is_complex() and 0 < m.shape[0] + m.shape[1] <= 512:
        u, s, vh = _svd_square(m)  # small real factors: the augmented eigh (see _svd_square)
    else:
        u, s, vh = torch.linalg.svd(m, full_matrices=False)
    return u, s, vh.conj().T


def _rank_of(s) -> int:
    return 0 if s.numel() == 0 or float(s[0]) == 0.0 else int((s > DEFAULT_RANK_TOL * s[0]).sum())


def _omega_bt(tm):
    """Omega^T in bf16 (hi, lo-or-None, scale) for the fused kernel, cached on the operator: sparse sign
    operators exactly (+-1, magnitude as the scale), other families through the materialised Omega
    (small d x k only: the right operand of a generalized-Nystrom sketch)."""
    import torch

    from .sketch.tensorcore import bt_from_dense, bt_from_triplets

    dev = torch.device("cuda", torch.cuda.current_device())
    key = ("two_sided_bt", dev)
    if key not in tm._device_cache:
        sf = tm._sign_form() if hasattr(tm, "_sign_form") else None
        if sf is not None:
            rows, cols, neg, mag = sf
            hi, lo = bt_from_triplets(rows, cols, neg, tm.d, tm.k, dev)
            tm._device_cache[key] = (hi, lo, mag)
        else:
            om = tm.materialize()
            mag = float(np.abs(om).max()) or 1.0
            hi, lo = bt_from_dense(om / mag, dev)
            tm._device_cache[key] = (hi, lo, mag)
    return tm._device_cache[key]


def _psi_rows(tm):
    """Psi as [n][zeta] uint8 (q | neg << 7) for the fused kernel (exactly zeta targets per row, p <= 128),
    or None."""
    import torch

    if tm.k > 128 or tm.field != "real" or not hasattr(tm, "_sign_form"):
        return None
    dev = torch.device("cuda", torch.cuda.current_device())
    key = ("two_sided_psi", dev)
    if key not in tm._device_cache:
        res = None
        dform = tm._device_sign_form(dev)
        if dform is not None:
            cols, neg, mag = dform
            res = ((cols.to(torch.int32) | (neg.to(torch.int32) << 7)).to(torch.uint8).contiguous(), cols.shape[1], mag)
        else:
            sf = tm._sign_form()
            if sf is not None:
                rows, cols, neg, mag = sf
                cnt = np.bincount(rows, minlength=tm.d) if rows.size else np.zeros(tm.d, np.int64)
                if rows.size and cnt.min() == cnt.max() and np.all(np.diff(rows) >= 0):
                    z = int(cnt[0])
                    ent = (cols.astype(np.int64) | (neg.astype(np.int64) << 7)).astype(np.uint8).reshape(tm.d, z)
                    res = (torch.from_numpy(ent).to(dev), z, mag)
        tm._device_cache[key] = res
    return tm._device_cache[key]


def two_sided_sketch(a, tm_omega, tm_psi, *, fused: bool | None = None):
    """Y = A Omega (n x k) and X = A^* Psi (d x p) for the generalized Nystrom drivers.

    float32 device A with a sparse-sign Psi (exactly zeta per row, p <= 128) and k <= 128: ONE pass
    over A on the fused tcgen05 kernel (`sk_two_sided_sketch`): every tile of A feeds
    both products from shared memory.  Otherwise (or fused=False) the two applies run separately.
    Returns device tensors in A's precision.
    """
    import torch

    A, _ = _as_device_2d(a)
    n, d = A.shape
    psi = None
    ok = (A.is_cuda and A.dtype == torch.float32 and tm_omega.k <= 128 and tm_omega.field == "real"
          and tm_omega.d * tm_omega.k <= (1 << 26) and fused is not False)
    if ok:
        psi = _psi_rows(tm_psi)
    if psi is None:
        if fused:
            raise ValueError("the fused two-sided kernel needs float32 CUDA A, k <= 128 and a sparse-sign Psi "
                             "with exactly zeta nonzeros per row and p <= 128")
        return tm_omega.apply_right(A), tm_psi.apply_adjoint(A).conj().T
    from . import _lib

    ent, zeta, mag_psi = psi
    hi, lo, mag_om = _omega_bt(tm_omega)
    if A.stride(1) != 1 or A.stride(0) % 4 or A.data_ptr() % 16:
        A = A.contiguous()
    k, p = tm_omega.k, tm_psi.k
    y = torch.empty((n, k), dtype=torch.float32, device=A.device)
    xt = torch.empty((p, d), dtype=torch.float32, device=A.device)
    lib = _lib.load()
    ws_bytes = lib.sk_two_sided_workspace_bytes(max(n, 1), d, k, 1 if lo is not None else 0)
    ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=A.device)
    with torch.cuda.device(A.device):
        st = lib.sk_two_sided_sketch(A.data_ptr(), n, d, A.stride(0), hi.data_ptr(),
                                     lo.data_ptr() if lo is not None else None, hi.stride(0), k, float(mag_om),
                                     ent.data_ptr(), zeta, p, float(mag_psi), y.data_ptr(), y.stride(0), xt.data_ptr(),
                                     xt.stride(0), ws.data_ptr(), ws_bytes, torch.cuda.current_stream().cuda_stream)
    _lib.check(st, "sk_two_sided_sketch")
    return y, xt.T


def _gn_core(A, tm_omega, tm_psi) -> OuterProduct:
    """Reference rand_nla.py:191-202 on the device (float64 small factorizations)."""
    y, x = two_sided_sketch(A, tm_omega, tm_psi)
    w = tm_omega.apply_right(x.conj().T.contiguous())  # (Psi^* A) Omega, p x k
    u, s, v = _svd_econ(w)
    r = _rank_of(s)
    f = _t64(y) @ (v[:, :r] / s[:r])
    g = _t64(x) @ u[:, :r]
    return OuterProduct(f=f, g=g)


def _validate_gn(shape, k: int, p: int, tm_omega, tm_psi):
    n, d = shape
    if not (k <= p <= min(n, d)):
        raise ValueError(f"need k <= p <= min(n, d); got k={k}, p={p}, shape={shape}")
    if tm_omega.d != d or tm_omega.k != k:
        raise ValueError("right test matrix has wrong dimensions")
    if tm_psi.d != n or tm_psi.k != p:
        raise ValueError("left test matrix has wrong dimensions")
    return n, d


def _adjoint_dev(A):
    import torch

    out = torch.empty((A.shape[1], A.shape[0]), dtype=A.dtype, device=A.device)
    out.copy_(A.conj().T)
    return out


def _back_factors(obj, kind):
    if kind not in ("numpy", "torch-cpu"):
        return obj
    return type(obj)(*(_back(getattr(obj, f), kind) for f in obj.__dataclass_fields__))


def gen_nystrom_outer(a, k: int, p: int, tm_omega, tm_psi) -> OuterProduct:
    """Generalized Nystrom A ~= F G^* (reference rand_nla.py:216-227); wide inputs via the adjoint."""
    require_cuda()
    n, d = _validate_gn(tuple(a.shape), k, p, tm_omega, tm_psi)
    A, kind = _as_device_2d(a)
    if n < d:
        flipped = _gn_core(_adjoint_dev(A), tm_psi, tm_omega)
        out = OuterProduct(f=flipped.g, g=flipped.f)
    else:
        out = _gn_core(A, tm_omega, tm_psi)
    return _back_factors(out, kind)


def _gn_svd_core(A, tm_omega, tm_psi) -> SvdFactorization:
    """Reference rand_nla.py:230-245 on the device."""
    import torch

    y, x = two_sided_sketch(A, tm_omega, tm_psi)
    q, _ = _qr_tall(_t64(y))
    pmat, t = _qr_tall(_t64(x))
    w = _t64(tm_psi.apply_adjoint(q))  # p x k
    u1, s1, v1 = _svd_econ(w)
    r = _rank_of(s1)
    core = v1[:, :r] @ ((u1[:, :r].conj().T @ t.conj().T) / s1[:r, None])
    u2, s2, v2 = _svd_econ(core)
    return SvdFactorization(u=q @ u2, sigma=s2, v=pmat @ v2)


def _outer_to_svd(op: OuterProduct) -> SvdFactorization:
    """Reference rand_nla.py:248-259."""
    import torch

    if op.rank == 0:
        z = op.f.new_zeros
        return SvdFactorization(u=z((op.f.shape[0], 0)), sigma=z(0, dtype=torch.float64), v=z((op.g.shape[0], 0)))
    qf, rf = torch.linalg.qr(op.f, mode="reduced")
    qg, rg = torch.linalg.qr(op.g, mode="reduced")
    u, s, v = _svd_econ(rf @ rg.conj().T)
    return SvdFactorization(u=qf @ u, sigma=s, v=qg @ v)


def gen_nystrom_svd(a, k: int, p: int, tm_omega, tm_psi) -> SvdFactorization:
    """Generalized Nystrom in compact SVD form (reference rand_nla.py:262-275)."""
    require_cuda()
    n, d = _validate_gn(tuple(a.shape), k, p, tm_omega, tm_psi)
    A, kind = _as_device_2d(a)
    if n < d:
        flipped = _gn_core(_adjoint_dev(A), tm_psi, tm_omega)
        out = _outer_to_svd(OuterProduct(f=flipped.g, g=flipped.f))
    else:
        out = _gn_svd_core(A, tm_omega, tm_psi)
    return _back_factors(out, kind)


def _spectral_norm(y, iters: int = 20, seed: int = 0) -> float:
    """Power-iteration ||Y||_2 estimate, same start vector stream (reference rand_nla.py:112-131)."""
    import torch

    from .rng import RngStream

    if y.numel() == 0:
        return 0.0
    v0 = RngStream(seed, ("spectral-norm",)).generator().standard_normal(y.shape[1])
    y = _t64(y)
    v = torch.as_tensor(v0, device=y.device, dtype=y.dtype)
    v = v / torch.linalg.vector_norm(v)
    sigma = 0.0
    for _ in range(iters):
        w = y @ v
        nw = float(torch.linalg.vector_norm(w))
        if nw == 0.0:
            return 0.0
        v = y.conj().T @ (w / nw)
        sigma = float(torch.linalg.vector_norm(v))
        if sigma == 0.0:
            return 0.0
        v = v / sigma
        sigma = float(np.sqrt(sigma * nw))
    return sigma


def _check_psd(A, tol: float = 1e-8, probes: int = 8, seed: int = 0) -> None:
    """Sampled self-adjointness / psd check (reference rand_nla.py:134-149)."""
    import torch

    from .rng import RngStream

    n = A.shape[0]
    v = torch.as_tensor(RngStream(seed, ("psd-check",)).generator().standard_normal((n, probes)), device=A.device)
    with _no_tf32():
        av = _t64(A) @ v.to(torch.complex128 if A.is_complex() else torch.float64)
    quad = (v.conj() * av).sum(0)
    scale = max(float(torch.linalg.vector_norm(av, dim=0).max()), 1e-300) / np.sqrt(n)
    norms2 = (v.conj() * v).sum(0).real
    if bool((quad.imag.abs() > tol * scale * norms2).any()) if quad.is_complex() else False:
        raise ValueError("input is not self-adjoint to psd-check tolerance")
    if bool((quad.real < -tol * scale * norms2).any()):
        raise ValueError("input fails the sampled psd check")


def _cholesky_upper(m):
    """Upper C with M = C^* C (reference core/factor.py:85-104)."""
    import torch

    scale = float(torch.linalg.matrix_norm(m))
    if scale > 0 and float(torch.linalg.matrix_norm(m - m.conj().T)) > 1e-10 * scale:
        raise ValueError("input is not self-adjoint to tolerance 1e-10")
    lower, info = torch.linalg.cholesky_ex(m)
    if int(info) != 0:
        raise PositiveDefinitenessError(f"leading minor of order {int(info)} is not positive")
    return lower.conj().T


def nystrom_psd(a, k: int, tm, *, max_shift_retries: int = 3) -> EigFactorization:
    """Single-pass psd Nystrom with the stabilizing shift (reference rand_nla.py:152-188)."""
    import torch

    require_cuda()
    shape = tuple(a.shape)
    n, n2 = shape
    if n != n2:
        raise ValueError("nystrom_psd needs a square matrix")
    if tm.d != n or tm.k != k:
        raise ValueError(f"test matrix {tm!r} incompatible with A {shape} and k={k}")
    A, kind = _as_device_2d(a)
    _check_psd(A, seed=tm.seed)
    y = _t64(tm.apply_right(A))
    omega = torch.as_tensor(np.ascontiguousarray(tm.materialize()), device=y.device).to(y.dtype)
    nu = np.sqrt(n) * EPS * _spectral_norm(y, seed=tm.seed)
    last_exc = None
    for _ in range(max_shift_retries + 1):
        y_nu = y + nu * omega if nu > 0 else y.clone()
        core = _t64(tm.apply_adjoint(y_nu))
        core = (core + core.conj().T) / 2.0
        try:
            c = _cholesky_upper(core)
        except PositiveDefinitenessError as exc:
            last_exc = exc
            if nu == 0.0:
                nu = np.sqrt(n) * EPS * max(_spectral_norm(y, seed=tm.seed), 1.0)
            nu *= 10.0
            continue
        b = torch.linalg.solve_triangular(c, y_nu, upper=True, left=False)  # X C = Y_nu
        u, s, _ = _svd_econ(b)
        lam = torch.clamp(s ** 2 - nu, min=0.0)
        return _back_factors(EigFactorization(u=u[:, :k], lam=lam[:k]), kind)
    raise PositiveDefinitenessError(f"Cholesky failed after {max_shift_retries} shift increases: {last_exc}")


def _matvec_blocks(A, v, block_rows):
    """A @ v in float64 (LSQR needs residuals below fp32 eps): float32 A streams once through the
    mixed-precision kernel (sk_gemv_f32_f64); float64 A uses cuBLAS."""
    import torch

    if A.dtype == torch.float64:
        return A @ v
    from . import _lib

    v = v.to(torch.float64).contiguous()
    out = torch.empty(A.shape[0], dtype=torch.float64, device=A.device)
    if A.stride(1) != 1:
        A = A.contiguous()
    lib = _lib.load()
    with torch.cuda.device(A.device):
        st = lib.sk_gemv_f32_f64(A.data_ptr(), A.shape[0], A.shape[1], A.stride(0), v.data_ptr(), out.data_ptr(),
                                 torch.cuda.current_stream().cuda_stream)
    _lib.check(st, "sk_gemv_f32_f64")
    return out


def _lsqr_fused_ok(A):
    import torch

    return (A.is_cuda and A.dtype == torch.float32 and A.stride(1) == 1 and A.shape[1] % 128 == 0
            and A.shape[1] <= 512 and A.stride(0) % 4 == 0 and A.data_ptr() % 16 == 0 and A.shape[0] > 0)


def _lsqr_step(A, v, alpha, u):
    """u <- A v - alpha u (in place) and [A^T u_new, ||u_new||^2] in one pass over float32 A
    (sk_lsqr_step_f32_f64): the fused bidiagonalisation step of sketch_precondition_lsqr."""
    import torch

    from . import _lib

    n, d = A.shape
    v = v.to(torch.float64).contiguous()
    zb = torch.empty(d + 1, dtype=torch.float64, device=A.device)
    lib = _lib.load()
    ws_bytes = lib.sk_lsqr_step_f32_f64_workspace_bytes(n, d)
    ws = torch.empty(max(ws_bytes, 8) // 8, dtype=torch.float64, device=A.device)
    with torch.cuda.device(A.device):
        st = lib.sk_lsqr_step_f32_f64(A.data_ptr(), n, d, A.stride(0), v.data_ptr(), float(alpha), u.data_ptr(),
                                      zb.data_ptr(), ws.data_ptr(), ws_bytes, torch.cuda.current_stream().cuda_stream)
    _lib.check(st, "sk_lsqr_step_f32_f64")
    return zb


def _lsqr_fused_loop(A, u, v, R, alpha, beta, bnorm, red, atol, btol, iter_lim, kind, t_sketch):
    """LSQR iterations on the fused step (sk_lsqr_step_f32_f64) with the d-length recurrences on the host.

    Per iteration the device runs one pass over A and the host exchanges two d-vectors with it (R^-1 v
    up, [A^T u, ||u||^2] down: one synchronisation); v, w, x and the scalar recurrences (Paige &
    Saunders, as in the device loop above) are float64 NumPy.  The device u is kept unnormalised
    (u_dev = c u), so the step takes alpha / c and no pass rescales it.  R^-1 is formed once.
    """
    import torch

    d = A.shape[1]
    rinv_h = torch.linalg.solve_triangular(R, torch.eye(d, dtype=R.dtype, device=R.device), upper=True).cpu().numpy()
    vh = v.double().cpu().numpy()
    wh = vh.copy()
    xh = np.zeros(d)
    dev_v = torch.empty(d, dtype=torch.float64, device=A.device)
    c = 1.0  # u on the device is normalised on entry
    phibar, rhobar = beta, alpha
    anorm2 = ddnorm = 0.0
    istop, itn = 0, 0
    r1norm, arnorm, test2 = beta, alpha * beta, 0.0
    while itn < iter_lim:
        itn += 1
        dev_v.copy_(torch.from_numpy(rinv_h @ vh))
        zb = _lsqr_step(A, dev_v, alpha / c, u)
        red(zb)
        zh = zb.cpu().numpy()
        beta = float(np.sqrt(zh[d]))
        if beta > 0:
            c = beta
            anorm2 += alpha * alpha + beta * beta
            vh = (rinv_h.T @ zh[:d]) / beta - beta * vh
            alpha = float(np.linalg.norm(vh))
            if alpha > 0:
                vh /= alpha
        rho = float(np.hypot(rhobar, beta))
        cs, sn = rhobar / rho, beta / rho
        theta = sn * alpha
        rhobar = -cs * alpha
        phi = cs * phibar
        phibar = sn * phibar
        tau = sn * phi
        xh += (phi / rho) * wh
        ddnorm += float(wh @ wh) / (rho * rho)
        wh = vh - (theta / rho) * wh
        anorm = np.sqrt(anorm2)
        r1norm = phibar
        arnorm = alpha * abs(tau)
        test1 = r1norm / bnorm if bnorm > 0 else 0.0
        test2 = arnorm / (anorm * r1norm) if anorm * r1norm > 0 else 0.0
        if test2 <= atol:
            istop = 2
            break
        if btol > 0 and test1 <= btol + atol * anorm * float(np.linalg.norm(xh)) / bnorm:
            istop = 1
            break
    acond = float(np.sqrt(anorm2) * np.sqrt(ddnorm))
    x = torch.from_numpy(rinv_h @ xh).to(A.device)
    return LsqrResult(_back(x, kind), istop, itn, float(r1norm), float(arnorm), acond, t_sketch, float(test2))


_PINNED_SCAL = threading.local()


def _pinned_scal(device):
    """A cached 2 x 8 pinned float64 host buffer per host thread and device (pinning costs far more
    than an iteration; per thread, so concurrent solves — the reference runs trials on a thread pool —
    never share one)."""
    import torch

    cache = getattr(_PINNED_SCAL, "bufs", None)
    if cache is None:
        cache = _PINNED_SCAL.bufs = {}
    key = str(device)
    if key not in cache:
        cache[key] = torch.zeros((2, 8), dtype=torch.float64).pin_memory()
    return cache[key]


def _lsqr_device_loop(A, u, v, R, alpha, beta, bnorm, atol, btol, iter_lim, kind, t_sketch):
    """LSQR iterations with everything on the device: the fused step (one pass over A) and the
    recurrences (sk_lsqr_recur_f64: v, w, x and the Paige & Saunders scalars in one CTA).  The host
    reads 8 scalars per iteration for the stopping test, one iteration behind: iteration i + 1 is
    queued before iteration i's scalars are read, so the GPU never waits for the host — except once
    the normal-equation (or residual) test is within 30x of its tolerance, where the next pass is
    only queued after the check (a pass queued after the stopping iteration would be wasted; it is
    a no-op for x and the state).  Same iterates as
    `_lsqr_fused_loop` up to rounding (float64 everywhere)."""
    import torch

    from . import _lib

    d = A.shape[1]
    dev = A.device
    eye = torch.eye(d, dtype=torch.float64, device=dev)
    rinv = torch.linalg.solve_triangular(R.to(torch.float64), eye, upper=True).contiguous()
    rinvt = rinv.T.contiguous()
    v = v.to(torch.float64).contiguous().clone()
    w = v.clone()
    x = torch.zeros(d, dtype=torch.float64, device=dev)
    vnext = (rinv @ v) / alpha  # u on the device is normalised on entry: c = 1
    state = torch.tensor([alpha, 1.0, beta, alpha, 0.0, 0.0, bnorm, atol, btol, 0.0, 0.0], dtype=torch.float64,
                         device=dev)
    scal = torch.zeros((2, 8), dtype=torch.float64, device=dev)
    scal_h = _pinned_scal(dev)
    evs = [torch.cuda.Event(), torch.cuda.Event()]
    lib = _lib.load()
    n = A.shape[0]
    zb = torch.empty(d + 1, dtype=torch.float64, device=dev)
    ws_bytes = lib.sk_lsqr_step_f32_f64_workspace_bytes(n, d)
    ws = torch.empty(max(ws_bytes, 8) // 8, dtype=torch.float64, device=dev)
    ptrs = [p.data_ptr() for p in (rinv, rinvt, zb, v, w, x, vnext, state)]
    istop, itn = 0, 0
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream().cuda_stream

        def launch(i):  # iteration i (1-based) into scalar slot i % 2
            st = lib.sk_lsqr_step_f32_f64(A.data_ptr(), n, d, A.stride(0), vnext.data_ptr(), 1.0, u.data_ptr(),
                                          zb.data_ptr(), ws.data_ptr(), ws_bytes, stream)
            _lib.check(st, "sk_lsqr_step_f32_f64")
            st = lib.sk_lsqr_recur_f64(d, *ptrs, scal[i % 2].data_ptr(), stream)
            _lib.check(st, "sk_lsqr_recur_f64")
            scal_h[i % 2].copy_(scal[i % 2], non_blocking=True)
            evs[i % 2].record()

        if iter_lim > 0:
            launch(1)
        i, launched = 1, 1
        near = False  # close to the stopping test: no speculative iteration (it would be a wasted pass)
        while i <= iter_lim:
            if launched == i and i < iter_lim and not near:
                launch(i + 1)  # queued behind iteration i: no GPU idle while the host checks i
                launched = i + 1
            evs[i % 2].synchronize()
            itn, istop = int(scal_h[i % 2, 0]), int(scal_h[i % 2, 1])
            r1norm, arnorm, test2, acond = (float(scal_h[i % 2, j]) for j in (2, 3, 4, 5))
            test1 = float(scal_h[i % 2, 6])
            if istop:
                break
            near = test2 <= 30.0 * atol or (btol > 0 and test1 <= 30.0 * btol)
            if launched == i and i < iter_lim:
                launch(i + 1)
                launched = i + 1
            i += 1
    if iter_lim <= 0:
        r1norm, arnorm, test2, acond = beta, alpha * beta, 0.0, 0.0
    return LsqrResult(_back(rinv @ x, kind), istop, itn, r1norm, arnorm, acond, t_sketch, test2)


def _rmatvec_blocks(A, u, block_rows):
    """A^T @ u in float64 (sk_gemv_t_f32_f64 for float32 A: one pass, ordered float64 reduction)."""
    import torch

    if A.dtype == torch.float64:
        return A.T @ u
    from . import _lib

    u = u.to(torch.float64).contiguous()
    if A.stride(1) != 1:
        A = A.contiguous()
    n, d = A.shape
    out = torch.empty(d, dtype=torch.float64, device=A.device)
    lib = _lib.load()
    ws_bytes = lib.sk_gemv_t_f32_f64_workspace_bytes(n, d)
    ws = torch.empty(max(ws_bytes, 8) // 8, dtype=torch.float64, device=A.device)
    with torch.cuda.device(A.device):
        st = lib.sk_gemv_t_f32_f64(A.data_ptr(), n, d, A.stride(0), u.data_ptr(), out.data_ptr(), ws.data_ptr(),
                                   ws_bytes, torch.cuda.current_stream().cuda_stream)
    _lib.check(st, "sk_gemv_t_f32_f64")
    return out


def sketch_precondition_lsqr(a, b, tm_psi, *, atol: float = 1e-6, btol: float = 1e-6, iter_lim: int = 200,
                             block_rows: int = 1 << 16, allreduce=None, _host_scaffold: bool = False) -> LsqrResult:
    """min ||A x - b|| by sketch-and-precondition: S A = Q R, then LSQR on A R^-1.

    `allreduce(t)` (in place sum across ranks) makes the solver distributed: every rank holds a row
    block of A and b, applies its row block of S, and the two reductions per iteration (A^T u and
    the norms) are all-reduced.
    """
    import time

    import torch

    A, kind = _as_device_2d(a, _host_scaffold)
    bt = _as_vec(b, A)
    n, d = A.shape
    if tm_psi.d != n:
        raise ValueError("left test matrix must act on the row space of A")
    red = allreduce if allreduce is not None else (lambda t: t)

    sync = torch.cuda.synchronize if A.is_cuda else (lambda: None)
    sync()
    t0 = time.perf_counter()
    sa = tm_psi.apply_adjoint(A)  # k x d (this rank's partial when distributed)
    sa = _t64(sa)
    red(sa)
    sync()
    t_sketch = time.perf_counter() - t0
    # R of S A = Q R: CholeskyQR2 (two d x d Gram matrices, ~1 ms at config 4) unless S A is too
    # ill-conditioned for it, then Householder QR (cuSOLVER geqrf: 3.9 ms at 2048 x 512)
    qr2 = _cholqr2_qr(sa) if sa.is_cuda else None
    R = qr2[1] if qr2 is not None else torch.linalg.qr(sa, mode="reduced")[1]
    # guard rank deficiency: columns with a vanishing pivot are regularised
    diag = R.diagonal().abs()
    if float(diag.min()) <= DEFAULT_RANK_TOL * float(diag.max()):
        raise np.linalg.LinAlgError("sketched matrix is numerically rank deficient")

    def rinv(v):  # R^-1 v
        return torch.linalg.solve_triangular(R, v[:, None], upper=True)[:, 0]

    def rinvt(v):  # R^-T v
        return torch.linalg.solve_triangular(R.T, v[:, None], upper=False)[:, 0]

    def mv(v):  # (A R^-1) v   (rows of this rank)
        return _matvec_blocks(A, rinv(v), block_rows)

    def rmv(u):  # (A R^-1)^T u   (summed over ranks)
        t = _rmatvec_blocks(A, u, block_rows)
        red(t)
        return rinvt(t)

    def norm(v):
        t = (v.double() ** 2).sum().reshape(1)
        red(t)
        return float(t.sqrt())

    # Paige & Saunders LSQR (damp = 0), bidiagonalisation with the standard estimates
    u = bt.double().clone()
    beta = norm(u)
    bnorm = beta
    x = torch.zeros(d, dtype=torch.float64, device=A.device)
    if beta > 0:
        u /= beta
    v = rmv(u)
    alpha = float(torch.linalg.norm(v))
    if alpha > 0:
        v /= alpha
    w = v.clone()
    phibar, rhobar = beta, alpha
    anorm2 = 0.0
    ddnorm = torch.zeros((), dtype=torch.float64, device=A.device)  # read once at the end (no sync)
    istop, itn = 0, 0
    r1norm, arnorm = beta, alpha * beta
    test1 = test2 = 0.0  # iter_lim = 0 returns the initial estimates
    if arnorm == 0:
        return LsqrResult(_back(rinv(x), kind), 0, 0, r1norm, 0.0, 0.0, t_sketch)
    # float32 A with d = 128 q <= 512: u <- A R^-1 v - alpha u, A^T u and ||u||^2 in one pass over A
    # (sk_lsqr_step_f32_f64), one all-reduce of [A^T u, ||u||^2] per iteration when distributed
    fused = _lsqr_fused_ok(A) and os.environ.get("SKETCH_B200_LSQR_FUSED", "1") != "0"
    if fused and allreduce is None and os.environ.get("SKETCH_B200_LSQR_DEVLOOP", "1") != "0":
        return _lsqr_device_loop(A, u.contiguous(), v, R, alpha, beta, bnorm, atol, btol, iter_lim, kind, t_sketch)
    if fused:
        return _lsqr_fused_loop(A, u.contiguous(), v, R, alpha, beta, bnorm, red, atol, btol, iter_lim, kind,
                                t_sketch)
    while itn < iter_lim:
        itn += 1
        if fused:
            zb = _lsqr_step(A, rinv(v), alpha, u)
            red(zb)
            beta = float(zb[d].sqrt())
            if beta > 0:
                u /= beta
                anorm2 += alpha * alpha + beta * beta
                v = rinvt(zb[:d]) / beta - beta * v
                alpha = float(torch.linalg.norm(v))
                if alpha > 0:
                    v /= alpha
        else:
            u = mv(v) - alpha * u
            beta = norm(u)
            if beta > 0:
                u /= beta
                anorm2 += alpha * alpha + beta * beta
                v = rmv(u) - beta * v
                alpha = float(torch.linalg.norm(v))
                if alpha > 0:
                    v /= alpha
        rho = float(np.hypot(rhobar, beta))
        cs, sn = rhobar / rho, beta / rho
        theta = sn * alpha
        rhobar = -cs * alpha
        phi = cs * phibar
        phibar = sn * phibar
        tau = sn * phi
        x += (phi / rho) * w
        ddnorm += (w ** 2).sum() / (rho * rho)
        w = v - (theta / rho) * w
        anorm = np.sqrt(anorm2)
        r1norm = phibar
        arnorm = alpha * abs(tau)
        test1 = r1norm / bnorm if bnorm > 0 else 0.0
        test2 = arnorm / (anorm * r1norm) if anorm * r1norm > 0 else 0.0
        if test2 <= atol:
            istop = 2
            break
        # btol = 0 disables the consistent-system test: for inconsistent problems (config 4) only the
        # normal-equation test ||(A R^-1)^T r|| <= atol ||A R^-1|| ||r|| may stop the iteration
        if btol > 0 and test1 <= btol + atol * anorm * float(torch.linalg.norm(x)) / bnorm:
            istop = 1
            break
    acond = float(np.sqrt(anorm2) * np.sqrt(float(ddnorm)))
    return LsqrResult(_back(rinv(x), kind), istop, itn, float(r1norm), float(arnorm), acond, t_sketch, float(test2))
