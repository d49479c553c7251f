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

import numpy as np

from ._device import require_cuda, to_operand

__all__ = ["SvdFactorization", "LsqrResult", "orth", "rsvd", "rsvd_residual", "sketch_and_solve",
           "truncated_pinv_apply", "sketch_precondition_lsqr", "EPS", "DEFAULT_RANK_TOL"]

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
    """Orthonormal basis of the numerical range (reference core/factor.py:63-82), on the device."""
    import torch

    m = _t64(m)
    if not bool(torch.isfinite(m).all()):
        raise ValueError("matrix has nonfinite entries")
    if m.shape[1] == 0:
        return m.clone()
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


def _as_device_2d(a):
    import torch

    if isinstance(a, torch.Tensor) and a.dim() == 2 and a.dtype in (torch.float32, torch.float64):
        return a, ("cuda" if a.is_cuda else "tensor")  # torch input stays where it is
    op = to_operand(a, allow_vector=False)
    return op.tensor, op.kind


def _as_vec(b, like):
    import torch

    if isinstance(b, torch.Tensor):
        t = b
    else:
        t = torch.as_tensor(np.asarray(b)).to(like.device)
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
        # second pass over A: B = Q^* A as an fp32/fp64 GEMM in A's precision (no TF32)
        with _no_tf32():
            b = (q.to(A.dtype).conj().T @ A).to(q.dtype)
        u, s, vh = torch.linalg.svd(_t64(b), full_matrices=False)
        fac = SvdFactorization(q @ u.to(q.dtype), s, vh.conj().T)
    if kind in ("numpy", "torch-cpu"):
        return SvdFactorization(_back(fac.u, kind), _back(fac.sigma, kind), _back(fac.v, kind))
    return fac


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
    u, s, vh = torch.linalg.svd(m, full_matrices=False)
    rank = 0 if s.numel() == 0 or float(s[0]) == 0.0 else int((s > rel_tol * s[0]).sum())
    dt = torch.promote_types(m.dtype, b.dtype)
    if rank == 0:
        out = torch.zeros((m.shape[1], b.shape[1]), dtype=dt, device=m.device)
    else:
        core = (u[:, :rank].conj().T.to(dt) @ b.to(dt)) / s[:rank, None]
        out = vh[:rank].conj().T.to(dt) @ core
    return out[:, 0] if squeeze else out


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


def _matvec_blocks(A, v, block_rows):
    """A @ v in float64 (float32 A is widened block by block: LSQR needs residuals below fp32 eps)."""
    import torch

    if A.dtype == torch.float64:
        return A @ v
    out = torch.empty(A.shape[0], dtype=torch.float64, device=A.device)
    for r0 in range(0, A.shape[0], block_rows):
        out[r0:r0 + block_rows] = A[r0:r0 + block_rows].double() @ v
    return out


def _rmatvec_blocks(A, u, block_rows):
    """A^T @ u in float64, accumulated across row blocks."""
    import torch

    if A.dtype == torch.float64:
        return A.T @ u
    out = torch.zeros(A.shape[1], dtype=torch.float64, device=A.device)
    for r0 in range(0, A.shape[0], block_rows):
        out += A[r0:r0 + block_rows].double().T @ u[r0:r0 + block_rows]
    return out


def sketch_precondition_lsqr(a, b, tm_psi, *, atol: float = 1e-6, btol: float = 1e-6, iter_lim: int = 200,
                             block_rows: int = 1 << 16, allreduce=None) -> LsqrResult:
    """min ||A x - b|| by sketch-and-precondition: S A = Q R, then LSQR on A R^-1.

    `allreduce(t)` (in place sum across ranks) makes the solver distributed: every rank holds a row
    block of A and b, applies its row block of S, and the two reductions per iteration (A^T u and
    the norms) are all-reduced.
    """
    import time

    import torch

    A, kind = _as_device_2d(a)
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
    _, R = torch.linalg.qr(sa, mode="reduced")
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
    anorm2, ddnorm = 0.0, 0.0
    istop, itn = 0, 0
    r1norm, arnorm = beta, alpha * beta
    if arnorm == 0:
        return LsqrResult(_back(rinv(x), kind), 0, 0, r1norm, 0.0, 0.0, t_sketch)
    while itn < iter_lim:
        itn += 1
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
        ddnorm += float((w ** 2).sum()) / (rho * rho)
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
    acond = float(np.sqrt(anorm2) * np.sqrt(ddnorm))
    return LsqrResult(_back(rinv(x), kind), istop, itn, float(r1norm), float(arnorm), acond, t_sketch, float(test2))
