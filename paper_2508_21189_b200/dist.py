"""Row-block multi-GPU execution of the sketch path (one process per GPU, torch.distributed/NCCL).

Work is partitioned by row blocks of A:
  * Y = A Omega needs no communication — every rank applies Omega to its own rows.
  * S A = Omega^* A sums the per-rank partials Omega[rows_g]^* A_g with ONE all-reduce
    (NCCL over NVLink/NVSwitch; 2048 x 512 fp32 = 4 MiB at config 4).
  * the randomized SVD orthonormalises the row-sharded Y with CholeskyQR2 (two all-reduced
    float64 Gram matrices) and forms B = sum_g Q_g^* A_g with one all-reduce.
  * sketch-and-precondition LSQR all-reduces A^T u and the norms once per iteration.
Every helper degrades to the single-process path when torch.distributed is not initialised.
"""

from __future__ import annotations

import numpy as np

__all__ = ["row_range", "world", "allreduce_sum", "sharded_right", "sharded_adjoint", "cholesky_qr2",
           "sharded_rsvd", "sharded_lsqr"]


def world(group=None):
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def row_range(n: int, world_size: int, rank: int):
    """Contiguous, balanced row block [r0, r1) of rank `rank` among `world_size`."""
    base, extra = divmod(n, world_size)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def allreduce_sum(t, group=None):
    """In-place sum across ranks (no-op in a single process)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def sharded_right(tm, a_local):
    """Y_g = A_g Omega: purely local (no collective)."""
    return tm.apply_right(a_local)


def _row_block_of(tm, r0: int, rows: int):
    """Rows [r0, r0 + rows) of `tm` (sparse families); other families have no row blocks."""
    if not hasattr(tm, "row_block"):
        raise NotImplementedError(f"{type(tm).__name__} has no row blocks: row-sharded adjoints need a sparse "
                                  "test matrix (SparseUniformTM, SparseStackTM, SparseIIDTM, SparseColTM)")
    return tm.row_block(r0, r0 + rows)


def sharded_adjoint(tm, a_local, r0: int, group=None, dtype=None):
    """S A summed over ranks: rank g applies Omega[r0 : r0 + n_g]^* to its rows, then all-reduce."""
    import torch

    blk = _row_block_of(tm, r0, a_local.shape[0])
    part = blk.apply_adjoint(a_local)
    if dtype is not None:
        part = part.to(dtype)
    elif part.dtype == torch.float32:
        part = part.to(torch.float64)  # reduce partial sums in float64
    return allreduce_sum(part, group)


def cholesky_qr2(y_local, group=None):
    """Orthonormal Q_g for the row-sharded Y (CholeskyQR2: two all-reduced Gram matrices, float64)."""
    import torch

    q = y_local.to(torch.float64)
    for _ in range(2):
        g = q.T @ q
        allreduce_sum(g, group)
        r = torch.linalg.cholesky(g, upper=True)
        q = torch.linalg.solve_triangular(r, q, upper=True, left=False)
    return q


def sharded_rsvd(a_local, k: int, tm, group=None):
    """Randomized SVD of a row-sharded A: returns (U_g, sigma, V) with U_g this rank's rows."""
    import torch

    from .rand_nla import SvdFactorization, _qt_a

    y = tm.apply_right(a_local)
    q = cholesky_qr2(y, group)
    b = _qt_a(q, a_local).to(torch.float64)  # this rank's Q_g^T A_g (tensor cores for float32 CUDA)
    allreduce_sum(b, group)
    u, s, vh = torch.linalg.svd(b, full_matrices=False)
    return SvdFactorization(q @ u, s, vh.T)


def sharded_residual(a_local, fac, group=None, block_rows: int = 8192) -> float:
    """Relative Frobenius residual ||A - U S V^T|| / ||A|| of a row-sharded A (float64 sums)."""
    import torch

    from .rand_nla import _no_tf32

    w = (fac.sigma[None, :] * fac.v).T.to(a_local.dtype)
    acc = torch.zeros(2, dtype=torch.float64, device=a_local.device)
    with _no_tf32():
        for s0 in range(0, a_local.shape[0], block_rows):
            blk = a_local[s0:s0 + block_rows]
            res = blk - fac.u[s0:s0 + block_rows].to(a_local.dtype) @ w
            acc[0] += (res.double() ** 2).sum()
            acc[1] += (blk.double() ** 2).sum()
    allreduce_sum(acc, group)
    return float(torch.sqrt(acc[0] / acc[1])) if float(acc[1]) > 0 else 0.0


def sharded_lsqr(a_local, b_local, tm, r0: int, group=None, **kw):
    """Sketch-and-precondition LSQR over row-sharded (A, b): every rank returns the same x."""
    from .rand_nla import sketch_precondition_lsqr

    blk = _row_block_of(tm, r0, a_local.shape[0])
    return sketch_precondition_lsqr(a_local, b_local, blk, allreduce=lambda t: allreduce_sum(t, group), **kw)
