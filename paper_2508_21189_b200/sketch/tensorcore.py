"""Dense tensor-core apply (K-TC, `sk_dense_right_tc`) and the device forms of Omega^T it consumes.

The kernel computes Y = scale * A * B for float32 A with B supplied as B^T in bf16 (k x d, rows
padded to a multiple of 8 elements).  +-1 matrices (sparse sign) are exact in bf16, so only A is
split (hi + lo); general matrices (Gaussian) also pass the bf16 residual of B.  Khatri-Rao has its
own entry (sk_kr_right, sketch/kron.py) that never forms Omega.  The kernel tiles N in blocks of <= 256 columns and splits K across
CTAs (workspace + ordered reduction) when there are too few row tiles to fill the GPU.
"""

from __future__ import annotations

import numpy as np

from .. import _lib

__all__ = ["dense_right_tc", "dense_tn_tc", "split_wt", "bt_from_triplets", "bt_from_dense"]

MAX_K = 512


def _pad8(d: int) -> int:
    return (d + 7) // 8 * 8


def bt_from_triplets(rows, cols, neg, d: int, k: int, device):
    """Exact +-1 bf16 B^T (k x ldb) from sparse triplets (duplicates add; sign-sparse families)."""
    import torch

    ldb = _pad8(d)
    bt = torch.zeros((k, ldb), dtype=torch.float32, device=device)
    r = torch.as_tensor(np.asarray(rows, dtype=np.int64), device=device)
    c = torch.as_tensor(np.asarray(cols, dtype=np.int64), device=device)
    v = torch.as_tensor(np.where(np.asarray(neg, dtype=bool), -1.0, 1.0).astype(np.float32), device=device)
    bt.index_put_((c, r), v, accumulate=True)
    exact = bool(torch.all(bt.abs() <= 256).item())  # small integers are exact in bf16
    if not exact:
        raise ValueError("sparse pattern not exactly representable in bf16")
    return bt.to(torch.bfloat16), None


def bt_from_dense(omega: np.ndarray, device):
    """bf16 hi + lo split of a general float64 d x k Omega, transposed (k x ldb)."""
    import torch

    d, k = omega.shape
    ldb = _pad8(d)
    om = torch.zeros((k, ldb), dtype=torch.float64, device=device)
    om[:, :d] = torch.as_tensor(np.ascontiguousarray(omega.T), device=device)
    hi = om.to(torch.bfloat16)
    lo = (om - hi.to(torch.float64)).to(torch.bfloat16)
    if bool(torch.all(lo == 0).item()):
        return hi, None
    return hi, lo


def dense_right_tc(a, bt_hi, bt_lo, k: int, scale: float):
    """Y = scale * a @ B for float32 CUDA `a` (n x d) and B^T given as bf16 (k x ldb) [+ residual]."""
    import torch

    if a.dtype != torch.float32:
        raise TypeError("dense_right_tc needs float32 A")
    n, d = a.shape
    if a.stride(1) != 1 or a.stride(0) % 4 or a.data_ptr() % 16 or d % 4:
        a = a.contiguous()
        if d % 4:
            raise ValueError("dense_right_tc needs d % 4 == 0")
    y = torch.empty((n, k), dtype=torch.float32, device=a.device)
    if n == 0:
        return y
    lib = _lib.load()
    stream = torch.cuda.current_stream(a.device).cuda_stream  # the operand's device, not the current one
    ldb = bt_hi.stride(0)
    ws_bytes = lib.sk_dense_tc_workspace_bytes(n, d, k, 1 if bt_lo is not None else 0)
    ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=a.device)
    with torch.cuda.device(a.device):
        st = lib.sk_dense_right_tc(a.data_ptr(), n, d, a.stride(0), bt_hi.data_ptr(),
                                   bt_lo.data_ptr() if bt_lo is not None else None, ldb, k, float(scale),
                                   y.data_ptr(), y.stride(0), ws.data_ptr(), ws_bytes, stream)
    _lib.check(st, "sk_dense_right_tc")
    return y


def split_wt(w, device):
    """W^T as bf16 hi + lo (k x ldw, ldw = n rounded up to 8) for dense_tn_tc, from a float n x k W."""
    import torch

    n, k = w.shape
    wt = torch.zeros((k, _pad8(n)), dtype=torch.float64, device=device)
    wt[:, :n] = torch.as_tensor(w, device=device).T.to(torch.float64)
    hi = wt.to(torch.bfloat16)
    lo = (wt - hi.to(torch.float64)).to(torch.bfloat16)
    return hi, lo


def dense_tn_tc(a, w=None, scale: float = 1.0, *, wt=None):
    """scale * a^T @ w on the tensor cores (sk_dense_tn_tc) for float32 CUDA `a` (n x d), read in place,
    and a float32/float64 `w` (n x k) or its precomputed split `wt` = (hi, lo) from split_wt: BF16x3,
    fp32 accumulation in bounded chunks. Returns (d x k)."""
    import torch

    if a.dtype != torch.float32 or not a.is_cuda:
        raise TypeError("dense_tn_tc needs a float32 CUDA A")
    n, d = a.shape
    if n == 0 or d == 0:
        k = (wt[0].shape[0] if wt is not None else w.shape[1])
        return torch.zeros((d, k), dtype=torch.float32, device=a.device)
    if a.stride(1) != 1 or a.stride(0) % 4 or a.data_ptr() % 16 or d % 4:
        if d % 4:  # ragged column count: zero-padded copy (the extra columns give zero rows of the result)
            pad = torch.zeros((n, d + (-d) % 4), dtype=a.dtype, device=a.device)
            pad[:, :d] = a
            return dense_tn_tc(pad, w, scale, wt=wt)[:d]
        a = a.contiguous()
    if wt is None:
        wt = split_wt(w.to(device=a.device), a.device)
        wt = (wt[0], wt[1])
    hi, lo = wt
    k = hi.shape[0]
    ldw = hi.stride(0)
    y = torch.empty((d, k), dtype=torch.float32, device=a.device)
    lib = _lib.load()
    stream = torch.cuda.current_stream(a.device).cuda_stream
    ws_bytes = lib.sk_dense_tn_tc_workspace_bytes(n, d, k)
    ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=a.device)
    with torch.cuda.device(a.device):
        st = lib.sk_dense_tn_tc(a.data_ptr(), n, d, a.stride(0), hi.data_ptr(), lo.data_ptr(), ldw, k, float(scale),
                                y.data_ptr(), y.stride(0), ws.data_ptr(), ws_bytes, stream)
    _lib.check(st, "sk_dense_tn_tc")
    return y
