"""Operand plumbing between the reference-style API and the CUDA library.

`apply_right(A)` / `apply_adjoint(B)` accept what the reference accepts (NumPy arrays, SciPy
sparse matrices) plus torch tensors.  Host operands are uploaded to the current CUDA device,
the kernel runs there, and the result comes back in the caller's container; CUDA tensors stay
on the device.  There is no CPU compute path: without a CUDA device every apply raises.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None


class NoDeviceError(RuntimeError):
    """The B200 sketch path needs a CUDA device; there is no CPU fallback."""


def require_cuda():
    if torch is None or not torch.cuda.is_available():
        raise NoDeviceError("paper_2508_21189_b200 applies run on a CUDA device only (none visible)")


@dataclass
class Operand:
    tensor: "torch.Tensor"  # 2-D, on the CUDA device, unit column stride
    kind: str  # "numpy" | "torch-cpu" | "cuda"
    squeeze: bool  # a 1-D input was promoted to a column
    pinned: bool = False


def current_stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def _compute_dtype(dt, complex_ok: bool):
    if dt in (torch.float32, torch.float64):
        return dt
    if complex_ok and dt in (torch.complex64, torch.complex128):
        return dt
    if dt.is_complex:
        return torch.complex128
    return torch.float64


def to_operand(x, *, allow_vector: bool, complex_ok: bool = True) -> Operand:
    """Normalise A/B to a row-major CUDA tensor (float32/float64, or complex for library paths)."""
    require_cuda()
    squeeze = False
    if hasattr(x, "toarray") and not isinstance(x, np.ndarray) and not (torch is not None and isinstance(x, torch.Tensor)):
        x = x.toarray()  # scipy sparse -> dense (reference: sketch/base.py:83-84, sparse.py:63-66)
    if isinstance(x, torch.Tensor):
        kind = "cuda" if x.is_cuda else "torch-cpu"
        t = x
        pinned = (not x.is_cuda) and x.is_pinned()
    else:
        arr = np.asarray(x)
        if arr.dtype == object:
            raise TypeError("unsupported operand dtype object")
        kind = "numpy"
        t = torch.from_numpy(np.ascontiguousarray(arr))
        pinned = False
    if t.dim() == 1:
        if not allow_vector:
            raise ValueError(f"expected a 2-d operand, got shape {tuple(t.shape)}")
        t = t[:, None]
        squeeze = True
    if t.dim() != 2:
        raise ValueError(f"expected a 2-d operand, got shape {tuple(t.shape)}")
    dt = _compute_dtype(t.dtype, complex_ok)
    if not t.is_cuda:
        t = t.to(device=torch.device("cuda", torch.cuda.current_device()), dtype=dt, non_blocking=pinned)
    elif t.dtype != dt:
        t = t.to(dt)
    if t.shape[1] > 1 and t.stride(1) != 1 or (t.shape[0] > 1 and t.stride(0) < t.shape[1]):
        t = t.contiguous()
    return Operand(t, kind, squeeze, pinned)


def from_result(y: "torch.Tensor", op: Operand):
    """Return in the caller's container: NumPy (float64/complex128, as the reference) or torch."""
    if op.squeeze:
        y = y[:, 0]
    if op.kind == "cuda":
        return y
    if op.kind == "torch-cpu":
        return y.cpu()
    host = y.cpu().numpy()
    if np.iscomplexobj(host):
        return host.astype(np.complex128, copy=False)
    return host.astype(np.float64, copy=False)
