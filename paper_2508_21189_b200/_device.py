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
    if not t.is_cuda and not pinned and t.numel() * t.element_size() >= STAGED_UPLOAD_MIN_BYTES:
        t = _upload_staged(t, torch.device("cuda", torch.cuda.current_device()), dt)
    elif not t.is_cuda:
        t = t.to(device=torch.device("cuda", torch.cuda.current_device()), dtype=dt, non_blocking=pinned)
    elif t.dtype != dt:
        t = t.to(dt)
    if t.shape[1] > 1 and t.stride(1) != 1 or (t.shape[0] > 1 and t.stride(0) < t.shape[1]):
        t = t.contiguous()
    return Operand(t, kind, squeeze, pinned)


STAGED_UPLOAD_MIN_BYTES = 64 << 20


def _upload_staged(t, dev, dt):
    """Pageable host tensor -> device through a pinned double buffer of 128 MB chunks: torch's
    multi-threaded host copy (with the dtype conversion) into one buffer while the other's H2D runs
    on a side stream (a pageable cudaMemcpy runs through the driver's own staging at a fraction of
    the PCIe rate)."""
    if t.dim() == 1 or not t.is_contiguous():
        t = t.reshape(t.shape[0], -1).contiguous() if t.dim() != 1 else t.contiguous()
    out = torch.empty(t.shape, dtype=dt, device=dev)
    row_bytes = max(1, (t.numel() // max(1, t.shape[0])) * out.element_size())
    rows = max(1, PIPELINE_CHUNK_BYTES // row_bytes)
    n = t.shape[0]
    stage = [torch.empty((min(rows, n),) + tuple(t.shape[1:]), dtype=dt, pin_memory=True) for _ in range(2)]
    evs = [torch.cuda.Event(), torch.cuda.Event()]
    side = _pipeline_streams(dev)[0]
    cur = torch.cuda.current_stream(dev)
    side.wait_stream(cur)
    for i, r0 in enumerate(range(0, n, rows)):
        b = i % 2
        m = min(rows, n - r0)
        if i >= 2:
            evs[b].synchronize()  # the H2D out of this buffer has finished
        stage[b][:m].copy_(t[r0:r0 + m])
        with torch.cuda.stream(side):
            out[r0:r0 + m].copy_(stage[b][:m], non_blocking=True)
            evs[b].record(side)
    cur.wait_stream(side)
    for e in evs:
        e.synchronize()  # the staging buffers return to the pinned cache only when their copies are done
    return out


def from_result(y: "torch.Tensor", op: Operand):
    """Return in the caller's container: NumPy (float64/complex128, as the reference) or torch."""
    if op.squeeze:
        y = y[:, 0]
    if op.kind == "cuda":
        return y
    if op.kind == "torch-cpu":
        return y.cpu()
    # widen before the copy back (on the device: a NumPy astype of a large result runs single-threaded)
    y = y.to(torch.complex128 if y.is_complex() else torch.float64)
    return y.cpu().numpy()


PIPELINE_MIN_BYTES = 256 << 20  # host operands at least this large stream through the device in chunks
PIPELINE_CHUNK_BYTES = 128 << 20


def host_tensor_of(x):
    """(torch CPU tensor view of x, kind) for host operands, or (None, None) for device tensors."""
    if torch is None:
        return None, None
    if isinstance(x, torch.Tensor):
        return (None, None) if x.is_cuda else (x, "torch-cpu")
    arr = np.asarray(x)
    if arr.dtype == object:
        raise TypeError("unsupported operand dtype object")
    return torch.from_numpy(np.ascontiguousarray(arr)), "numpy"


_STREAMS = {}


def _pipeline_streams(dev):
    """Three streams per device, created once: the caching allocator keeps per-stream pools, so
    fresh streams every call would turn each chunk's output allocation into a cudaMalloc."""
    key = dev.index
    if key not in _STREAMS:
        _STREAMS[key] = tuple(torch.cuda.Stream(dev) for _ in range(3))
    return _STREAMS[key]


def pipelined_right(apply_dev, host, k: int):
    """Row-chunked host -> device -> host pipeline for a row-independent right apply.

    Three CUDA streams overlap the H2D copy of chunk i+1, the kernel on chunk i and the D2H copy of
    chunk i-1, so an end-to-end call runs at the PCIe rate instead of copy + compute + copy.
    Pageable inputs are staged through a pinned double buffer.
    """
    require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    n, d = host.shape
    dt = _compute_dtype(host.dtype, complex_ok=False)
    esz = torch.empty((), dtype=dt).element_size()
    rows = max(1, min(n, PIPELINE_CHUNK_BYTES // max(1, d * esz)))
    pinned = host.is_pinned() and host.dtype == dt and host.is_contiguous()
    y_host = None
    s_h2d, s_cmp, s_d2h = _pipeline_streams(dev)
    outer = torch.cuda.current_stream(dev)
    for s in (s_h2d, s_cmp, s_d2h):
        s.wait_stream(outer)
    bufs = [torch.empty((rows, d), dtype=dt, device=dev) for _ in range(2)]
    stage = None if pinned else [torch.empty((rows, d), dtype=dt, pin_memory=True) for _ in range(2)]
    ev_loaded = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    ev_staged = [torch.cuda.Event() for _ in range(2)]
    used = [False, False]
    keep = []
    for i, r0 in enumerate(range(0, n, rows)):
        b = i % 2
        m = min(rows, n - r0)
        with torch.cuda.stream(s_h2d):
            if used[b]:
                s_h2d.wait_event(ev_free[b])
            if pinned:
                src = host[r0:r0 + m]
            else:
                if used[b]:
                    ev_staged[b].synchronize()  # the previous H2D out of this staging buffer is done
                src = stage[b][:m]
                src.copy_(host[r0:r0 + m])
            bufs[b][:m].copy_(src, non_blocking=True)
            ev_loaded[b].record(s_h2d)
            if not pinned:
                ev_staged[b].record(s_h2d)
        with torch.cuda.stream(s_cmp):
            s_cmp.wait_event(ev_loaded[b])
            y = apply_dev(bufs[b][:m])
            ev_free[b].record(s_cmp)
        if y_host is None:
            y_host = torch.empty((n, y.shape[1]), dtype=y.dtype, pin_memory=True)
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_stream(s_cmp)
            y_host[r0:r0 + m].copy_(y, non_blocking=True)
        # keep the chunk result alive until the end of the call instead of record_stream: blocks
        # come back to the caching allocator only after the final synchronize, so steady-state
        # calls reuse them (record_stream let the pool grow and occasionally hit cudaMalloc/cudaFree)
        keep.append(y)
        used[b] = True
    for s in (s_h2d, s_cmp, s_d2h):
        outer.wait_stream(s)
    s_d2h.synchronize()
    s_cmp.synchronize()
    del keep
    if y_host is None:
        y_host = torch.empty((0, k), dtype=dt)
    return y_host


def transposed(x):
    """A fresh row-major copy of x^T (standard strides even when a dimension is 1)."""
    out = torch.empty((x.shape[1], x.shape[0]), dtype=x.dtype, device=x.device)
    out.copy_(x.T)
    return out
