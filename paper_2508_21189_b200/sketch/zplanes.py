"""Complex-field applies on the float64 DMMA engine (K5d, `sk_kr_right_z` / `sk_kr_adjoint_z`).

The reference's default Khatri-Rao base is complex_spherical (sketch/khatri_rao.py:101) and its
Gaussian family has a complex field (sketch/gaussian.py:19-30); their applies compute in complex128
(core/containers.py:41-46).  A complex product is formed from real products over planar data:

    right    Y = A Omega:    Re Y = Ar Re(O) - Ai Im(O),   Im Y = Ar Im(O) + Ai Re(O)
    adjoint  X = Omega^H B:  Re X = Re(O)^T Br + Im(O)^T Bi, Im X = Re(O)^T Bi - Im(O)^T Br

with Omega = W (x) F given by the planes of its Khatri-Rao factors (the engine synthesises the
requested part of W[P, :] * F[q, :] in shared memory) or, for one block (W = NULL), a dense Omega
whose planes are F itself.  float64 / complex128 inputs only (complex64 keeps the torch path).
"""

from __future__ import annotations

import numpy as np

from .. import _lib

__all__ = ["ZOperands", "z_operands", "z_apply"]


class ZOperands:
    """Device planes of a complex Omega: F (dl x k) and W (P x k; None for one dense block), row
    strides padded to an even number of float64 (16-byte rows for the engine's vector loads)."""

    def __init__(self, fr, fi, wr, wi, P: int, dl: int, k: int):
        self.fr, self.fi, self.wr, self.wi = fr, fi, wr, wi
        self.P, self.dl, self.k = P, dl, k


def _padded_plane(x, device):
    """float64 2-D device tensor with unit column stride, an even row stride and a 16-byte base."""
    import torch

    x = torch.as_tensor(x, device=device, dtype=torch.float64) if not isinstance(x, torch.Tensor) else x
    r, c = x.shape
    if x.stride(1) == 1 and x.stride(0) % 2 == 0 and x.stride(0) >= c and x.data_ptr() % 16 == 0:
        return x
    out = torch.zeros((r, c + (c & 1)), dtype=torch.float64, device=x.device)
    out[:, :c] = x
    return out


def z_operands(w, f, device) -> ZOperands:
    """Planes of W (P x k complex, or None) and F (dl x k complex) on `device`."""
    k = f.shape[1]

    def planes(m):
        return (_padded_plane(np.ascontiguousarray(m.real), device), _padded_plane(np.ascontiguousarray(m.imag), device))

    fr, fi = planes(f)
    if w is None:
        return ZOperands(fr, fi, None, None, 1, f.shape[0], k)
    wr, wi = planes(w)
    return ZOperands(fr, fi, wr, wi, w.shape[0], f.shape[0], k)


def z_apply(ops: ZOperands, x, adjoint: bool, scale: float):
    """scale * (x Omega) (right, x: n x P*dl) or scale * Omega^H x (adjoint, x: P*dl x m); x float64 or
    complex128 on the device; returns complex128."""
    import torch

    lib = _lib.load()
    rows = x.shape[1] if adjoint else x.shape[0]
    shape = (ops.k, rows) if adjoint else (rows, ops.k)
    out_r = torch.empty(shape, dtype=torch.float64, device=x.device)
    out_i = torch.empty(shape, dtype=torch.float64, device=x.device)
    if rows == 0:
        return torch.complex(out_r, out_i)
    if x.is_complex():
        xv = torch.view_as_real(x.to(torch.complex128))
        xr, xi = _padded_plane(xv[..., 0], x.device), _padded_plane(xv[..., 1], x.device)
    else:
        xr, xi = _padded_plane(x.to(torch.float64), x.device), None
    fn = lib.sk_kr_adjoint_z if adjoint else lib.sk_kr_right_z
    stream = torch.cuda.current_stream(x.device).cuda_stream

    def call(xp, part, s, acc, out):
        if ops.wr is None:  # dense Omega: its planes are F
            f, fi, w, wi, ldw = (ops.fr if part == 0 else ops.fi), None, None, None, 0
        else:
            f, fi, w, wi, ldw = ops.fr, ops.fi.data_ptr(), ops.wr.data_ptr(), ops.wi.data_ptr(), ops.wr.stride(0)
        st = fn(xp.data_ptr(), rows, ops.P, ops.dl, xp.stride(0), f.data_ptr(), fi, f.stride(0), w, wi, ldw, ops.k,
                part, float(s), acc, out.data_ptr(), out.stride(0), stream)
        _lib.check(st, "sk_kr_adjoint_z" if adjoint else "sk_kr_right_z")

    with torch.cuda.device(x.device):
        if not adjoint:
            call(xr, 0, scale, 0, out_r)
            call(xr, 1, scale, 0, out_i)
            if xi is not None:
                call(xi, 1, -scale, 1, out_r)
                call(xi, 0, scale, 1, out_i)
        else:
            call(xr, 0, scale, 0, out_r)
            call(xr, 1, -scale, 0, out_i)
            if xi is not None:
                call(xi, 1, scale, 1, out_r)
                call(xi, 0, scale, 1, out_i)
    return torch.complex(out_r, out_i)
