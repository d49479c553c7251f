"""Trigonometric transforms and the sparse randomized trigonometric transform (SRTT) on the B200.

SparseRttTM restates src/sketch/rtt.py:75-186: Omega = D F S with a random diagonal D drawn
from stream (SparseRttTM, "diagonal"), a unitary transform F (WHT / DCT / DFT) and a SparseColTM
sampler S with the same seed.  The real WHT right-apply — BASELINE config 2 — runs as one fused
kernel (K3, `sk_srtt_right`): sign flip, in-register/shared-memory Walsh-Hadamard butterflies and
the sampled gather in a single pass over A.  Other transforms / fields use the dense device GEMM.

`wht` on device arrays reuses the same kernel with the identity sampler (k = d, xi = 1).
"""

from __future__ import annotations

import math

import numpy as np
import scipy.fft

from .. import _lib
from .._device import from_result, to_operand
from .encode import srtt_sampler_encode
from .sparse_rows import SparseColTM
from .tensorcore import bt_from_dense, dense_right_tc, dense_tn_tc, split_wt
from .testmatrix import TestMatrix, entry_sample

__all__ = ["wht", "dct2_ortho", "dft_unitary", "dct3_rows", "SparseRttTM", "TRANSFORMS"]


def _require_pow2(d: int) -> int:
    m = d.bit_length() - 1
    if d <= 0 or (1 << m) != d:
        raise ValueError(f"WHT requires a power-of-two length, got {d}")
    return m


def _wht_host(x, axis: int = 0) -> np.ndarray:
    """Host WHT (1/sqrt(d) normalised) used only by `materialize` for small diagnostic matrices."""
    x = np.asarray(x, dtype=np.result_type(x, np.float64))
    d = x.shape[axis]
    _require_pow2(d)
    y = np.moveaxis(x, axis, 0).reshape(d, -1).copy()
    h = 1
    while h < d:
        v = y.reshape(d // (2 * h), 2, h, -1)
        y = np.concatenate([v[:, :1] + v[:, 1:], v[:, :1] - v[:, 1:]], axis=1).reshape(d, -1)
        h *= 2
    y = (y / np.sqrt(d)).reshape(np.moveaxis(x, axis, 0).shape)
    return np.moveaxis(y, 0, axis)


def _identity_sampler(d: int):
    return srtt_sampler_encode(np.arange(d)[:, None], np.zeros((d, 1), bool))


_SEG_L = 12  # segment length 2^12 for the two-level transform of long rows


def _large_rows(d: int, dtype) -> bool:
    """Rows longer than the single-pass kernels take (float32 d > 2^14, float64 d > 2^13)."""
    import torch

    return d > ((1 << 14) if dtype == torch.float32 else (1 << 13))


def _wht_segments(x):
    """Unnormalised WHT of every length-2^12 segment of the rows of a contiguous device tensor."""
    n, d = x.shape
    seg = 1 << _SEG_L
    z = _srtt_native(x.reshape(-1, seg), np.ones(seg), _identity_sampler(seg), 1, seg, 1.0, pm1=True)
    return z.view(n, d // seg, seg)


def _hadamard_signs(rows_hi, d1: int, device, dtype):
    """(-1)^popcount(r & a) for r in rows_hi, a < d1: the H_{d1} rows the sampled outputs need."""
    import torch

    a = torch.arange(d1, device=device)
    bits = torch.bitwise_and(rows_hi[:, None], a[None, :])
    par = torch.zeros_like(bits)
    while bool(bits.any()):
        par ^= bits & 1
        bits = bits >> 1
    return (1 - 2 * par).to(dtype)


def _wht_rows_large(x):
    """Unnormalised WHT of long rows: H_d = H_{d/2^12} (x) H_{2^12} (index j = 2^12 a + b) — the
    segment transforms run in the K3 kernel, the short outer transform as an exact +-1 contraction."""
    import torch

    n, d = x.shape
    z = _wht_segments(x.contiguous())
    d1 = z.shape[1]
    h = _hadamard_signs(torch.arange(d1, device=x.device), d1, x.device, x.dtype)
    return torch.einsum("ra,nab->nrb", h, z).reshape(n, d)


def wht(x, axis: int = 0):
    """Walsh-Hadamard transform with 1/sqrt(d) normalisation (self-inverse), computed on the GPU.

    Same contract as reference src/sketch/rtt.py:28-44 (rejects non-power-of-two lengths).
    Real NumPy input returns float64 NumPy; torch input returns torch.
    """
    import torch

    shape = np.shape(x) if not isinstance(x, torch.Tensor) else tuple(x.shape)
    if len(shape) == 0:
        raise ValueError("wht needs at least a 1-d array")
    d = shape[axis]
    _require_pow2(int(d))
    if isinstance(x, np.ndarray) and np.iscomplexobj(x):  # real and imaginary parts on the device
        return wht(np.ascontiguousarray(x.real), axis) + 1j * wht(np.ascontiguousarray(x.imag), axis)
    if isinstance(x, torch.Tensor) and x.is_complex():
        return torch.complex(wht(x.real, axis), wht(x.imag, axis))
    if isinstance(x, torch.Tensor):
        t = torch.movedim(x, axis, -1)
        lead = t.shape[:-1]
        op = to_operand(t.reshape(-1, d), allow_vector=False, complex_ok=False)
        if _large_rows(d, op.tensor.dtype):
            y = _wht_rows_large(op.tensor) / np.sqrt(d)
        else:
            y = _srtt_native(op.tensor, np.ones(d), _identity_sampler(d), 1, d, 1.0 / np.sqrt(d), pm1=True)
        return torch.movedim(from_result(y, op).reshape(*lead, d), -1, axis)
    t = np.moveaxis(np.asarray(x, dtype=np.float64), axis, -1)
    lead = t.shape[:-1]
    op = to_operand(np.ascontiguousarray(t.reshape(-1, d)), allow_vector=False, complex_ok=False)
    if _large_rows(d, op.tensor.dtype):
        y = _wht_rows_large(op.tensor) / np.sqrt(d)
    else:
        y = _srtt_native(op.tensor, np.ones(d), _identity_sampler(d), 1, d, 1.0 / np.sqrt(d), pm1=True)
    return np.moveaxis(from_result(y, op).reshape(*lead, d), -1, axis)


def dct2_ortho(x, axis: int = 0) -> np.ndarray:
    """Orthonormal DCT-II (reference rtt.py:47-49); host SciPy, used for materialize/diagnostics."""
    return scipy.fft.dct(np.asarray(x), type=2, norm="ortho", axis=axis)


def dft_unitary(x, axis: int = 0) -> np.ndarray:
    """Unitary DFT (reference rtt.py:52-55); host NumPy, used for materialize/diagnostics."""
    x = np.asarray(x)
    return np.fft.fft(x, axis=axis) / np.sqrt(x.shape[axis])


def _dct2_adjoint(x, axis: int = 0) -> np.ndarray:
    return scipy.fft.dct(np.asarray(x), type=3, norm="ortho", axis=axis)


def _dft_adjoint(x, axis: int = 0) -> np.ndarray:
    x = np.asarray(x)
    return np.fft.ifft(x, axis=axis) * np.sqrt(x.shape[axis])


TRANSFORMS = {
    "wht": (_wht_host, _wht_host, False),
    "dct": (dct2_ortho, _dct2_adjoint, False),
    "dft": (dft_unitary, _dft_adjoint, True),
}


def _srtt_native(a, dvals, samp, xi: int, k: int, scale: float, pm1: bool, transform: int = _lib.SK_WHT):
    """Launch sk_srtt_right on a row-major CUDA tensor `a` (n x d); dvals/samp: host or device arrays."""
    import torch

    code = _lib.SK_F32 if a.dtype == torch.float32 else _lib.SK_F64
    n, d = a.shape
    dv = dvals if isinstance(dvals, torch.Tensor) else torch.as_tensor(np.asarray(dvals, dtype=np.float64))
    dv = dv.to(device=a.device, dtype=a.dtype)
    sp = samp if isinstance(samp, torch.Tensor) else torch.as_tensor(np.asarray(samp, dtype=np.int32))
    sp = sp.to(a.device)
    y = torch.empty((n, k), dtype=a.dtype, device=a.device)
    if n == 0:
        return y
    lib = _lib.load()
    flags = transform | (_lib.SK_DIAG_PM1 if pm1 else 0)
    with torch.cuda.device(a.device):
        st = lib.sk_srtt_right(code, a.data_ptr(), n, d, a.stride(0), dv.data_ptr(), flags, sp.data_ptr(), xi, k,
                               float(scale), y.data_ptr(), y.stride(0), torch.cuda.current_stream().cuda_stream)
    _lib.check(st, "sk_srtt_right")
    return y


def dct3_rows(x):
    """Orthonormal DCT-III along the last axis of a real device tensor (inverse of DCT-II ortho).

    Same transform as the reference's `_dct2_adjoint` = scipy.fft.dct(type=3, norm="ortho")
    (src/sketch/rtt.py:58-60), computed in O(d log d) on the GPU: with s_k the ortho weights,
    v = N * IFFT(s_k e^{i pi k / 2N} X_k) gives x_{2n} = Re v_n and x_{2n+1} = Re v_{N-1-n}.
    Complex64 for float32 input (~1e-7 relative), complex128 for float64 (~1e-16).
    """
    import math

    import torch

    n_ = x.shape[-1]
    ct = torch.complex64 if x.dtype == torch.float32 else torch.complex128
    key = (x.device, ct, n_)
    w = _DCT_TWIDDLE.get(key)
    if w is None:
        k = torch.arange(n_, dtype=torch.float64, device=x.device)
        s = torch.full((n_,), math.sqrt(2.0 / n_), dtype=torch.float64, device=x.device)
        s[0] = math.sqrt(1.0 / n_)
        w = _DCT_TWIDDLE[key] = torch.polar(s, math.pi * k / (2 * n_)).to(ct) * n_
    v = torch.fft.ifft(x.to(ct) * w, dim=-1)
    out = torch.empty_like(x)
    h = (n_ + 1) // 2
    out[..., 0::2] = v[..., :h].real
    out[..., 1::2] = v[..., h:].real.flip(-1)
    return out


_DCT_TWIDDLE: dict = {}
_DCT_CHUNK_ELEMS = 1 << 26  # rows per FFT batch bounded to ~64M elements (complex intermediates)


class SparseRttTM(TestMatrix):
    """Sparse randomized trigonometric transform Omega = D F S (reference rtt.py:75-186)."""

    def __init__(self, d: int, k: int, xi: int | None = None, transform: str | None = None, *,
                 diagonal: str | None = None, field: str = "real", seed: int = 0):
        super().__init__(d, k, field, seed)
        if xi is None:
            xi = int(np.ceil(1.5 * np.log(max(2, k))))
        if transform is None:
            transform = "dft" if field == "complex" else "dct"
        if transform not in TRANSFORMS:
            raise ValueError(f"unknown transform {transform!r}")
        if transform == "wht":
            _require_pow2(d)
        if transform == "dft" and field != "complex":
            raise ValueError("the DFT transform requires the complex field")
        if diagonal is None:
            diagonal = "real_rademacher"
        if diagonal not in ("real_rademacher", "uniform_symmetric", "steinhaus"):
            raise ValueError(f"unsupported diagonal distribution {diagonal!r}")
        if diagonal == "steinhaus" and field != "complex":
            raise ValueError("a Steinhaus diagonal requires the complex field")
        self.xi = int(xi)
        if not 1 <= self.xi <= d:
            raise ValueError(f"need 1 <= xi <= d, got xi={self.xi}")
        self.transform = transform
        self.diagonal = diagonal
        self._dvals = None
        self._sampler = None

    def _parts(self):
        """(D values, SparseColTM sampler) — reference rtt.py:114-121."""
        if self._dvals is None:
            self._dvals = entry_sample(self.diagonal, self._rng("diagonal"), self.d).astype(self.dtype)
            self._sampler = SparseColTM(self.d, self.k, self.xi, field=self.field, seed=self.seed)
        return self._dvals, self._sampler

    def materialize(self) -> np.ndarray:
        dvals, sampler = self._parts()
        fs = TRANSFORMS[self.transform][0](sampler.materialize(), axis=0)
        return (dvals[:, None] * fs).astype(self.dtype)

    def _dct_bt_device(self, device):
        """Omega^T = (D C^T S)^T for the real DCT, formed on the device (bf16 hi + lo, k x ldb) from the
        closed form of `materialize` (dct2_ortho of the sampler's columns, rtt.py:129-140):
        Omega[j, c] = d_j s_j sum_x v_{c,x} cos(pi j (2 r_{c,x} + 1) / 2N), s the ortho weights, with the
        angle reduced exactly in integers (j (2r + 1) mod 4N) before the float64 cosine."""
        import torch

        dvals, sampler = self._parts()
        coo = sampler.matrix.tocoo()
        n = self.d
        ldb = (n + 7) // 8 * 8
        omt = torch.zeros((self.k, ldb), dtype=torch.float64, device=device)
        j = torch.arange(n, dtype=torch.int64, device=device)
        rows = torch.as_tensor(coo.row.astype(np.int64), device=device)
        cols = torch.as_tensor(coo.col.astype(np.int64), device=device)
        vals = torch.as_tensor(np.real(coo.data).astype(np.float64), device=device)
        step = max(1, (1 << 22) // max(n, 1))  # entries per chunk: <= 4M cosines at a time
        for e0 in range(0, rows.numel(), step):
            r, c, v = rows[e0:e0 + step], cols[e0:e0 + step], vals[e0:e0 + step]
            ang = (j[None, :] * (2 * r[:, None] + 1)) % (4 * n)
            omt[:, :n].index_add_(0, c, torch.cos(ang.to(torch.float64) * (math.pi / (2 * n))) * v[:, None])
        w = torch.full((n,), math.sqrt(2.0 / n), dtype=torch.float64, device=device)
        w[0] = math.sqrt(1.0 / n)
        omt[:, :n] *= (torch.as_tensor(np.asarray(dvals, dtype=np.float64), device=device) * w)[None, :]
        hi = omt.to(torch.bfloat16)
        lo = (omt - hi.to(torch.float64)).to(torch.bfloat16)
        return hi, lo

    def _native_ok(self, dtype) -> bool:
        import torch

        return self.field == "real" and self.transform == "wht" and dtype in (torch.float32, torch.float64)

    def _dct_ok(self, dtype) -> bool:
        import torch

        return self.field == "real" and self.transform == "dct" and dtype in (torch.float32, torch.float64)

    def _dct_right(self, a):
        """Y = (A D) C^T S for the real DCT transform: DCT-III of every row through ONE real inverse
        FFT of half-spectrum length (Makhoul): with Z = A D / s (s the ortho weights),
        V_k = e^{i pi k / 2N} (Z_k - i Z_{N-k}) for k <= N/2 (Hermitian), v = irfft(V, N), and the
        transformed row is x_{2n} = v_n, x_{2n+1} = v_{N-1-n}; only the sampled x_j are gathered."""
        import math

        import torch

        if self.d % 2:
            return self._dct_right_complex(a)
        key = ("srtt_dct_r", a.device, a.dtype)
        n_, h = self.d, self.d // 2
        if key not in self._device_cache:
            dvals, sampler = self._parts()
            rows, neg, mag = sampler.column_draws()
            j = rows.reshape(-1).astype(np.int64)
            vidx = np.where(j % 2 == 0, j // 2, n_ - 1 - (j - 1) // 2)
            s = np.full(n_, math.sqrt(2.0 / n_))
            s[0] = math.sqrt(1.0 / n_)
            ct = torch.complex64 if a.dtype == torch.float32 else torch.complex128
            k = torch.arange(h + 1, dtype=torch.float64)
            tw = torch.polar(torch.ones(h + 1, dtype=torch.float64), math.pi * k / (2 * n_)).to(a.device, ct)
            self._device_cache[key] = (
                torch.from_numpy(np.ascontiguousarray(vidx)).to(a.device),
                torch.from_numpy(np.where(neg, -mag, mag).reshape(self.k, self.xi)).to(a.device, a.dtype),
                torch.from_numpy(np.ascontiguousarray(dvals / s)).to(device=a.device, dtype=a.dtype),
                tw)
        vidx, sgn, w, tw = self._device_cache[key]
        n = a.shape[0]
        y = torch.empty((n, self.k), dtype=a.dtype, device=a.device)
        step = max(1, _DCT_CHUNK_ELEMS // max(1, self.d))
        code = _lib.SK_F32 if a.dtype == torch.float32 else _lib.SK_F64
        twr = torch.view_as_real(tw).contiguous()
        ct = tw.dtype
        spec = torch.empty((min(n, step), h + 1), dtype=ct, device=a.device)
        lib = _lib.load()
        for r0 in range(0, n, step):
            blk = a[r0:r0 + step]
            m = blk.shape[0]
            with torch.cuda.device(a.device):
                st = lib.sk_dct3_prep(code, blk.data_ptr(), m, n_, blk.stride(0), w.data_ptr(), twr.data_ptr(),
                                      spec.data_ptr(), 2 * spec.stride(0), torch.cuda.current_stream().cuda_stream)
            _lib.check(st, "sk_dct3_prep")
            v = torch.fft.irfft(spec[:m], n=n_, dim=1)
            y[r0:r0 + step] = (v[:, vidx].view(-1, self.k, self.xi) * sgn).sum(-1)
        return y

    def _dct_right_complex(self, a):
        """Odd d: the complex-FFT DCT-III (dct3_rows) and the sampled gather."""
        import torch

        key = ("srtt_dct", a.device, a.dtype)
        if key not in self._device_cache:
            dvals, sampler = self._parts()
            rows, neg, mag = sampler.column_draws()
            idx = torch.from_numpy(np.ascontiguousarray(rows.reshape(-1))).to(a.device)
            sgn = torch.from_numpy(np.where(neg, -mag, mag).reshape(self.k, self.xi)).to(a.device, a.dtype)
            dv = torch.from_numpy(np.ascontiguousarray(dvals)).to(device=a.device, dtype=a.dtype)
            self._device_cache[key] = (idx, sgn, dv)
        idx, sgn, dv = self._device_cache[key]
        n = a.shape[0]
        y = torch.empty((n, self.k), dtype=a.dtype, device=a.device)
        step = max(1, _DCT_CHUNK_ELEMS // max(1, self.d))
        for r0 in range(0, n, step):
            z = dct3_rows(a[r0:r0 + step] * dv)
            y[r0:r0 + step] = (z[:, idx].view(-1, self.k, self.xi) * sgn).sum(-1)
        return y

    def _adjoint_device(self, b):
        """Omega^T B with B read in place (reference rtt.py:142-154): float32 on the tcgen05 TN engine
        (B^T Omega with Omega = D F S materialised once as exact-or-split bf16, X = its transpose),
        float64 on the library's CUDA-core contraction kernel (base class)."""
        import torch

        if self.field == "real" and b.dtype == torch.float32 and b.dim() == 2:
            key = ("srtt_adj_tn", b.device)
            if key not in self._device_cache:
                om = self.materialize()
                mag = float(np.abs(om).max()) or 1.0
                self._device_cache[key] = (split_wt(om / mag, b.device), mag)
            wt, mag = self._device_cache[key]
            return dense_tn_tc(b, scale=mag, wt=wt).T.contiguous()
        return super()._adjoint_device(b)

    def _dct_fft_tables(self, device, dtype):
        """Host tables of the fused DCT-III row kernel (csrc/srtt_dct.cu), cached per device and dtype:
        w = D / s, the sampled output -> index-in-v map and the scale (sampler magnitude / N); the
        kernel forms its trig tables itself."""
        import torch

        key = ("srtt_dct_fft", device, dtype)
        if key not in self._device_cache:
            n_, m_ = self.d, self.d // 2
            dvals, sampler = self._parts()
            rows, neg, mag = sampler.column_draws()
            s = np.full(n_, np.sqrt(2.0 / n_))
            s[0] = np.sqrt(1.0 / n_)
            j = rows.reshape(-1).astype(np.int64)
            t = np.where(j % 2 == 0, j // 2, n_ - 1 - (j - 1) // 2)
            samp = (t | (neg.reshape(-1).astype(np.int64) << 31)).astype(np.uint32).view(np.int32)
            self._device_cache[key] = (torch.from_numpy(np.ascontiguousarray(dvals / s)).to(device, dtype),
                                       torch.from_numpy(np.ascontiguousarray(samp)).to(device), float(mag) / n_)
        return self._device_cache[key]

    def _dct_fft_right(self, a):
        """Y through the fused DCT-III row kernel (sk_srtt_dct_right): no intermediate in HBM."""
        import torch

        w, samp, scale = self._dct_fft_tables(a.device, a.dtype)
        if a.stride(1) != 1 or a.data_ptr() % 16 or (a.stride(0) * a.element_size()) % 16:
            a = a.contiguous()
        n = a.shape[0]
        y = torch.empty((n, self.k), dtype=a.dtype, device=a.device)
        if n == 0:
            return y
        lib = _lib.load()
        code = _lib.SK_F32 if a.dtype == torch.float32 else _lib.SK_F64
        with torch.cuda.device(a.device):
            st = lib.sk_srtt_dct_right(code, a.data_ptr(), n, self.d, a.stride(0), w.data_ptr(), samp.data_ptr(),
                                       self.xi, self.k, scale, y.data_ptr(), y.stride(0),
                                       torch.cuda.current_stream().cuda_stream)
        _lib.check(st, "sk_srtt_dct_right")
        return y

    def dct_path(self, dtype) -> str:
        """'tc' (float32, k <= 1024: the materialised Omega = D C^T S on the tcgen05 GEMM), 'fft' (the fused
        DCT-III row kernel: float64 and large k, power-of-two d) or 'cufft' (other even d: prep kernel +
        cuFFT irfft); SKETCH_B200_DCT=tc|fft|cufft overrides."""
        import os

        import torch

        code = _lib.SK_F32 if dtype == torch.float32 else _lib.SK_F64
        fft_ok = _lib.load().sk_srtt_dct_supported(code, self.d) == 1
        forced = os.environ.get("SKETCH_B200_DCT", "auto")
        if forced == "fft" and fft_ok:
            return "fft"
        if forced == "cufft":
            return "cufft"
        tc_ok = (dtype == torch.float32 and self.k <= 1024 and self.d % 4 == 0 and self.d * self.k <= (1 << 26)
                 and _lib.load().sk_dense_tc_supported(self.k) == 1)
        if tc_ok and forced in ("tc", "auto"):
            return "tc"  # float32, k <= 1024: config-2 shape 1.21 ms (fused FFT kernel 2.47, cuFFT 4.04)
        if fft_ok:
            return "fft"  # float64 (the reference's dtype): 2.31 ms vs 3.97 for cuFFT at 32768 x 8192
        return "cufft"

    def _right_device(self, a):
        if self._dct_ok(a.dtype):
            path = self.dct_path(a.dtype)
            if path == "fft":
                return self._dct_fft_right(a)
            if path == "tc":
                key = ("srtt_dct_tc", a.device)
                if key not in self._device_cache:
                    self._device_cache[key] = self._dct_bt_device(a.device)
                hi, lo = self._device_cache[key]
                return dense_right_tc(a, hi, lo, self.k, 1.0)
            return self._dct_right(a)
        if not self._native_ok(a.dtype):
            return super()._right_device(a)
        import torch

        key = ("srtt", a.device, a.dtype)
        if key not in self._device_cache:
            dvals, sampler = self._parts()
            rows, neg, mag = sampler.column_draws()
            samp = torch.from_numpy(srtt_sampler_encode(rows, neg)).to(a.device)
            dv = torch.from_numpy(np.ascontiguousarray(dvals)).to(device=a.device, dtype=a.dtype)
            pm1 = bool(np.all(np.abs(dvals) == 1.0))
            self._device_cache[key] = (dv, samp, (1.0 / np.sqrt(self.d)) * mag, pm1)
        dv, samp, scale, pm1 = self._device_cache[key]
        if _large_rows(self.d, a.dtype):
            import torch

            if (a.dtype == torch.float32 and pm1 and self.d % 8192 == 0 and a.data_ptr() % 16 == 0
                    and a.stride(0) % 4 == 0 and a.stride(1) == 1):
                return self._large_right_tc(a, dv, samp, scale)
            return self._large_right(a, dv, scale)
        return _srtt_native(a, dv, samp, self.xi, self.k, scale, pm1)

    def _large_right_tc(self, a, dv, samp, scale):
        """float32, +-1 D, d a multiple of 8192: segment transforms on the tcgen05 kernel
        (sk_wht_segments_f32), then the sampled outputs of the outer H_{d/8192} (sk_srtt_outer_f32)."""
        import torch

        n = a.shape[0]
        y = torch.empty((n, self.k), dtype=a.dtype, device=a.device)
        step = max(1, (512 << 20) // (self.d * 4))  # scratch of at most 512 MB per batch
        z = torch.empty((min(n, step), self.d), dtype=torch.float32, device=a.device)
        lib = _lib.load()
        stream = torch.cuda.current_stream(a.device).cuda_stream
        for r0 in range(0, n, step):
            blk = a[r0:r0 + step]
            m = blk.shape[0]
            with torch.cuda.device(a.device):
                st = lib.sk_wht_segments_f32(blk.data_ptr(), m, self.d, blk.stride(0), dv.data_ptr(), z.data_ptr(),
                                             z.stride(0), stream)
                _lib.check(st, "sk_wht_segments_f32")
                st = lib.sk_srtt_outer_f32(z.data_ptr(), m, self.d, z.stride(0), samp.data_ptr(), self.xi, self.k,
                                           scale, y[r0:r0 + m].data_ptr(), y.stride(0), stream)
                _lib.check(st, "sk_srtt_outer_f32")
        return y

    def _large_right(self, a, dv, scale):
        """Long rows: D, segment WHTs (K3), then only the sampled outputs of the outer transform:
        Y[:, j] = sum_a H_{d1}[j >> 12, a] Z[:, a, j & 4095] for the k*xi sampled j."""
        import torch

        key = ("srtt_large", a.device, a.dtype)
        if key not in self._device_cache:
            _, sampler = self._parts()
            rows, neg, mag = sampler.column_draws()
            j = torch.from_numpy(np.ascontiguousarray(rows.reshape(-1))).to(a.device)
            d1 = self.d >> _SEG_L
            hs = _hadamard_signs(j >> _SEG_L, d1, a.device, a.dtype)  # (k xi) x d1
            sgn = torch.from_numpy(np.where(neg, -1.0, 1.0).reshape(self.k, self.xi)).to(a.device, a.dtype)
            self._device_cache[key] = (j & ((1 << _SEG_L) - 1), hs, sgn)
        jlo, hs, sgn = self._device_cache[key]
        n = a.shape[0]
        y = torch.empty((n, self.k), dtype=a.dtype, device=a.device)
        step = max(1, (256 << 20) // (self.d * a.element_size()))
        for r0 in range(0, n, step):
            z = _wht_segments((a[r0:r0 + step] * dv).contiguous())  # m x d1 x 4096
            zs = z[:, :, jlo]                                      # m x d1 x (k xi)
            yj = torch.einsum("mak,ka->mk", zs, hs)
            y[r0:r0 + step] = (yj.view(-1, self.k, self.xi) * sgn).sum(-1) * scale
        return y

    def redraw(self, seed: int) -> "SparseRttTM":
        return SparseRttTM(self.d, self.k, self.xi, self.transform, diagonal=self.diagonal, field=self.field,
                           seed=seed)
