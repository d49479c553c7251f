"""The sketching-operator interface (drop-in for sketchkit's TestMatrix), applied on a B200.

Mirrors the reference API of src/sketch/base.py:48-130: a TestMatrix is a d-by-k random map
with a field, a dtype (float64 / complex128, as the reference), a seed, host-side `materialize`
and `redraw`, and the two apply paths

    apply_right(A)    -> A Omega      (A: n x d)        reference sketch/base.py:75-79
    apply_adjoint(B)  -> Omega^* B    (B: d x m or (d,)) reference sketch/base.py:81-91

with the same ValueError texts on a shape mismatch (base.py:63-69).  Unlike the reference, the
apply paths run on the current CUDA device: host operands are uploaded, the family's CUDA
kernel (libsketch_b200.so) runs, and the result is returned in the caller's container (NumPy
float64 for NumPy input, a torch tensor for torch input).  Families or fields without a
dedicated kernel use a dense device GEMM of the materialized Omega (cuBLAS through torch);
nothing ever computes on the CPU.
"""

from __future__ import annotations

from abc import ABC, abstractmethod

import numpy as np

from .. import _device
from .._device import from_result, to_operand
from ..rng import RngStream

__all__ = ["TestMatrix", "ExplicitTM", "entry_sample", "dtype_of"]

_DTYPES = {"real": np.dtype(np.float64), "complex": np.dtype(np.complex128)}


def dtype_of(field: str) -> np.dtype:
    """Double-precision dtype of a field tag (reference core/containers.py:41-46)."""
    try:
        return _DTYPES[field]
    except KeyError:
        raise ValueError(f"unknown field {field!r}; expected 'real' or 'complex'") from None


def entry_sample(distribution: str, rng: np.random.Generator, size) -> np.ndarray:
    """iid unit-variance entries by name — same draws as reference sketch/base.py:23-45."""
    if distribution == "real_rademacher":
        return rng.integers(0, 2, size=size).astype(np.float64) * 2.0 - 1.0
    if distribution == "complex_rademacher":
        re = rng.integers(0, 2, size=size) * 2.0 - 1.0
        im = rng.integers(0, 2, size=size) * 2.0 - 1.0
        return (re + 1j * im) / np.sqrt(2.0)
    if distribution == "steinhaus":
        return np.exp(1j * rng.uniform(0.0, 2.0 * np.pi, size=size))
    if distribution == "real_gaussian":
        return rng.standard_normal(size)
    if distribution == "complex_gaussian":
        return (rng.standard_normal(size) + 1j * rng.standard_normal(size)) / np.sqrt(2.0)
    if distribution == "uniform_symmetric":
        return rng.uniform(-np.sqrt(3.0), np.sqrt(3.0), size=size)
    raise ValueError(f"unknown entry distribution {distribution!r}")


def _shape_of(x) -> tuple:
    shape = getattr(x, "shape", None)
    return tuple(int(v) for v in (shape if shape is not None else np.shape(x)))


class _Shaped:
    __slots__ = ("shape",)

    def __init__(self, shape):
        self.shape = shape


def _is_scipy_sparse(x) -> bool:
    try:
        import scipy.sparse as sp
    except ImportError:  # pragma: no cover
        return False
    return sp.issparse(x)


class TestMatrix(ABC):
    """Abstract random sketching operator Omega in F^{d x k}, applied on the GPU."""

    __test__ = False  # not a pytest class

    def __init__(self, d: int, k: int, field: str, seed: int):
        if d < 1 or k < 1:
            raise ValueError(f"dimensions must be positive, got d={d}, k={k}")
        self.d = int(d)
        self.k = int(k)
        self.field = field
        self.dtype = dtype_of(field)
        self.seed = int(seed)
        self._device_cache: dict = {}

    # -- streams and checks (reference base.py:60-69) ---------------------------------------
    def _rng(self, *labels) -> np.random.Generator:
        return RngStream(self.seed, (type(self).__name__,) + labels).generator()

    def _check_right(self, a) -> None:
        if a.shape[1] != self.d:
            raise ValueError(f"apply_right needs A with {self.d} columns, got {tuple(a.shape)}")

    def _check_adjoint(self, b) -> None:
        if b.shape[0] != self.d:
            raise ValueError(f"apply_adjoint needs B with {self.d} rows, got {tuple(b.shape)}")

    # -- host-side description ----------------------------------------------------------------
    @abstractmethod
    def materialize(self) -> np.ndarray:
        """Explicit dense d-by-k matrix (host, float64/complex128) for diagnostics and oracles."""

    @abstractmethod
    def redraw(self, seed: int) -> "TestMatrix":
        """A fresh operator with the same parameters and a new seed."""

    # -- device applies -----------------------------------------------------------------------
    def apply_right(self, a):
        """A Omega for A with d columns (NumPy / SciPy sparse / torch; computed on the GPU)."""
        shape = _shape_of(a)
        if len(shape) != 2:
            raise ValueError(f"apply_right needs a 2-d A, got shape {shape}")
        self._check_right(_Shaped(shape))
        if _is_scipy_sparse(a) and self._sparse_input_ok():
            return self._right_sparse_input(a)
        host, kind = _device.host_tensor_of(a) if not hasattr(a, "toarray") else (None, None)
        if host is not None and not host.is_complex() and \
                host.numel() * host.element_size() >= _device.PIPELINE_MIN_BYTES:
            y = _device.pipelined_right(self._right_device, host, self.k)
            if kind == "numpy":
                # widened by torch's multi-threaded CPU copy (NumPy's astype is single-threaded: ~47 ms for
                # a config-2 result)
                import torch

                return y.to(torch.complex128 if y.is_complex() else torch.float64).numpy()
            return y
        op = to_operand(a, allow_vector=False)
        return from_result(self._right_device(op.tensor), op)

    def apply_adjoint(self, b):
        """Omega^* B for B with d rows; a 1-D B is treated as a column and squeezed back."""
        shape = _shape_of(b)
        if len(shape) not in (1, 2):
            raise ValueError(f"apply_adjoint needs a 1-d or 2-d B, got shape {shape}")
        self._check_adjoint(_Shaped(shape if len(shape) == 2 else (shape[0], 1)))
        if _is_scipy_sparse(b) and len(shape) == 2 and self._sparse_input_ok():
            # Omega^T B = (B^T Omega)^T with B^T in CSR: the sparse-input row kernel
            return np.ascontiguousarray(self._right_sparse_input(b.T.tocsr()).T)
        op = to_operand(b, allow_vector=True)
        return from_result(self._adjoint_device(op.tensor), op)

    def _sparse_input_ok(self) -> bool:
        """Families that apply SciPy-sparse input without densifying it (sparse sign: K1s)."""
        return False

    def _right_sparse_input(self, a):
        raise NotImplementedError

    # dense complex families (Gaussian, explicit) whose complex128 applies run on the FP64 DMMA engine
    # over the planes of the materialised Omega; the sparse families keep their own paths
    _planar_complex = False

    def _dense_z(self, x, adjoint: bool):
        """Complex-field A Omega / Omega^H B (float64 or complex128 operand) on the FP64 DMMA engine over
        the real and imaginary planes of the materialised Omega (sk_kr_right_z / sk_kr_adjoint_z)."""
        from .zplanes import z_apply, z_operands

        key = ("dense_z", x.device)
        if key not in self._device_cache:
            self._device_cache[key] = z_operands(None, np.asarray(self.materialize()), x.device)
        return z_apply(self._device_cache[key], x, adjoint, 1.0)

    def _dense_cc(self, x, adjoint: bool):
        """A Omega (or Omega^T B) with the materialized real Omega on the library's contraction kernels
        (sk_kr_right_cc / sk_kr_adjoint_cc with one block: W = NULL, F = Omega): float64 on the FP64
        tensor cores (K5d), float32 on the CUDA cores with float64 accumulation."""
        import torch

        from .. import _lib

        key = ("dense_cc", x.device, x.dtype)
        if key not in self._device_cache:
            f = torch.as_tensor(np.ascontiguousarray(self.materialize()), device=x.device).to(x.dtype)
            self._device_cache[key] = f
        f = self._device_cache[key]
        if x.stride(1) != 1 or x.stride(0) < x.shape[1]:
            x = x.contiguous()
        rows = x.shape[1] if adjoint else x.shape[0]
        out = torch.empty((self.k, rows) if adjoint else (rows, self.k), dtype=x.dtype, device=x.device)
        if rows == 0:
            return out
        lib = _lib.load()
        code = _lib.SK_F64 if x.dtype == torch.float64 else _lib.SK_F32
        fn = lib.sk_kr_adjoint_cc if adjoint else lib.sk_kr_right_cc
        with torch.cuda.device(x.device):
            st = fn(code, x.data_ptr(), rows, 1, self.d, x.stride(0), f.data_ptr(), f.stride(0), None, 0, self.k, 1.0,
                    out.data_ptr(), out.stride(0), torch.cuda.current_stream().cuda_stream)
        _lib.check(st, "sk_kr_adjoint_cc" if adjoint else "sk_kr_right_cc")
        return out

    def _right_device(self, a):
        """Dense apply of the materialized Omega: real fields on the library's CUDA-core kernel (K4c
        with one block), complex fields as a device GEMM through torch; families override with kernels."""
        import torch

        if self.field == "real" and a.dtype in (torch.float32, torch.float64):
            return self._dense_cc(a, adjoint=False)
        if self._planar_complex and a.dtype in (torch.float64, torch.complex128):
            return self._dense_z(a, adjoint=False)
        om = self._dense_on(a.device, a.dtype)
        dt = torch.promote_types(a.dtype, om.dtype)
        return a.to(dt) @ om.to(dt)

    def _adjoint_device(self, b):
        import torch

        if self.field == "real" and b.dtype in (torch.float32, torch.float64):
            return self._dense_cc(b, adjoint=True)
        if self._planar_complex and b.dtype in (torch.float64, torch.complex128):
            return self._dense_z(b, adjoint=True)
        om = self._dense_on(b.device, b.dtype)
        dt = torch.promote_types(b.dtype, om.dtype)
        return om.to(dt).conj().T @ b.to(dt)

    def _dense_on(self, device, dtype):
        import torch

        real = not np.iscomplexobj(np.empty(0, self.dtype))
        want = dtype if real else (torch.complex64 if dtype == torch.float32 else torch.complex128)
        if not real and dtype in (torch.complex64, torch.complex128):
            want = dtype
        key = ("dense", device, want)
        if key not in self._device_cache:
            self._device_cache[key] = torch.as_tensor(np.ascontiguousarray(self.materialize())).to(device=device,
                                                                                                   dtype=want)
        return self._device_cache[key]

    def release_device(self) -> None:
        """Drop cached device copies of Omega."""
        self._device_cache.clear()

    def sample_adjoint_sqnorms(self, x, trials: int, seed: int) -> np.ndarray:
        """Monte Carlo samples of ||Omega^* x||^2 over fresh draws (reference base.py:93-106)."""
        x = np.asarray(x)
        out = np.empty(trials)
        for t in range(trials):
            y = np.asarray(self.redraw(seed=seed + t).apply_adjoint(x))
            out[t] = float(np.real(np.vdot(y, y)))
        return out

    def __repr__(self):
        return f"{type(self).__name__}(d={self.d}, k={self.k}, field={self.field!r}, seed={self.seed})"


class ExplicitTM(TestMatrix):
    """A user-supplied explicit matrix wrapped as a sketching operator (reference base.py:116-130)."""

    _planar_complex = True

    def __init__(self, matrix, field: str | None = None):
        matrix = np.asarray(matrix)
        if field is None:
            field = "complex" if np.iscomplexobj(matrix) else "real"
        super().__init__(matrix.shape[0], matrix.shape[1], field, seed=0)
        self._matrix = matrix.astype(self.dtype, copy=False)

    def materialize(self) -> np.ndarray:
        return self._matrix

    def redraw(self, seed: int) -> "ExplicitTM":
        return self
