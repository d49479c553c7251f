"""ctypes binding of libsketch_b200.so (the C ABI declared in include/sketch_b200.h).

There is no fallback: if the library cannot be loaded, or no CUDA device is visible, every
apply raises.  The binding passes raw device pointers, sizes and the current torch CUDA stream.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import _build

SK_OK = 0
SK_EINVAL = -1
SK_EUNSUPPORTED = -2
SK_ECUDA = -3
SK_F32 = 0
SK_F64 = 1
SK_WHT = 0
SK_DCT3 = 1
SK_DIAG_PM1 = 0x100
ABI_VERSION = 2  # include/sketch_b200.h SK_ABI_VERSION

_c_i64 = ctypes.c_int64
_c_int = ctypes.c_int
_c_p = ctypes.c_void_p
_c_dbl = ctypes.c_double
_c_size = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/sketch_b200.h
SIGNATURES = {
    "sk_abi_version": (_c_int, []),
    "sk_last_error": (ctypes.c_char_p, []),
    "sk_device_sm_count": (_c_int, [_c_int]),
    "sk_sparse_right_chunk_rows": (_c_int, [_c_int, _c_i64, _c_i64]),
    "sk_sparse_right": (_c_int, [_c_int, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, ctypes.c_int32, _c_i64,
                                 _c_i64, _c_dbl, _c_p, _c_i64, _c_p]),
    "sk_sparse_right_csr": (_c_int, [_c_int, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_dbl, _c_p, _c_i64,
                                     _c_p]),
    "sk_philox_u32": (_c_int, [_c_p, _c_p, ctypes.c_uint64, _c_i64, _c_p, _c_p]),
    "sk_sparse_adjoint_chunk_rows": (_c_int, [_c_int, _c_i64, _c_i64]),
    "sk_sparse_adjoint_workspace_bytes": (_c_size, [_c_int, _c_i64, _c_i64, _c_i64]),
    "sk_sparse_adjoint": (_c_int, [_c_int, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, ctypes.c_int32, _c_p,
                                   ctypes.c_int32, _c_i64, _c_dbl, _c_p, _c_i64, _c_int, _c_p, _c_size, _c_p]),
    "sk_sparse_adjoint_wide_encode": (_c_i64, [_c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_p, _c_p]),
    "sk_sparse_adjoint_wide_segments": (_c_i64, [_c_i64, _c_i64]),
    "sk_sparse_adjoint_wide_workspace_bytes": (_c_size, [_c_i64, _c_i64, _c_i64]),
    "sk_sparse_adjoint_wide": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, ctypes.c_int32, _c_i64, _c_dbl, _c_p,
                                        _c_i64, _c_int, _c_p, _c_size, _c_p]),
    "sk_sparse_adjoint_wide_rows": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_p, ctypes.c_int32,
                                             _c_i64, _c_dbl, _c_p, _c_i64, _c_int, _c_p, _c_size, _c_p]),
    "sk_sparse_adjoint_narrow": (_c_int, [_c_int, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_int, _c_i64, _c_dbl,
                                          _c_p, _c_i64, _c_p]),
    "sk_sparse_adjoint_gather_pieces": (_c_i64, [_c_int, _c_i64, _c_i64, _c_i64, _c_p]),
    "sk_sparse_adjoint_gather_workspace_bytes": (_c_size, [_c_int, _c_i64, _c_i64, _c_i64]),
    "sk_sparse_adjoint_gather": (_c_int, [_c_int, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_i64, _c_dbl, _c_p,
                                          _c_i64, _c_int, _c_p, _c_size, _c_p]),
    "sk_sparse_adjoint_wide_workspace_bytes_f64": (_c_size, [_c_i64, _c_i64, _c_i64]),
    "sk_sparse_adjoint_wide_f64": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, ctypes.c_int32, _c_i64, _c_dbl,
                                            _c_p, _c_i64, _c_int, _c_p, _c_size, _c_p]),
    "sk_sparse_adjoint_wide_rows_f64": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_p,
                                                 ctypes.c_int32, _c_i64, _c_dbl, _c_p, _c_i64, _c_int, _c_p, _c_size,
                                                 _c_p]),
    "sk_srtt_right": (_c_int, [_c_int, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_int, _c_p, ctypes.c_int32, _c_i64,
                               _c_dbl, _c_p, _c_i64, _c_p]),
    "sk_wht_segments_f32": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_i64, _c_p]),
    "sk_srtt_outer_f32": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, ctypes.c_int32, _c_i64, _c_dbl, _c_p, _c_i64,
                                   _c_p]),
    "sk_dct3_prep": (_c_int, [_c_int, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_i64, _c_p]),
    "sk_gemv_f32_f64": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p]),
    "sk_gemv_t_f32_f64_workspace_bytes": (_c_size, [_c_i64, _c_i64]),
    "sk_gemv_t_f32_f64": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_size, _c_p]),
    "sk_lsqr_step_f32_f64_workspace_bytes": (_c_size, [_c_i64, _c_i64]),
    "sk_lsqr_step_f32_f64": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_dbl, _c_p, _c_p, _c_p, _c_size, _c_p]),
    "sk_dense_tc_supported": (_c_int, [_c_i64]),
    "sk_dense_tc_workspace_bytes": (_c_size, [_c_i64, _c_i64, _c_i64, _c_int]),
    "sk_dense_right_tc": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_i64, _c_i64, _c_dbl, _c_p, _c_i64,
                                   _c_p, _c_size, _c_p]),
    "sk_dense_tn_tc_workspace_bytes": (_c_size, [_c_i64, _c_i64, _c_i64]),
    "sk_dense_tn_tc": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_i64, _c_i64, _c_dbl, _c_p, _c_i64,
                                _c_p, _c_size, _c_p]),
    "sk_kr_workspace_bytes": (_c_size, [_c_i64, _c_i64, _c_i64, _c_i64, _c_int, _c_int]),
    "sk_kr_right": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_i64, _c_p, _c_i64, _c_i64, _c_dbl,
                             _c_p, _c_i64, _c_p, _c_size, _c_p]),
    "sk_kr_adjoint": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_i64, _c_p, _c_i64, _c_i64, _c_dbl,
                               _c_p, _c_i64, _c_p, _c_size, _c_p]),
    "sk_sparse_right_ring_supported": (_c_int, [_c_int, _c_i64, _c_i64, _c_i64]),
    "sk_sparse_right_ring_workspace_bytes": (_c_size, [_c_i64, _c_i64]),
    "sk_sparse_right_ring": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_i64, _c_i64, _c_dbl, _c_p, _c_i64,
                                      _c_p, _c_size, _c_p]),
    "sk_sparse_right_ring_slab": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_i64, _c_i64, _c_dbl, _c_p,
                                           _c_i64, _c_int, _c_p, _c_size, _c_p]),
    "sk_kr_right_signs": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_i64, _c_p, _c_i64, _c_p, _c_i64,
                                   _c_dbl, _c_i64, _c_dbl, _c_p, _c_i64, _c_p, _c_size, _c_p]),
    "sk_lsqr_recur_f64": (_c_int, [_c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p]),
    "sk_sparse_right_cols_groups": (_c_int, [_c_i64]),
    "sk_sparse_right_cols_supported": (_c_int, [_c_int, _c_i64, _c_i64, ctypes.c_int32]),
    "sk_sparse_right_cols_encode": (_c_int, [_c_int, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, ctypes.c_int32, _c_p,
                                             _c_p, _c_p, _c_p]),
    "sk_sparse_right_cols": (_c_int, [_c_int, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_i64, ctypes.c_int32,
                                      _c_dbl, _c_p, _c_i64, _c_int, _c_p]),
    "sk_two_sided_workspace_bytes": (_c_size, [_c_i64, _c_i64, _c_i64, _c_int]),
    "sk_two_sided_sketch": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_i64, _c_i64, _c_dbl, _c_p,
                                     ctypes.c_int32, _c_i64, _c_dbl, _c_p, _c_i64, _c_p, _c_i64, _c_p, _c_size,
                                     _c_p]),
    "sk_srtt_dct_supported": (_c_int, [_c_int, _c_i64]),
    "sk_srtt_dct_right": (_c_int, [_c_int, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, ctypes.c_int32, _c_i64, _c_dbl,
                                   _c_p, _c_i64, _c_p]),
    "sk_kr_right_z": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_i64, _c_p, _c_p, _c_i64, _c_i64,
                               _c_int, _c_dbl, _c_int, _c_p, _c_i64, _c_p]),
    "sk_kr_adjoint_z": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_i64, _c_p, _c_p, _c_i64, _c_i64,
                                 _c_int, _c_dbl, _c_int, _c_p, _c_i64, _c_p]),
    "sk_kr_right_cc": (_c_int, [_c_int, _c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i64, _c_i64,
                                _c_dbl, _c_p, _c_i64, _c_p]),
    "sk_kr_adjoint_cc": (_c_int, [_c_int, _c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i64, _c_i64,
                                  _c_dbl, _c_p, _c_i64, _c_p]),
}

_lock = threading.Lock()
_lib = None


class SketchLibraryError(RuntimeError):
    """libsketch_b200.so is missing, failed to load, or returned an error status."""


def library_path() -> str:
    return os.environ.get("SKETCH_B200_LIB", _build.lib_path())


def load(build_if_missing: bool = True):
    """Load (building first if needed and nvcc exists) and bind every declared symbol."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = library_path()
        if build_if_missing and "SKETCH_B200_LIB" not in os.environ:
            try:
                if _build.needs_build():
                    _build.build()
            except RuntimeError as exc:
                if not os.path.exists(path):
                    raise SketchLibraryError(f"cannot build {path}: {exc}") from exc
        if not os.path.exists(path):
            raise SketchLibraryError(f"{path} not found; run __graft_entry__.build()")
        try:
            lib = ctypes.CDLL(path)
        except OSError as exc:
            raise SketchLibraryError(f"cannot load {path}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.sk_abi_version() != ABI_VERSION:
            raise SketchLibraryError("libsketch_b200.so ABI version mismatch")
        _lib = lib
        return lib


def check(status: int, what: str) -> None:
    if status != SK_OK:
        msg = load().sk_last_error().decode(errors="replace")
        kind = {SK_EINVAL: ValueError, SK_EUNSUPPORTED: NotImplementedError}.get(status, SketchLibraryError)
        raise kind(f"{what}: status {status}: {msg}")
