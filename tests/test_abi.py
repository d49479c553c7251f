"""The C-ABI library builds, loads without a GPU, and exports every symbol include/*.h declares."""

import ctypes
import glob
import os
import re

from conftest import ROOT


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        names |= set(re.findall(r"SK_API\s+[\w\s\*]+?\b(sk_\w+)\s*\(", text))
    return names


def test_header_declares_entry_points():
    names = declared_symbols()
    assert {"sk_sparse_right", "sk_sparse_adjoint", "sk_srtt_right", "sk_last_error"} <= names


def test_library_exports_every_declared_symbol():
    from paper_2508_21189_b200 import _lib

    lib = _lib.load()
    raw = ctypes.CDLL(_lib.library_path())
    for name in declared_symbols():
        assert hasattr(raw, name), name
    assert set(_lib.SIGNATURES) >= declared_symbols()
    assert lib.sk_abi_version() == 2


def test_error_path_without_device():
    from paper_2508_21189_b200 import _lib

    lib = _lib.load()
    # invalid shape is rejected before any CUDA call
    st = lib.sk_sparse_right(0, None, 4, 0, 0, None, None, 512, 0, 4, 1.0, None, 4, None)
    assert st == _lib.SK_EINVAL
    assert b"sk_sparse_right" in lib.sk_last_error()
    assert lib.sk_sparse_right_chunk_rows(0, 100, 10) == 512
    assert lib.sk_sparse_right_chunk_rows(7, 100, 10) == _lib.SK_EINVAL


def test_argument_checks_without_device():
    """Every new entry point rejects bad shapes / dtypes / pointers before touching the device."""
    from paper_2508_21189_b200 import _lib

    lib = _lib.load()
    E = _lib.SK_EINVAL
    # K2g: bad dtype, bad leading dimension, null pointers
    assert lib.sk_sparse_adjoint_gather(7, None, 10, 4, 4, None, None, 3, 1.0, None, 4, 0, None, 0, None) == E
    assert lib.sk_sparse_adjoint_gather(0, None, 10, 4, 2, None, None, 3, 1.0, None, 4, 0, None, 0, None) == E
    assert lib.sk_sparse_adjoint_gather(0, None, 10, 4, 4, None, None, 3, 1.0, None, 4, 0, None, 0, None) == E
    assert b"sk_sparse_adjoint_gather" in lib.sk_last_error()
    assert lib.sk_sparse_adjoint_gather_pieces(0, 0, 4, 3, None) == E
    assert lib.sk_sparse_adjoint_gather_workspace_bytes(0, 0, 4, 3) == 0
    # K2w float64, TN product, mixed-precision GEMV
    assert lib.sk_sparse_adjoint_wide_f64(None, 0, 4, 4, None, None, 24, 3, 1.0, None, 4, 0, None, 0, None) == E
    assert lib.sk_dense_tn_tc(None, 0, 4, 4, None, None, 8, 3, 1.0, None, 3, None, 0, None) == E
    assert lib.sk_dense_tn_tc(None, 8, 4, 4, None, None, 8, 3, 1.0, None, 3, None, 0, None) == E
    assert lib.sk_gemv_f32_f64(None, 4, 0, 0, None, None, None) == E
    assert lib.sk_gemv_t_f32_f64(None, 4, 4, 2, None, None, None, 0, None) == E
    assert lib.sk_lsqr_step_f32_f64(None, 4, 128, 128, None, 0.0, None, None, None, 0, None) == E
    assert lib.sk_lsqr_step_f32_f64_workspace_bytes(0, 128) == 0
    assert lib.sk_philox_u32(None, None, 0, 8, None, None) == E
