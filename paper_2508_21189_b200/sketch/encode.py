"""Compact device encodings of test matrices (built once per operator, cached per device).

bcsc — "blocked column lists" for sparse Omega whose nonzeros share one magnitude (every real
SparseStack / SparseUniform / SparseIID / SparseCol matrix): rows of Omega are cut into chunks
of R rows; for chunk h and column c the entries ent[ptr[h*k + c] : ptr[h*k + c + 1]] are uint16
(local_row << 1) | negative, ascending in row.  The common magnitude travels as the kernel's
`scale`.  This is the layout both the right-apply gather (K1) and the adjoint gather (K2) read.
"""

from __future__ import annotations

import numpy as np

__all__ = ["bcsc_encode", "bcsc_decode", "bcsc_segments", "srtt_sampler_encode", "sign_bits"]

ADJ_GROUP = 1024  # output rows per CTA group of the adjoint fast path (sparse_adjoint.cu V2_CG)
PTR_PAD = 1028    # ints the fast path may read past the pointer array
ENT_PAD = 8       # entries the fast path may read past the entry array


def bcsc_encode(rows, cols, neg, d: int, k: int, chunk_rows: int):
    """(rows, cols, neg) triplets -> (ptr int32[nchunks*k + 1], ent uint16[nnz])."""
    if chunk_rows < 1 or chunk_rows > 32768 or chunk_rows & (chunk_rows - 1):
        raise ValueError("chunk_rows must be a power of two <= 32768")
    rows = np.asarray(rows, dtype=np.int64).ravel()
    cols = np.asarray(cols, dtype=np.int64).ravel()
    neg = np.asarray(neg, dtype=bool).ravel()
    nnz = rows.size
    if nnz >= 2**31:
        raise ValueError("too many nonzeros for int32 offsets")
    nchunks = (d + chunk_rows - 1) // chunk_rows
    key = (rows // chunk_rows) * k + cols
    # stable: entries with equal (chunk, column) keep ascending row order when rows are sorted
    order = np.argsort(key, kind="stable") if nnz else np.zeros(0, np.int64)
    if nnz and np.any(np.diff(rows) < 0):
        order = np.lexsort((rows, key))
    local = (rows[order] % chunk_rows).astype(np.uint32)
    ent = ((local << 1) | neg[order].astype(np.uint32)).astype(np.uint16)
    counts = np.bincount(key, minlength=nchunks * k) if nnz else np.zeros(nchunks * k, np.int64)
    ptr = np.zeros(nchunks * k + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    return ptr.astype(np.int32), ent


def bcsc_segments(ptr, d: int, k: int, chunk_rows: int, group: int = ADJ_GROUP):
    """Per (chunk, group of `group` columns): [first entry rounded down to 8, count rounded up to 8].

    Returns (seg int32[nchunks * ngroups * 2], ent_cap) for sk_sparse_adjoint's fast path.
    """
    ptr = np.asarray(ptr, dtype=np.int64)
    nchunks = (d + chunk_rows - 1) // chunk_rows
    ngroups = (k + group - 1) // group
    h = np.arange(nchunks)[:, None]
    g0 = np.arange(ngroups)[None, :] * group
    g1 = np.minimum(g0 + group, k)
    start = ptr[h * k + g0]
    end = ptr[h * k + g1]
    e0 = start // 8 * 8
    cnt = (end - e0 + 7) // 8 * 8
    seg = np.stack([e0, cnt], axis=-1).astype(np.int32).ravel()
    return seg, int(cnt.max()) if cnt.size else 0


def bcsc_decode(ptr, ent, d: int, k: int, chunk_rows: int):
    """Inverse of bcsc_encode (tests): returns (rows, cols, neg) sorted by (chunk, col, row)."""
    ptr = np.asarray(ptr, dtype=np.int64)
    ent = np.asarray(ent, dtype=np.uint32)
    nchunks = (d + chunk_rows - 1) // chunk_rows
    counts = np.diff(ptr)
    keys = np.repeat(np.arange(nchunks * k), counts)
    chunk, cols = keys // k, keys % k
    rows = chunk * chunk_rows + (ent >> 1)
    return rows, cols, (ent & 1).astype(bool)


def srtt_sampler_encode(rows_kx, neg_kx) -> np.ndarray:
    """SparseCol sampler (k, xi) rows + signs -> int32 entries row | neg << 31 (c-major)."""
    rows = np.asarray(rows_kx, dtype=np.int64).ravel()
    neg = np.asarray(neg_kx, dtype=bool).ravel()
    if rows.size and rows.max() >= 2**31:
        raise ValueError("row index too large")
    ent = rows.astype(np.uint32) | (neg.astype(np.uint32) << 31)
    return ent.view(np.int32)


def sign_bits(neg) -> np.ndarray:
    """Pack a boolean array (flattened, C order) into uint32 words, bit i of word i // 32."""
    neg = np.asarray(neg, dtype=bool).ravel()
    pad = (-neg.size) % 32
    if pad:
        neg = np.concatenate([neg, np.zeros(pad, bool)])
    return np.packbits(neg.reshape(-1, 32), axis=1, bitorder="little").view("<u4").astype(np.uint32).ravel()
