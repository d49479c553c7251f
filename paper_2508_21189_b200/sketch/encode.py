"""Compact device encodings of test matrices (built once per operator, cached per device).

bcsc — "blocked column lists" for sparse Omega whose nonzeros share one magnitude (every real
SparseStack / SparseUniform / SparseIID / SparseCol matrix): rows of Omega are cut into chunks
of R rows; for chunk h and column c the entries ent[ptr[h*k + c] : ptr[h*k + c + 1]] are uint16
(local_row << 1) | negative, ascending in row.  The common magnitude travels as the kernel's
`scale`.  This is the layout both the right-apply gather (K1) and the adjoint gather (K2) read.
"""

from __future__ import annotations

import numpy as np

__all__ = ["bcsc_encode", "bcsc_decode", "bcsc_segments", "srtt_sampler_encode", "sign_bits", "wide_encode_device",
           "gather_encode", "ring_encode", "ring_decode", "cols_encode", "COLS_MAXP"]

RING_RC = 64     # rows of Omega per stage of the K1r ring kernel (sparse_right_ring.cu RC)
RING_UC = 128    # rows of Omega per consumer unit (two stages, sparse_right_ring.cu UC)
RING_WARPS = 16  # consumer warps (NCONS), 16 output columns each (CPW)

COLS_MAXP = (32, 64, 96, 128)  # list positions per lane the K1c kernel is built for (sparse_right_cols.cu)

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


# K2w segment layout (adjoint_wide.cu): rows of Omega in chunks of 128, output columns in groups of
# 256 = 16 warps x 16; a segment = 24-uint16 header (17 warp offsets) + per-warp entry lists
# (row_in_chunk << 9) | (neg << 4) | (c mod 16), each padded to a multiple of 4 with no-op 32.
WIDE_R, WIDE_CG, WIDE_CPW, WIDE_WARPS, WIDE_HDR, WIDE_NOOP = 128, 256, 16, 16, 24, 32


def wide_encode_device(cols, neg, zeta: int, d: int, k: int):
    """K2w encoding built on the GPU from device draws (rows implicit: entry e is row e // zeta).

    Same bytes as the host encoder `sk_sparse_adjoint_wide_encode` fed the same entries in
    row-major order: a stable sort by (segment, warp) keeps each list in entry order.
    Returns (enc int16 device tensor, seg_off int64 device tensor, seg_cap).
    """
    import torch

    dev = cols.device
    c = cols.reshape(-1).to(torch.int64)
    g = neg.reshape(-1).to(torch.int64)
    nnz = c.numel()
    r = torch.arange(nnz, device=dev, dtype=torch.int64) // zeta
    nchunks, ngroups = -(-d // WIDE_R), -(-k // WIDE_CG)
    nseg = nchunks * ngroups
    if nnz and (int(c.min()) < 0 or int(c.max()) >= k):
        raise ValueError("column index out of range")
    key = ((r // WIDE_R) * ngroups + c // WIDE_CG) * WIDE_WARPS + (c % WIDE_CG) // WIDE_CPW
    cnt = torch.bincount(key, minlength=nseg * WIDE_WARPS)
    padded = ((cnt + 3) // 4 * 4).view(nseg, WIDE_WARPS)
    n_seg = padded.sum(1)
    if nseg and int(n_seg.max()) > 65535:
        raise ValueError("K2w segment over 65535 entries")
    seg_len = WIDE_HDR + (n_seg + 7) // 8 * 8
    seg_off = torch.zeros(nseg + 1, dtype=torch.int64, device=dev)
    torch.cumsum(seg_len, 0, out=seg_off[1:])
    total = int(seg_off[-1])
    warp_off = padded.cumsum(1) - padded  # exclusive, within the segment's entry area
    enc = torch.full((total,), WIDE_NOOP, dtype=torch.int32, device=dev)
    hdr = torch.zeros(nseg, WIDE_HDR, dtype=torch.int32, device=dev)
    hdr[:, :WIDE_WARPS] = warp_off.to(torch.int32)
    hdr[:, WIDE_WARPS] = n_seg.to(torch.int32)
    idx = seg_off[:-1, None] + torch.arange(WIDE_HDR, device=dev)[None, :]
    enc[idx.reshape(-1)] = hdr.reshape(-1)
    # rank of each entry inside its (segment, warp) list, in entry order
    order = torch.sort(key, stable=True).indices
    start = torch.cumsum(cnt, 0) - cnt
    rank = torch.empty_like(key)
    rank[order] = torch.arange(nnz, device=dev, dtype=torch.int64) - start[key[order]]
    sg = key // WIDE_WARPS
    pos = seg_off[sg] + WIDE_HDR + warp_off.reshape(-1)[key] + rank
    code = ((r % WIDE_R) << 9) | (g << 4) | (c % WIDE_CPW)
    enc[pos] = code.to(torch.int32)
    enc16 = torch.where(enc >= 32768, enc - 65536, enc).to(torch.int16)
    cap = int(seg_len.max()) if nseg else WIDE_HDR
    return enc16, seg_off, cap


def gather_encode(rows, cols, neg, d: int, k: int, piece_rows: int, device):
    """K2g encoding (adjoint_gather.cu): S = Omega^T in CSR by target row — for output row q the A
    rows j it sums, ascending, as int32 words j | neg << 31 — and off[q][p], the start of row piece
    p (rows [p * piece_rows, ...)) inside q's list. Built with torch ops on `device`.
    Returns (ent int32 tensor, off int64 tensor [k, npieces + 1])."""
    import torch

    j = torch.as_tensor(rows, device=device).reshape(-1).to(torch.int64)
    q = torch.as_tensor(cols, device=device).reshape(-1).to(torch.int64)
    g = torch.as_tensor(neg, device=device).reshape(-1).to(torch.int64)
    if d >= 2**31:
        raise ValueError("K2g needs d < 2^31")
    key = q * d + j
    skey, order = torch.sort(key)
    word = j[order] | (g[order] << 31)
    ent = torch.where(word >= 2**31, word - 2**32, word).to(torch.int32)
    npieces = -(-d // piece_rows)
    bounds = (torch.arange(k, device=device, dtype=torch.int64)[:, None] * d
              + torch.clamp(torch.arange(npieces + 1, device=device, dtype=torch.int64) * piece_rows, max=d)[None, :])
    off = torch.searchsorted(skey, bounds.reshape(-1)).reshape(k, npieces + 1).to(torch.int64)
    return ent.contiguous(), off.contiguous()


def ring_encode(rows, cols, neg, d: int, k: int):
    """(rows, cols, neg) triplets -> (lists uint8 [16-byte units], seg uint32[nunits*16 + 1]) for K1r.

    For unit h (rows h*128 .. h*128+127 of Omega, two 64-row stages) and consumer warp w (columns
    w*16 .. w*16+15) the segment at byte 16*seg[h*16 + w] holds 16 uint8 column counts, then the
    entries of those columns in column order as little-endian uint16 stage << 15 | (row % 64) << 3 |
    neg (stage = (row // 64) % 2: the byte offset of the row's column inside the unit's two ring
    stages of 64 x 64 float64), padded to 16 bytes.  Duplicated (row, column) entries stay separate
    (their adds sum, as the reference's CSR duplicates do).
    """
    rows = np.asarray(rows, dtype=np.int64).ravel()
    cols = np.asarray(cols, dtype=np.int64).ravel()
    neg = np.asarray(neg, dtype=bool).ravel()
    if k > RING_WARPS * 16:
        raise ValueError("ring encoding needs k <= 256")
    nch = (d + RING_UC - 1) // RING_UC
    nseg = nch * RING_WARPS
    h = rows // RING_UC
    w = cols // 16
    j = cols % 16
    key = (h * RING_WARPS + w) * 16 + j
    order = np.lexsort((rows, key))
    cnt = np.bincount(key, minlength=nseg * 16).reshape(nseg, 16)
    if cnt.size and cnt.max() > 255:
        raise ValueError("more than 255 entries of one column in a 128-row unit")
    per_seg = cnt.sum(axis=1)
    units = 1 + (2 * per_seg + 15) // 16
    seg = np.zeros(nseg + 1, dtype=np.int64)
    np.cumsum(units, out=seg[1:])
    lists = np.zeros(int(seg[-1]) * 16, dtype=np.uint8)
    hdr = (seg[:-1] * 16)[:, None] + np.arange(16)[None, :]
    lists[hdr.ravel()] = cnt.ravel().astype(np.uint8)
    # entry e of segment s lands at 16*seg[s] + 16 + 2 * (its rank inside the segment)
    skey = key[order] // 16
    first = np.zeros(nseg + 1, dtype=np.int64)
    np.cumsum(per_seg, out=first[1:])
    rank = np.arange(rows.size, dtype=np.int64) - first[skey]
    pos = seg[skey] * 16 + 16 + 2 * rank
    r = rows[order] % RING_UC
    ent = ((r // RING_RC) << 15) | ((r % RING_RC) << 3) | neg[order].astype(np.int64)
    lists[pos] = (ent & 0xff).astype(np.uint8)
    lists[pos + 1] = (ent >> 8).astype(np.uint8)
    return lists, seg.astype(np.uint32)


def ring_decode(lists, seg, d: int, k: int):
    """Inverse of ring_encode: (rows, cols, neg) sorted by (unit, warp, column, row)."""
    lists = np.asarray(lists, dtype=np.uint8)
    seg = np.asarray(seg, dtype=np.int64)
    nseg = seg.size - 1
    out_r, out_c, out_n = [], [], []
    for s in range(nseg):
        h, w = divmod(s, RING_WARPS)
        base = int(seg[s]) * 16
        cnt = lists[base:base + 16].astype(np.int64)
        m = int(cnt.sum())
        b = lists[base + 16: base + 16 + 2 * m].astype(np.int64)
        ents = b[0::2] | (b[1::2] << 8)
        cols = np.repeat(w * 16 + np.arange(16), cnt)
        out_r.append(h * RING_UC + (ents >> 15) * RING_RC + ((ents >> 3) & 63))
        out_c.append(cols)
        out_n.append((ents & 1).astype(bool))
    return np.concatenate(out_r), np.concatenate(out_c), np.concatenate(out_n)


def cols_encode(lib, code: int, rows, cols, neg, d: int, k: int):
    """(rows, cols, neg) triplets -> K1c encoding (ent uint32[groups*8, maxp, 32], colmap int32[groups*256],
    tw int32[groups*8], maxp) through sk_sparse_right_cols_encode, or None when the longest warp needs
    more than 128 positions (the caller cuts Omega into row slabs).

    Lane l of warp w computes column colmap[32 w + l]; ent[w, t, l] is half the byte offset into a row
    of A of that lane's t-th entry with its sign in bit 31 (the kernel forms base + 2 * ent, which
    drops the sign bit) (t < tw[w]; positions past a lane's list read
    the zeroed pad after the row).  Columns are dealt to lanes by decreasing list length and each
    lane's order is chosen so that lanes of one 128-byte wavefront read distinct bank slots.
    """
    import ctypes

    from .. import _lib

    rows = np.ascontiguousarray(rows, dtype=np.int64).ravel()
    cols = np.ascontiguousarray(cols, dtype=np.int64).ravel()
    neg = np.ascontiguousarray(neg, dtype=np.uint8).ravel()
    groups = int(lib.sk_sparse_right_cols_groups(k))
    colmap = np.empty(groups * 256, np.int32)
    tw = np.empty(groups * 8, np.int32)
    need = ctypes.c_int32(0)
    args = (code, d, k, rows.size, rows.ctypes.data, cols.ctypes.data, neg.ctypes.data)
    st = lib.sk_sparse_right_cols_encode(*args, 0, None, colmap.ctypes.data, tw.ctypes.data, ctypes.byref(need))
    _lib.check(st, "sk_sparse_right_cols_encode")
    maxp = next((m for m in COLS_MAXP if m >= need.value), None)
    if maxp is None:
        return None
    ent = np.empty(groups * 8 * maxp * 32, np.uint32)
    st = lib.sk_sparse_right_cols_encode(*args, maxp, ent.ctypes.data, colmap.ctypes.data, tw.ctypes.data,
                                         ctypes.byref(need))
    _lib.check(st, "sk_sparse_right_cols_encode")
    return ent.reshape(groups * 8, maxp, 32), colmap, tw, maxp
