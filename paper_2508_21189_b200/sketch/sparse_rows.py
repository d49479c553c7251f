"""Sparse sign test matrices on the B200: SparseStack, SparseUniform, SparseIID, SparseCol.

Constructors and random draws restate the reference src/sketch/sparse.py (same RNG stream
path, same draw order, so the index/sign arrays are bit-identical for a seed).  Storage is a
COO triplet (rows, cols, neg) plus one magnitude instead of a SciPy CSR; `matrix` still builds
the reference CSR on demand for code that reads it.  Real operators apply through the native
bcsc kernels: K1 (`sk_sparse_right`, replaces sparse.py:63-66) and K2 (`sk_sparse_adjoint`,
replaces sparse.py:68-78).  Complex-field operators use the dense device GEMM.
"""

from __future__ import annotations

import ctypes

import numpy as np

from .. import _lib
from ..devrng import DevicePhilox, device_draws_enabled
from .encode import (ENT_PAD, PTR_PAD, RING_UC, RING_WARPS, bcsc_encode, bcsc_segments, cols_encode, gather_encode,
                     ring_encode,
                     wide_encode_device)
from .tensorcore import bt_from_triplets, dense_right_tc
from .testmatrix import TestMatrix, entry_sample

__all__ = ["SparseStackTM", "SparseUniformTM", "SparseIIDTM", "SparseColTM", "sample_without_replacement"]


def sample_without_replacement(rng, n_sets: int, take: int, universe: int) -> np.ndarray:
    """n_sets uniform `take`-subsets of range(universe) — same draws as reference sparse.py:18-43.

    iid draws with per-set rejection on duplicates; per-set permutations when the acceptance
    probability is below 5%.
    """
    if take > universe:
        raise ValueError(f"cannot take {take} distinct items from {universe}")
    if take == universe:
        return np.tile(np.arange(universe), (n_sets, 1)) if n_sets else np.empty((0, take), dtype=int)
    if np.prod(1.0 - np.arange(take) / universe) < 0.05:
        out = np.empty((n_sets, take), dtype=np.int64)
        for i in range(n_sets):
            out[i] = rng.permutation(universe)[:take]
        return out
    out = rng.integers(0, universe, size=(n_sets, take))
    while True:
        srt = np.sort(out, axis=1)
        redo = np.flatnonzero((srt[:, 1:] == srt[:, :-1]).any(axis=1))
        if redo.size == 0:
            return out
        out[redo] = rng.integers(0, universe, size=(redo.size, take))


class _SignSparseTM(TestMatrix):
    """Sparse Omega stored as COO (rows, cols, complex-or-real values); native when real +-mag."""

    def __init__(self, d, k, field, seed):
        super().__init__(d, k, field, seed)
        self._coo = None  # (rows int64, cols int64, values float64/complex128)
        self._matrix_cache = None

    def _draw(self):
        """Return (rows, cols, values) in the reference CSR order."""
        raise NotImplementedError

    def _triplets(self):
        if self._coo is None:
            self._coo = self._draw()
        return self._coo

    @property
    def matrix(self):
        """The reference's scipy CSR view (src/sketch/sparse.py:51-55)."""
        if self._matrix_cache is None:
            import scipy.sparse as sp

            rows, cols, vals = self._triplets()
            m = sp.csr_array(sp.coo_array((vals.astype(self.dtype), (rows, cols)), shape=(self.d, self.k)))
            m.sort_indices()
            self._matrix_cache = m
        return self._matrix_cache

    def materialize(self) -> np.ndarray:
        rows, cols, vals = self._triplets()
        out = np.zeros((self.d, self.k), dtype=self.dtype)
        np.add.at(out, (rows, cols), vals)
        return out

    # -- native path ------------------------------------------------------------------------------
    def _sign_form(self):
        """(rows, cols, neg, magnitude) if every value is +-magnitude (real field), else None (cached)."""
        cached = self.__dict__.get("_sign_cache", False)
        if cached is not False:
            return cached
        res = None
        if self.field == "real":
            rows, cols, vals = self._triplets()
            if vals.size == 0:
                res = (rows, cols, np.zeros(0, bool), 1.0)
            else:
                mag = float(np.abs(vals[0]))
                if mag != 0.0 and np.all(np.abs(vals) == mag):
                    res = (rows, cols, vals < 0, mag)
        self._sign_cache = res
        return res

    def _signed_real(self) -> bool:
        """Every value is +-magnitude in the real field (the native sparse kernels apply)."""
        return self._sign_form() is not None

    def _device_sign_form(self, device):
        """(cols (d, zeta), neg (d, zeta), magnitude) as device tensors when the draws live on the
        GPU (rows implicit), else None."""
        return None

    def _bcsc_on(self, device, kind: str, dtype_code: int):
        key = ("bcsc", kind, device, dtype_code)
        if key not in self._device_cache:
            import torch

            lib = _lib.load()
            r = (lib.sk_sparse_right_chunk_rows if kind == "right" else lib.sk_sparse_adjoint_chunk_rows)(
                dtype_code, self.d, self.k)
            _lib.check(min(r, 0), "chunk_rows")
            rows, cols, neg, mag = self._sign_form()
            ptr, ent = bcsc_encode(rows, cols, neg, self.d, self.k, r)
            seg, cap = None, 0
            if kind == "adjoint":
                seg, cap = bcsc_segments(ptr, self.d, self.k, r)
                ptr = np.concatenate([ptr, np.full(PTR_PAD, ptr[-1], np.int32)])
                ent = np.concatenate([ent, np.zeros(ENT_PAD, np.uint16)])
            self._device_cache[key] = (
                torch.from_numpy(ptr).to(device),
                torch.from_numpy(ent.view(np.int16)).to(device),
                int(r),
                mag,
                None if seg is None else torch.from_numpy(seg).to(device),
                cap,
            )
        return self._device_cache[key]

    def right_path(self, dtype) -> str:
        """Kernel used by apply_right for this dtype: 'gather' (K1), 'tc' (K-TC dense) or 'dense'."""
        import os

        import torch

        if self._sign_form() is None or dtype not in (torch.float32, torch.float64):
            return "dense"
        forced = os.environ.get("SKETCH_B200_SPARSE_RIGHT", "auto")
        tc_ok = dtype == torch.float32 and self.k <= 4 * 512 and self.d % 4 == 0
        if forced in ("gather", "tc"):
            return forced if (forced == "gather" or tc_ok) else "gather"
        rows, _, _, _ = self._sign_form()
        per_row = rows.size / max(1, self.d)
        # the dense tensor-core form wins when each row of Omega carries many nonzeros relative to k
        return "tc" if (tc_ok and self.k <= 512 and per_row >= 6) else "gather"

    def _tc_on(self, device):
        key = ("tc", device)
        if key not in self._device_cache:
            rows, cols, neg, mag = self._sign_form()
            hi, lo = bt_from_triplets(rows, cols, neg, self.d, self.k, device)
            self._device_cache[key] = (hi, lo, mag)
        return self._device_cache[key]

    def _right_device(self, a):
        import torch

        path = self.right_path(a.dtype)
        if path == "dense":
            return super()._right_device(a)
        if path == "tc":
            hi, lo, mag = self._tc_on(a.device)
            return dense_right_tc(a, hi, lo, self.k, mag)
        code = _lib.SK_F32 if a.dtype == torch.float32 else _lib.SK_F64
        cols = self._cols_on(a.device, code)
        if cols is not None:
            y = self._right_cols(a, cols, code)
            if y is not None:
                return y
        ring = self._ring_on(a.device) if code == _lib.SK_F64 else None
        if ring is not None:
            return self._right_ring(a, ring)
        ptr, ent, r, mag, _, _ = self._bcsc_on(a.device, "right", code)
        n = a.shape[0]
        y = torch.empty((n, self.k), dtype=a.dtype, device=a.device)
        if n == 0:
            return y
        lib = _lib.load()
        with torch.cuda.device(a.device):
            st = lib.sk_sparse_right(code, a.data_ptr(), n, self.d, a.stride(0), ptr.data_ptr(), ent.data_ptr(), r,
                                     ent.numel(), self.k, mag, y.data_ptr(), y.stride(0),
                                     torch.cuda.current_stream().cuda_stream)
        _lib.check(st, "sk_sparse_right")
        return y

    def _cols_on(self, device, code):
        """K1c encoding (lanes = output columns, sparse_right_cols.cu), cached per device and dtype: a
        list of up to 4 row slabs of Omega (s0, width, ent, colmap, tw, maxp) — one slab unless a
        column's list exceeds 128 entries or a row of A exceeds the shared-memory ring — and the
        magnitude; None when the kernel does not take this operator (SKETCH_B200_K1=ring / classic
        select the older kernels)."""
        import os

        import torch

        key = ("cols", device, code)
        if key not in self._device_cache:
            res = None
            if os.environ.get("SKETCH_B200_K1", "cols") == "cols":
                lib = _lib.load()
                rows, cols, neg, mag = self._sign_form()
                es = 8 if code == _lib.SK_F64 else 4
                # a column longer than 4 slabs x 128 positions cannot fit: skip the encodes outright
                longest = int(np.bincount(cols, minlength=self.k).max()) if cols.size else 0
                nslab = 1 if longest <= 4 * 128 + 64 else 8
                # beyond 4 slabs (lists of > ~400 entries per column) the Y re-reads and the spilling
                # 128-position variant lose to K1r's per-unit walk (tools/k1c_probe.py)
                while res is None and nslab <= 4 and (self.d * es) % 16 == 0:
                    # slab boundaries on multiples of 8 columns of A (16-byte aligned slab starts)
                    cuts = sorted({min(self.d, (self.d * i // nslab) // 8 * 8) for i in range(nslab)} | {self.d})
                    slabs = []
                    for s0, s1 in zip(cuts[:-1], cuts[1:]):
                        m = (rows >= s0) & (rows < s1)
                        enc = cols_encode(lib, code, rows[m] - s0, cols[m], neg[m], s1 - s0, self.k)
                        if enc is None or not lib.sk_sparse_right_cols_supported(code, s1 - s0, self.k, enc[3]):
                            slabs = None
                            break
                        ent, colmap, tw, maxp = enc
                        slabs.append((s0, s1 - s0, torch.from_numpy(ent.view(np.int32)).to(device),
                                      torch.from_numpy(colmap).to(device), torch.from_numpy(tw).to(device), maxp))
                    if slabs:
                        res = (slabs, mag)
                    nslab *= 2
            self._device_cache[key] = res
        return self._device_cache[key]

    def _right_cols(self, a, plan, code):
        """Y = A Omega through K1c (slabs in order, Y = then Y +=); None when A's rows are not 16-byte
        aligned (the caller takes K1r / K1)."""
        import torch

        slabs, mag = plan
        es = a.element_size()
        if a.stride(1) != 1 or a.data_ptr() % 16 or (a.stride(0) * es) % 16:
            return None
        n = a.shape[0]
        y = torch.empty((n, self.k), dtype=a.dtype, device=a.device)
        if n == 0:
            return y
        lib = _lib.load()
        with torch.cuda.device(a.device):
            stream = torch.cuda.current_stream().cuda_stream
            for i, (s0, width, ent, colmap, tw, maxp) in enumerate(slabs):
                st = lib.sk_sparse_right_cols(code, a.data_ptr() + es * s0, n, width, a.stride(0), ent.data_ptr(),
                                              colmap.data_ptr(), tw.data_ptr(), self.k, maxp, mag, y.data_ptr(),
                                              y.stride(0), 1 if i else 0, stream)
                _lib.check(st, "sk_sparse_right_cols")
        return y

    def _ring_on(self, device):
        """K1r encoding (float64 right apply on the warp-specialised ring, k <= 256), cached per
        device: a list of row slabs of Omega (s0, width, lists, seg, bytes) whose lists each fit
        shared memory (one slab when the whole operator does), and the magnitude; None when the ring
        kernel does not take this operator (SKETCH_B200_K1=classic forces the round-1 kernel)."""
        import os

        import torch

        key = ("ring", device)
        if key not in self._device_cache:
            res = None
            if os.environ.get("SKETCH_B200_K1", "ring") != "classic" and self.k <= 256:
                rows, cols, neg, mag = self._sign_form()
                try:
                    lists, seg = ring_encode(rows, cols, neg, self.d, self.k)
                except ValueError:
                    lists = None
                if lists is not None:
                    slabs = self._ring_slabs(lists, seg, device)
                    if slabs is not None:
                        res = (slabs, mag)
            self._device_cache[key] = res
        return self._device_cache[key]

    def _ring_slabs(self, lists, seg, device):
        """Cut the unit sequence (128 rows of Omega each; entries are unit-local, so a slab's lists are a
        contiguous byte range of the full encoding) into the fewest slabs that fit shared memory."""
        import torch

        lib = _lib.load()
        nunits = (self.d + RING_UC - 1) // RING_UC
        w = RING_WARPS  # segments per unit (consumer warps)
        off = seg.astype(np.int64) * 16
        out = []
        h0 = 0
        while h0 < nunits:
            h1 = h0 + 1
            if not self._slab_fits(lib, off, w, h0, h1):
                return None
            while h1 < nunits and self._slab_fits(lib, off, w, h0, h1 + 1):
                h1 += 1
            s0, s1 = h0 * RING_UC, min(self.d, h1 * RING_UC)
            b0, b1 = int(off[h0 * w]), int(off[h1 * w])
            sl = np.ascontiguousarray(lists[b0:b1])
            sg = (seg[h0 * w:h1 * w + 1].astype(np.int64) - seg[h0 * w]).astype(np.uint32)
            out.append((s0, s1 - s0, torch.from_numpy(sl).to(device), torch.from_numpy(sg.view(np.int32)).to(device),
                        int(b1 - b0)))
            h0 = h1
        return out

    def _slab_fits(self, lib, off, w, h0, h1):
        width = min(self.d, h1 * RING_UC) - h0 * RING_UC
        return bool(lib.sk_sparse_right_ring_supported(_lib.SK_F64, width, self.k, int(off[h1 * w] - off[h0 * w])))

    def _right_ring(self, a, ring):
        import torch

        slabs, mag = ring
        if a.stride(1) != 1 or a.data_ptr() % 8:
            a = a.contiguous()
        n = a.shape[0]
        y = torch.empty((n, self.k), dtype=a.dtype, device=a.device)
        if n == 0:
            return y
        lib = _lib.load()
        ws_bytes = max(lib.sk_sparse_right_ring_workspace_bytes(n, s[1]) for s in slabs)  # stream-K partials
        ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=a.device)
        with torch.cuda.device(a.device):
            stream = torch.cuda.current_stream().cuda_stream
            for i, (s0, width, lists, seg, nbytes) in enumerate(slabs):
                st = lib.sk_sparse_right_ring_slab(a.data_ptr() + 8 * s0, n, width, a.stride(0), lists.data_ptr(),
                                                   seg.data_ptr(), nbytes, self.k, mag, y.data_ptr(), y.stride(0),
                                                   1 if i else 0, ws.data_ptr(), ws_bytes, stream)
                _lib.check(st, "sk_sparse_right_ring_slab")
        return y

    def _adjoint_wide_on(self, device):
        """K2w encoding, cached on `device`: built on the GPU from device draws (wide_encode_device),
        else on the host (sk_sparse_adjoint_wide_encode) and uploaded."""
        key = ("adjw", device)
        if key not in self._device_cache:
            import torch

            dform = self._device_sign_form(device)
            if dform is not None:
                cols, neg, mag = dform
                enc, seg_off, cap = wide_encode_device(cols, neg, cols.shape[1], self.d, self.k)
                self._device_cache[key] = (enc, seg_off, cap, mag)
                return self._device_cache[key]
            lib = _lib.load()
            rows, cols, neg, mag = self._sign_form()
            rows = np.ascontiguousarray(rows, dtype=np.int64)
            cols = np.ascontiguousarray(cols, dtype=np.int64)
            negu = np.ascontiguousarray(neg, dtype=np.uint8)
            nseg1 = int(lib.sk_sparse_adjoint_wide_segments(self.d, self.k))
            _lib.check(min(nseg1, 0), "sk_sparse_adjoint_wide_segments")
            seg_off = np.zeros(nseg1, np.int64)
            cap = ctypes.c_int32(0)
            args = (self.d, self.k, rows.size, rows.ctypes.data, cols.ctypes.data, negu.ctypes.data)
            total = lib.sk_sparse_adjoint_wide_encode(*args, None, 0, seg_off.ctypes.data, ctypes.byref(cap))
            _lib.check(min(int(total), 0), "sk_sparse_adjoint_wide_encode")
            enc = np.zeros(max(int(total), 1), np.uint16)
            total = lib.sk_sparse_adjoint_wide_encode(*args, enc.ctypes.data, enc.size, seg_off.ctypes.data,
                                                      ctypes.byref(cap))
            _lib.check(min(int(total), 0), "sk_sparse_adjoint_wide_encode")
            self._device_cache[key] = (torch.from_numpy(enc.view(np.int16)).to(device),
                                       torch.from_numpy(seg_off).to(device), int(cap.value), mag)
        return self._device_cache[key]

    def _gather_csr_on(self, device):
        """S = Omega^T in CSR by target row (K2g entry words + row pointers), built once per device
        with torch ops (from the device draws when they exist)."""
        key = ("adjg_csr", device)
        if key not in self._device_cache:
            import torch

            dform = self._device_sign_form(device)
            if dform is not None:
                cols, neg, mag = dform
                rows = torch.arange(self.d, device=device).repeat_interleave(cols.shape[1])
                ent, off = gather_encode(rows, cols.reshape(-1), neg.reshape(-1), self.d, self.k, self.d, device)
            else:
                rows, cols, neg, mag = self._sign_form()
                ent, off = gather_encode(rows, cols, neg, self.d, self.k, self.d, device)
            rowptr = torch.cat([off[:, 0], off[-1:, 1]])
            self._device_cache[key] = (ent, rowptr, mag)
        return self._device_cache[key]

    def _adjoint_gather_on(self, device, dtype_code: int, m: int):
        """K2g encoding for the launch plan's row pieces: the CSR plus off[q][p] (start of piece p in
        q's list). Piece offsets are derived from the one CSR per piece size (cached)."""
        import ctypes as _ct

        import torch

        lib = _lib.load()
        prows = _ct.c_int64(0)
        npieces = int(lib.sk_sparse_adjoint_gather_pieces(dtype_code, self.d, m, self.k, _ct.byref(prows)))
        _lib.check(min(npieces, 0), "sk_sparse_adjoint_gather_pieces")
        ent, rowptr, mag = self._gather_csr_on(device)
        prows = int(prows.value)
        key = ("adjg_off", device, prows)
        if key not in self._device_cache:
            if npieces == 1:
                off = torch.stack([rowptr[:-1], rowptr[1:]], dim=1).contiguous()
            else:
                counts = rowptr[1:] - rowptr[:-1]
                q = torch.arange(self.k, device=device, dtype=torch.int64).repeat_interleave(counts)
                skey = q * self.d + (ent.to(torch.int64) & 0x7FFFFFFF)
                pstart = torch.clamp(torch.arange(npieces + 1, device=device, dtype=torch.int64) * prows, max=self.d)
                bounds = torch.arange(self.k, device=device, dtype=torch.int64)[:, None] * self.d + pstart[None, :]
                off = torch.searchsorted(skey, bounds.reshape(-1)).reshape(self.k, npieces + 1).contiguous()
                del q, skey
            self._device_cache[key] = off
        return ent, self._device_cache[key], mag

    def _tma_rows_ok(self, b) -> bool:
        """16-byte aligned rows with unit column stride: the TMA-fed adjoints (K2g, K2w) apply."""
        per16 = 16 // b.element_size()
        return b.data_ptr() % 16 == 0 and b.stride(0) % per16 == 0 and b.stride(1) == 1 and b.shape[1] >= 1

    def adjoint_path(self, b) -> str:
        """Kernel used by apply_adjoint: 'narrow' (m <= 8 columns), 'rowgather' (K2g, default for
        aligned float32 / float64), 'wide' (K2w), 'gather' (K2, any layout) or 'dense'.
        SKETCH_B200_SPARSE_ADJOINT picks one."""
        import os

        import torch

        if not self._signed_real() or b.dtype not in (torch.float32, torch.float64):
            return "dense"
        forced = os.environ.get("SKETCH_B200_SPARSE_ADJOINT", "auto")
        if forced == "gather":
            return "gather"
        if forced == "auto" and b.dim() == 2 and 1 <= b.shape[1] <= 8 and (b.shape[1] == 1 or b.stride(1) == 1):
            return "narrow"
        if not self._tma_rows_ok(b):
            return "gather"
        return "wide" if forced == "wide" else "rowgather"

    def _sparse_input_ok(self) -> bool:
        return self._sign_form() is not None

    def _omega_rows_on(self, device):
        """Omega by rows for K1s: int32 indptr[d+1], int32 entries c | neg << 31 (cached)."""
        key = ("omega_rows", device)
        if key not in self._device_cache:
            import torch

            rows, cols, neg, mag = self._sign_form()
            order = np.argsort(rows, kind="stable") if np.any(np.diff(rows) < 0) else slice(None)
            r, c, g = rows[order], cols[order], neg[order]
            ptr = np.zeros(self.d + 1, np.int64)
            np.cumsum(np.bincount(r, minlength=self.d), out=ptr[1:])
            ent = (c.astype(np.int64) | (g.astype(np.int64) << 31)).astype(np.uint32).view(np.int32)
            self._device_cache[key] = (torch.from_numpy(ptr.astype(np.int32)).to(device),
                                       torch.from_numpy(np.ascontiguousarray(ent)).to(device), mag)
        return self._device_cache[key]

    def _right_sparse_input(self, a):
        """A Omega for a SciPy-sparse A without densifying A (reference sparse.py:63-66)."""
        import scipy.sparse as sp
        import torch

        from .._device import require_cuda

        require_cuda()
        a = sp.csr_array(a)
        if np.iscomplexobj(a.data):
            raise NotImplementedError("complex sparse A: densify it first")
        dev = torch.device("cuda", torch.cuda.current_device())
        optr, oent, mag = self._omega_rows_on(dev)
        aptr = torch.from_numpy(a.indptr.astype(np.int64)).to(dev)
        aidx = torch.from_numpy(a.indices.astype(np.int32)).to(dev)
        aval = torch.from_numpy(a.data.astype(np.float64)).to(dev)
        n = a.shape[0]
        y = torch.empty((n, self.k), dtype=torch.float64, device=dev)
        lib = _lib.load()
        st = lib.sk_sparse_right_csr(_lib.SK_F64, n, self.d, aptr.data_ptr(), aidx.data_ptr(), aval.data_ptr(),
                                     optr.data_ptr(), oent.data_ptr(), self.k, mag, y.data_ptr(), y.stride(0),
                                     torch.cuda.current_stream().cuda_stream)
        _lib.check(st, "sk_sparse_right_csr")
        return y.cpu().numpy()

    def adjoint_rows(self, b_rows, r0: int, r1: int, out, accumulate: bool) -> None:
        """out (+)= Omega[r0:r1]^T b_rows for a float32 device block b_rows = B[r0:r1] (K2w).

        r0 must be a multiple of 128 (the encoding's row chunk); used to stream a tall operand
        through L2 one row block at a time while other kernels reuse the same block.
        """
        import torch

        if self.adjoint_path(b_rows) == "gather" or not self._tma_rows_ok(b_rows):
            raise NotImplementedError("adjoint_rows needs an aligned float32 or float64 device block (wide path)")
        enc, seg_off, cap, mag = self._adjoint_wide_on(b_rows.device)
        m = b_rows.shape[1]
        lib = _lib.load()
        f64 = b_rows.dtype == torch.float64
        ws_bytes = (lib.sk_sparse_adjoint_wide_workspace_bytes_f64 if f64 else
                    lib.sk_sparse_adjoint_wide_workspace_bytes)(r1 - r0, m, self.k)
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=b_rows.device)
        fn = lib.sk_sparse_adjoint_wide_rows_f64 if f64 else lib.sk_sparse_adjoint_wide_rows
        with torch.cuda.device(b_rows.device):
            st = fn(b_rows.data_ptr(), self.d, r0, r1, m, b_rows.stride(0),
                                                 enc.data_ptr(), seg_off.data_ptr(), cap, self.k, mag,
                                                 out.data_ptr(), out.stride(0), 1 if accumulate else 0,
                                                 ws.data_ptr(), ws_bytes, torch.cuda.current_stream().cuda_stream)
        _lib.check(st, "sk_sparse_adjoint_wide_rows")

    def _adjoint_device(self, b):
        import torch

        path = self.adjoint_path(b)
        if path == "dense":
            return super()._adjoint_device(b)
        if path == "narrow":
            code = _lib.SK_F32 if b.dtype == torch.float32 else _lib.SK_F64
            m = b.shape[1]
            ent, off, mag = self._adjoint_gather_on(b.device, code, m)
            out = torch.empty((self.k, m), dtype=b.dtype, device=b.device)
            lib = _lib.load()
            with torch.cuda.device(b.device):
                st = lib.sk_sparse_adjoint_narrow(code, b.data_ptr(), self.d, m, b.stride(0), ent.data_ptr(),
                                                  off.data_ptr(), off.shape[1] - 1, self.k, mag, out.data_ptr(),
                                                  out.stride(0), torch.cuda.current_stream().cuda_stream)
            _lib.check(st, "sk_sparse_adjoint_narrow")
            return out
        if path == "rowgather":
            code = _lib.SK_F32 if b.dtype == torch.float32 else _lib.SK_F64
            m = b.shape[1]
            ent, off, mag = self._adjoint_gather_on(b.device, code, m)
            out = torch.empty((self.k, m), dtype=b.dtype, device=b.device)
            lib = _lib.load()
            ws_bytes = lib.sk_sparse_adjoint_gather_workspace_bytes(code, self.d, m, self.k)
            ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=b.device)
            with torch.cuda.device(b.device):
                st = lib.sk_sparse_adjoint_gather(code, b.data_ptr(), self.d, m, b.stride(0), ent.data_ptr(),
                                                  off.data_ptr(), self.k, mag, out.data_ptr(), out.stride(0), 0,
                                                  ws.data_ptr(), ws_bytes, torch.cuda.current_stream().cuda_stream)
            _lib.check(st, "sk_sparse_adjoint_gather")
            return out
        if path == "wide":
            enc, seg_off, cap, mag = self._adjoint_wide_on(b.device)
            m = b.shape[1]
            out = torch.empty((self.k, m), dtype=b.dtype, device=b.device)
            lib = _lib.load()
            f64 = b.dtype == torch.float64
            ws_bytes = (lib.sk_sparse_adjoint_wide_workspace_bytes_f64 if f64 else
                        lib.sk_sparse_adjoint_wide_workspace_bytes)(self.d, m, self.k)
            ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=b.device)
            fn = lib.sk_sparse_adjoint_wide_f64 if f64 else lib.sk_sparse_adjoint_wide
            with torch.cuda.device(b.device):
                st = fn(b.data_ptr(), self.d, m, b.stride(0), enc.data_ptr(), seg_off.data_ptr(),
                                                cap, self.k, mag, out.data_ptr(), out.stride(0), 0, ws.data_ptr(),
                                                ws_bytes, torch.cuda.current_stream().cuda_stream)
            _lib.check(st, "sk_sparse_adjoint_wide")
            return out
        code = _lib.SK_F32 if b.dtype == torch.float32 else _lib.SK_F64
        ptr, ent, r, mag, seg, cap = self._bcsc_on(b.device, "adjoint", code)
        m = b.shape[1]
        out = torch.empty((self.k, m), dtype=b.dtype, device=b.device)
        if m == 0:
            return out
        lib = _lib.load()
        ws_bytes = lib.sk_sparse_adjoint_workspace_bytes(code, self.d, m, self.k)
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=b.device)
        with torch.cuda.device(b.device):
            st = lib.sk_sparse_adjoint(code, b.data_ptr(), self.d, m, b.stride(0), ptr.data_ptr(), ent.data_ptr(), r,
                                       seg.data_ptr() if seg is not None else None, cap, self.k, mag,
                                       out.data_ptr(), out.stride(0), 0, ws.data_ptr(), ws_bytes,
                                       torch.cuda.current_stream().cuda_stream)
        _lib.check(st, "sk_sparse_adjoint")
        return out


class SparseStackTM(_SignSparseTM):
    """zeta CountSketch blocks of width b side by side; one +-1/sqrt(zeta) per block per row.

    Reference: src/sketch/sparse.py:81-174 (same signature and defaults).
    """

    def __init__(self, d: int, zeta: int = 4, block_size: int | None = None, *, k: int | None = None,
                 distribution: str | None = None, field: str = "real", seed: int = 0):
        if zeta < 1:
            raise ValueError("row sparsity zeta must be >= 1")
        if block_size is None:
            if k is None:
                raise ValueError("give either block_size or k")
            if k % zeta:
                raise ValueError(f"k={k} must be divisible by zeta={zeta}")
            block_size = k // zeta
        if block_size < 1:
            raise ValueError("block size must be >= 1")
        super().__init__(d, block_size * zeta, field, seed)
        self.zeta = int(zeta)
        self.block_size = int(block_size)
        self.distribution = distribution or ("steinhaus" if field == "complex" else "real_rademacher")
        self._assigned = None

    @classmethod
    def from_assignments(cls, signs, buckets, block_size, field="real"):
        """Test-fixture constructor from explicit (d, zeta) sign / bucket arrays (sparse.py:118-126)."""
        signs = np.asarray(signs)
        buckets = np.asarray(buckets)
        d, zeta = signs.shape
        tm = cls(d, zeta, block_size, field=field, seed=0)
        tm._coo = tm._assemble(signs, buckets)
        return tm

    def _assemble(self, signs, buckets):
        d, zeta, b = self.d, self.zeta, self.block_size
        cols = (np.asarray(buckets) + np.arange(zeta)[None, :] * b).ravel()
        vals = (np.asarray(signs) / np.sqrt(zeta)).astype(self.dtype).ravel()
        return np.repeat(np.arange(d), zeta), cols.astype(np.int64), vals

    def _draw(self):
        rng = self._rng("entries")
        if self.distribution == "real_rademacher" and device_draws_enabled(self.d * self.zeta):
            import torch

            g = DevicePhilox(rng, torch.device("cuda", torch.cuda.current_device()))
            buckets = g.integers(self.block_size, (self.d, self.zeta)).cpu().numpy()
            signs = (g.integers(2, (self.d, self.zeta)) * 2 - 1).cpu().numpy().astype(np.float64)
            return self._assemble(signs, buckets)
        buckets = rng.integers(0, self.block_size, size=(self.d, self.zeta))
        signs = entry_sample(self.distribution, rng, (self.d, self.zeta))
        return self._assemble(signs, buckets)

    def redraw(self, seed: int) -> "SparseStackTM":
        return SparseStackTM(self.d, self.zeta, self.block_size, distribution=self.distribution, field=self.field,
                             seed=seed)


class SparseUniformTM(_SignSparseTM):
    """Exactly zeta nonzeros per row at columns sampled without replacement (sparse.py:177-220)."""

    def __init__(self, d: int, k: int, zeta: int = 4, *, field: str = "real", seed: int = 0):
        if zeta < 1 or zeta > k:
            raise ValueError(f"need 1 <= zeta <= k, got zeta={zeta}, k={k}")
        super().__init__(d, k, field, seed)
        self.zeta = int(zeta)

    def _draw(self):
        dd = self._device_draw()
        if dd is not None:
            cols, neg = dd
            mag = 1.0 / np.sqrt(self.zeta)
            vals = np.where(neg.cpu().numpy().ravel(), -mag, mag).astype(self.dtype)
            return np.repeat(np.arange(self.d), self.zeta), cols.cpu().numpy().ravel(), vals
        rng = self._rng("entries")
        cols = sample_without_replacement(rng, self.d, self.zeta, self.k)
        cols.sort(axis=1)
        signs = rng.integers(0, 2, size=(self.d, self.zeta)) * 2.0 - 1.0
        vals = (signs / np.sqrt(self.zeta)).astype(self.dtype).ravel()
        return np.repeat(np.arange(self.d), self.zeta), cols.ravel().astype(np.int64), vals

    def _device_draw(self):
        """(cols (d, zeta) int64 sorted per row, neg (d, zeta) bool) drawn on the GPU (devrng), cached;
        None when the host generator draws (small operators, permutation regime, no GPU)."""
        if "_dev_draw" in self.__dict__:
            return self._dev_draw
        res = None
        if device_draws_enabled(self.d * self.zeta):
            import torch

            g = DevicePhilox(self._rng("entries"), torch.device("cuda", torch.cuda.current_device()))
            cols = g.sample_without_replacement(self.d, self.zeta, self.k)
            if cols is not None:
                cols = torch.sort(cols, dim=1).values
                res = (cols, g.integers(2, (self.d, self.zeta)) == 0)
        self._dev_draw = res
        return res

    def _signed_real(self) -> bool:
        if self.field == "real" and self._coo is None and self._device_draw() is not None:
            return True  # +-1/sqrt(zeta) by construction; no host copy of the draws needed
        return super()._signed_real()

    def _device_sign_form(self, device):
        if self.field != "real" or self._device_draw() is None:
            return None
        cols, neg = self._device_draw()
        return cols.to(device), neg.to(device), 1.0 / np.sqrt(self.zeta)

    def redraw(self, seed: int) -> "SparseUniformTM":
        return SparseUniformTM(self.d, self.k, self.zeta, field=self.field, seed=seed)


class SparseIIDTM(_SignSparseTM):
    """iid zeta^{-1/2} * sign * Bernoulli(zeta/k) entries by geometric skipping (sparse.py:223-266)."""

    def __init__(self, d: int, k: int, zeta: float = 4.0, *, field: str = "real", seed: int = 0):
        if not (0.0 < zeta <= k):
            raise ValueError(f"expected row sparsity in (0, k], got {zeta}")
        super().__init__(d, k, field, seed)
        self.zeta = float(zeta)

    @staticmethod
    def _bernoulli_positions(rng, p: float, total: int) -> np.ndarray:
        if p >= 1.0:
            return np.arange(total)
        found = []
        pos = -1
        batch = int(total * p * 1.2) + 16
        while True:
            steps = np.cumsum(rng.geometric(p, size=batch)) + pos
            inside = steps[steps < total]
            found.append(inside)
            if inside.size < steps.size:
                break
            pos = int(steps[-1])
        return np.concatenate(found)

    def _draw(self):
        rng = self._rng("entries")
        flat = self._bernoulli_positions(rng, self.zeta / self.k, self.d * self.k)
        signs = rng.integers(0, 2, size=flat.size) * 2.0 - 1.0
        vals = (signs / np.sqrt(self.zeta)).astype(self.dtype)
        return (flat // self.k).astype(np.int64), (flat % self.k).astype(np.int64), vals

    def redraw(self, seed: int) -> "SparseIIDTM":
        return SparseIIDTM(self.d, self.k, self.zeta, field=self.field, seed=seed)


class SparseColTM(_SignSparseTM):
    """Column sampler: xi distinct rows per column, value +-sqrt(d/xi)/sqrt(k) (sparse.py:298-339)."""

    def __init__(self, d: int, k: int, xi: int = 8, *, field: str = "real", seed: int = 0):
        if xi < 1 or xi > d:
            raise ValueError(f"need 1 <= xi <= d, got xi={xi}, d={d}")
        super().__init__(d, k, field, seed)
        self.xi = int(xi)
        self._colwise = None

    def column_draws(self):
        """(rows (k, xi), neg (k, xi), magnitude) in draw order — the SRTT sampler encoding."""
        if self._colwise is None:
            rng = self._rng("entries")
            rows = sample_without_replacement(rng, self.k, self.xi, self.d)
            signs = rng.integers(0, 2, size=(self.k, self.xi)) * 2.0 - 1.0
            self._colwise = (rows.astype(np.int64), signs < 0, float(np.sqrt(self.d / self.xi) / np.sqrt(self.k)))
        return self._colwise

    def _draw(self):
        rows, neg, mag = self.column_draws()
        vals = np.where(neg, -1.0, 1.0) * mag
        cols = np.repeat(np.arange(self.k), self.xi)
        r = rows.ravel()
        order = np.lexsort((cols, r))
        return r[order], cols[order].astype(np.int64), vals.ravel()[order].astype(self.dtype)

    def redraw(self, seed: int) -> "SparseColTM":
        return SparseColTM(self.d, self.k, self.xi, field=self.field, seed=seed)


class SparseRowBlockTM(_SignSparseTM):
    """Rows [r0, r1) of a sparse test matrix, as an operator of its own (multi-GPU row shards).

    Rank g of a row-sharded job holds A[r0:r1, :] and applies this block: its adjoint partial
    Omega[r0:r1]^* A_g is summed across ranks by one all-reduce.  When the parent's
    draws live on the GPU (device-drawn SparseUniform), the block slices those device arrays — no
    host triplets of the whole operator are formed on any rank; host triplets of the block itself
    are only built if a host view (`matrix`, `materialize`) is asked for.
    """

    def __init__(self, parent: _SignSparseTM, r0: int, r1: int):
        if not (0 <= r0 < r1 <= parent.d):
            raise ValueError(f"bad row block [{r0}, {r1}) of d={parent.d}")
        super().__init__(r1 - r0, parent.k, parent.field, parent.seed)
        self.parent = parent
        self.row_offset = int(r0)
        self._dev = None
        dd = parent._device_draw() if hasattr(parent, "_device_draw") and parent._coo is None else None
        if dd is not None:
            cols, neg = dd
            self._dev = (cols[r0:r1], neg[r0:r1], 1.0 / np.sqrt(parent.zeta))
            self.zeta = parent.zeta
            return
        rows, cols, vals = parent._triplets()
        lo, hi = np.searchsorted(rows, [r0, r1])
        if np.any(np.diff(rows) < 0):  # unsorted rows (SparseCol CSR order is sorted; others row-major)
            sel = (rows >= r0) & (rows < r1)
            self._coo = (rows[sel] - r0, cols[sel], vals[sel])
        else:
            self._coo = (rows[lo:hi] - r0, cols[lo:hi], vals[lo:hi])

    def _device_draw(self):
        return None if self._dev is None else self._dev[:2]

    def _draw(self):
        if self._dev is None:
            return self._coo
        cols, neg, mag = self._dev
        z = cols.shape[1]
        vals = np.where(neg.cpu().numpy().ravel(), -mag, mag).astype(self.dtype)
        return np.repeat(np.arange(self.d), z), cols.cpu().numpy().ravel().astype(np.int64), vals

    def _signed_real(self) -> bool:
        if self._dev is not None and self._coo is None:
            return self.field == "real"
        return super()._signed_real()

    def _device_sign_form(self, device):
        if self._dev is None or self.field != "real":
            return None
        cols, neg, mag = self._dev
        return cols.to(device), neg.to(device), mag

    def redraw(self, seed: int):
        raise NotImplementedError("redraw the parent operator instead")


class EmptyRowBlockTM:
    """A zero-row block (a rank that holds no rows when n < world size): zero partials."""

    def __init__(self, parent, r0: int):
        self.parent = parent
        self.row_offset = int(r0)
        self.d = 0
        self.k = parent.k

    def apply_adjoint(self, b):
        import torch

        m = b.shape[1] if b.dim() == 2 else 1
        out = torch.zeros((self.k, m) if b.dim() == 2 else (self.k,), dtype=b.dtype, device=b.device)
        return out

    def apply_right(self, a):
        import torch

        return torch.zeros((a.shape[0], self.k), dtype=a.dtype, device=a.device)


def _row_block(self, r0: int, r1: int):
    """Rows [r0, r1) as an operator; cached on the parent so repeated sharded calls reuse its encoding.
    An empty range gives an operator with zero partials (ranks without rows when n < world size)."""
    if r0 == r1:
        if not 0 <= r0 <= self.d:
            raise ValueError(f"bad row block [{r0}, {r1}) of d={self.d}")
        return EmptyRowBlockTM(self, r0)
    cache = self.__dict__.setdefault("_row_blocks", {})
    key = (int(r0), int(r1))
    if key not in cache:
        cache[key] = SparseRowBlockTM(self, r0, r1)
    return cache[key]


_SignSparseTM.row_block = _row_block
