"""NumPy Generator draws reproduced on the GPU: test matrices built on the device,
bit-identical to the reference's host construction.

`DevicePhilox` takes a *fresh* `numpy.random.Generator(Philox(SeedSequence(...)))` — the stream the
reference opens for a test matrix (src/core/rng.py:18-70) — reads its key and counter, and produces
the same 32-bit outputs on the device with `sk_philox_u32`. On top of the raw stream it restates
`Generator.integers(0, high, size)` for int64 results (NumPy's Lemire bounded generation on 32-bit
draws: value = (u * high) >> 32, with the rejection of u when (u * high) mod 2^32 falls below
(2^32 - high) mod high — never for power-of-two ranges) and the reference's rejection sampler
`_sample_without_replacement` (src/sketch/sparse.py:18-43). Every call consumes the stream exactly
as NumPy would, so later draws line up.
"""

from __future__ import annotations

import numpy as np

from . import _lib

__all__ = ["DevicePhilox", "device_draws_enabled"]

_MIN_DEVICE_DRAWS = 1 << 16  # below this the host generator is faster than a device round trip


def device_draws_enabled(count: int) -> bool:
    """Large draws go to the GPU when one is present (SKETCH_B200_HOST_RNG=1 forces NumPy)."""
    import os

    if os.environ.get("SKETCH_B200_HOST_RNG") == "1" or count < _MIN_DEVICE_DRAWS:
        return False
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return torch.cuda.is_available()


class DevicePhilox:
    """The 32-bit output stream of a fresh NumPy Philox generator, on a CUDA device."""

    def __init__(self, generator: np.random.Generator, device):
        st = generator.bit_generator.state
        if st.get("bit_generator") != "Philox" or st["buffer_pos"] != 4 or st["has_uint32"] != 0:
            raise ValueError("DevicePhilox needs a fresh numpy Philox generator")
        self.key = np.ascontiguousarray(st["state"]["key"], dtype=np.uint64)
        self.counter = np.ascontiguousarray(st["state"]["counter"], dtype=np.uint64)
        self.device = device
        self.pos = 0  # 32-bit outputs consumed so far

    def _raw(self, start: int, count: int):
        """uint32 outputs [start, start + count) as an int64 device tensor (values < 2^32)."""
        import torch

        first = start // 8 * 8
        skip = start - first
        n = skip + count
        buf = torch.empty(max(8, (n + 7) // 8 * 8), dtype=torch.int32, device=self.device)
        lib = _lib.load()
        with torch.cuda.device(self.device):
            st = lib.sk_philox_u32(self.key.ctypes.data, self.counter.ctypes.data, first, n, buf.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream)
        _lib.check(st, "sk_philox_u32")
        return buf[skip:skip + count].to(torch.int64) & 0xFFFFFFFF

    def integers(self, high: int, size):
        """Generator.integers(0, high, size) (int64), consuming the stream as NumPy does."""
        import torch

        shape = tuple(size) if np.iterable(size) else (int(size),)
        n = int(np.prod(shape))
        high = int(high)
        if high < 1 or high > (1 << 31):
            raise ValueError("integers: need 1 <= high <= 2^31")
        if high == 1 or n == 0:  # rng == 0: NumPy returns the low bound without drawing
            return torch.zeros(shape, dtype=torch.int64, device=self.device)
        threshold = ((1 << 32) - high) % high
        if threshold == 0:
            u = self._raw(self.pos, n)
            self.pos += n
            return ((u * high) >> 32).view(shape)
        # rejection of u with (u * high) mod 2^32 < threshold: keep the first n accepted outputs
        out = []
        need = n
        while need:
            take = need + (need * threshold >> 31) + 64
            u = self._raw(self.pos, take)
            m = u * high
            ok = torch.nonzero((m & 0xFFFFFFFF) >= threshold).flatten()
            if ok.numel() >= need:
                last = int(ok[need - 1])
                out.append((m[ok[:need]] >> 32))
                self.pos += last + 1
                need = 0
            else:
                out.append(m[ok] >> 32)
                self.pos += take
                need -= ok.numel()
        return torch.cat(out).view(shape)

    def sample_without_replacement(self, n_sets: int, take: int, universe: int):
        """The reference's rejection sampler (sparse.py:18-43) on the device, or None when the
        reference would use per-set permutations (acceptance < 5%)."""
        import torch

        if take > universe:
            raise ValueError(f"cannot take {take} distinct items from {universe}")
        if take == universe:
            return torch.arange(universe, device=self.device).repeat(n_sets, 1)
        if np.prod(1.0 - np.arange(take) / universe) < 0.05:
            return None
        out = self.integers(universe, (n_sets, take))
        while True:
            srt = torch.sort(out, dim=1).values
            redo = torch.nonzero((srt[:, 1:] == srt[:, :-1]).any(dim=1)).flatten()
            if redo.numel() == 0:
                return out
            out[redo] = self.integers(universe, (redo.numel(), take))
