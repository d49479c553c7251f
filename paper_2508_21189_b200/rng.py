"""Seeded, path-addressable Philox streams — bit-compatible with the reference RngStream.

Restates src/core/rng.py:18-70 of the reference: a (root seed, label path) is flattened into
SeedSequence entropy words (ints -> [value mod 2^64, is_negative]; strings -> [little-endian
integer of the UTF-8 bytes, byte length, 2]) and fed to NumPy's Philox bit generator.  Every
test matrix in this package draws from `RngStream(seed, (ClassName, label))`, so the index,
sign and factor arrays are identical to the reference's for the same seed.
"""

from __future__ import annotations

import numpy as np

__all__ = ["RngStream", "derive_seed", "entropy_of"]


def _words(label) -> list[int]:
    if isinstance(label, (bool, np.bool_)):
        raise TypeError("bool is not a valid path label")
    if isinstance(label, (int, np.integer)):
        v = int(label)
        return [v % (1 << 64), 1 if v < 0 else 0]
    if isinstance(label, str):
        raw = label.encode("utf-8")
        return [int.from_bytes(raw, "little"), len(raw), 2]
    raise TypeError(f"unsupported path label type: {type(label)!r}")


def entropy_of(seed: int, path=()) -> list[int]:
    """SeedSequence entropy list for (seed, path) — reference core/rng.py:65-69."""
    ent = _words(int(seed))
    for p in path:
        ent += _words(p)
    return ent


def derive_seed(*parts) -> int:
    """Deterministic 63-bit seed from labels — reference core/rng.py:18-24."""
    ent = []
    for p in parts:
        ent += _words(p)
    s = np.random.SeedSequence(ent).generate_state(2, dtype=np.uint64)
    return int(s[0] ^ (s[1] << np.uint64(1))) & 0x7FFFFFFFFFFFFFFF


class RngStream:
    """Reproducible Philox stream addressed by (root seed, label path)."""

    __slots__ = ("seed", "path")

    def __init__(self, seed: int, path: tuple = ()):
        self.seed = int(seed)
        self.path = tuple(path)

    def substream(self, *labels) -> "RngStream":
        return RngStream(self.seed, self.path + labels)

    def generator(self) -> np.random.Generator:
        return np.random.Generator(np.random.Philox(np.random.SeedSequence(entropy_of(self.seed, self.path))))

    def __repr__(self):
        return f"RngStream({self.seed}, {self.path!r})"
