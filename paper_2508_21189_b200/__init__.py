"""paper_2508_21189_b200 — B200-native structured-sketch apply (Y = A Omega, S A) for arXiv 2508.21189.

The host layer mirrors the reference `sketchkit` test-matrix API (bit-exact Omega from the same
seeds); every apply runs through libsketch_b200.so (hand-written sm_100a kernels, C ABI in
include/sketch_b200.h).  There is no CPU fallback.
"""

from . import sketch
from .rng import RngStream, derive_seed

__all__ = ["sketch", "RngStream", "derive_seed", "load_library"]
__version__ = "0.1.0"


def load_library():
    """Load (building if needed) libsketch_b200.so and return the ctypes handle."""
    from . import _lib

    return _lib.load()
