"""Test matrices drawn on the GPU (devrng) are bit-identical to the host NumPy draws and to the
reference's full-size BASELINE matrices (golden sha1 digests made by importing sketchkit)."""

import hashlib

import numpy as np
import pytest

from paper_2508_21189_b200 import devrng
from paper_2508_21189_b200 import sketch as skb
from paper_2508_21189_b200.rng import RngStream

pytestmark = pytest.mark.gpu


def sha1(a):
    return hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("high", [2, 3, 200, 256, 2047, 2048, 1000003, 1 << 31])
def test_integers_match_numpy(high, cuda):
    gen = RngStream(7, ("devrng", str(high))).generator()
    g = devrng.DevicePhilox(gen, cuda)
    want = RngStream(7, ("devrng", str(high))).generator()
    for size in [(5,), (1000, 3), (77777,), (1,)]:
        got = g.integers(high, size).cpu().numpy()
        ref = want.integers(0, high, size=size)
        assert np.array_equal(got, ref), (high, size)


@pytest.mark.parametrize("d,k,zeta,seed", [(200000, 2048, 8, 1), (100000, 200, 8, 2), (70000, 12, 3, 3),
                                           (65536, 9, 9, 4), (300000, 64, 4, 5)])
def test_sparse_uniform_device_equals_host(d, k, zeta, seed, cuda, monkeypatch):
    dev = skb.SparseUniformTM(d, k, zeta, seed=seed)._triplets()
    monkeypatch.setenv("SKETCH_B200_HOST_RNG", "1")
    host = skb.SparseUniformTM(d, k, zeta, seed=seed)._triplets()
    for a, b in zip(dev, host):
        assert np.array_equal(a, b)


def test_sparse_stack_device_equals_host(cuda, monkeypatch):
    dev = skb.SparseStackTM(300000, 4, 64, seed=8)._triplets()
    monkeypatch.setenv("SKETCH_B200_HOST_RNG", "1")
    host = skb.SparseStackTM(300000, 4, 64, seed=8)._triplets()
    for a, b in zip(dev, host):
        assert np.array_equal(a, b)


def test_config_matrices_match_reference_digests(golden_hashes, cuda):
    for name, (d, k, zeta) in {"cfg1_sparseuniform_4096_256_4_s0": (4096, 256, 4),
                               "cfg3_sparseuniform_16384_200_8_s0": (16384, 200, 8),
                               "cfg4_sparseuniform_4194304_2048_8_s0": (4194304, 2048, 8)}.items():
        h = golden_hashes[name]
        assert devrng.device_draws_enabled(d * zeta) == (d * zeta >= 1 << 16)
        rows, cols, vals = skb.SparseUniformTM(d, k, zeta, seed=0)._triplets()
        assert sha1(cols) == h["indices"], name
        assert sha1(vals) == h["data"], name
