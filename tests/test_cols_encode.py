"""K1c encoding (sk_sparse_right_cols_encode, CPU side of the C ABI): every Omega entry lands in
exactly one (warp, position, lane) slot of its column's lane, padding reads the zeroed pad after the
row, and the bank-slot schedule leaves few extra wavefronts."""

import numpy as np
import pytest

from paper_2508_21189_b200 import _lib
from paper_2508_21189_b200.sketch.encode import cols_encode


def _triplets(d, k, zeta, seed):
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(d), zeta)
    cols = np.concatenate([rng.choice(k, zeta, replace=False) for _ in range(d)])
    neg = rng.random(rows.size) < 0.5
    return rows, cols, neg


def _decode(ent, colmap, tw, d, es):
    out, pads = [], 0
    for w in range(ent.shape[0]):
        for t in range(int(tw[w])):
            for ln in range(32):
                v = int(ent[w, t, ln])
                r = (v & 0x7FFFFFFF) * 2 // es
                if r < d:
                    assert colmap[w * 32 + ln] >= 0
                    out.append((r, int(colmap[w * 32 + ln]), v >> 31))
                else:
                    assert d <= r < d + 128 // es and not v >> 31
                    pads += 1
    return sorted(out), pads


def _extra_wavefronts(ent, tw, d, es):
    lanes = 16 if es == 8 else 32
    c = 128 // es
    extra = total = 0
    for w in range(ent.shape[0]):
        for t in range(int(tw[w])):
            for h in range(0, 32, lanes):
                cls = ((ent[w, t, h:h + lanes] & 0x7FFFFFFF) * 2 // es) % c
                extra += int(np.bincount(cls, minlength=c).max()) - 1
                total += 1
    return extra, total


@pytest.mark.parametrize("code,es", [(_lib.SK_F64, 8), (_lib.SK_F32, 4)])
@pytest.mark.parametrize("d,k,zeta", [(4096, 256, 4), (1000, 300, 5), (513, 17, 3), (64, 600, 4), (700, 64, 1)])
def test_cols_encode_roundtrip(code, es, d, k, zeta):
    lib = _lib.load()
    rows, cols, neg = _triplets(d, k, zeta, d + k)
    enc = cols_encode(lib, code, rows, cols, neg, d, k)
    assert enc is not None
    ent, colmap, tw, maxp = enc
    groups = (k + 255) // 256
    assert ent.shape == (groups * 8, maxp, 32) and maxp in (32, 64, 96, 128)
    assert np.all(tw % 8 == 0) and tw.max() <= maxp
    # lanes cover the columns once; every warp's positions cover its longest list
    used = colmap[colmap >= 0]
    assert sorted(used.tolist()) == list(range(k))
    got, _ = _decode(ent, colmap, tw, d, es)
    assert got == sorted(zip(rows.tolist(), cols.tolist(), neg.astype(int).tolist()))
    counts = np.bincount(cols, minlength=k)
    for w in range(tw.size):
        lane_cols = colmap[32 * w:32 * w + 32]
        assert tw[w] >= max([counts[c] for c in lane_cols if c >= 0] + [0])


def test_cols_encode_config1_schedule():
    """Config 1 operator shape: the shared-memory wavefronts of one row's gathers (one per half-warp
    and position, plus bank conflicts) within 20 % of the entries' floor (16 lane-loads each)."""
    lib = _lib.load()
    d, k = 4096, 256
    rows, cols, neg = _triplets(d, k, 4, 0)
    ent, colmap, tw, maxp = cols_encode(lib, _lib.SK_F64, rows, cols, neg, d, k)
    assert maxp == 96
    extra, total = _extra_wavefronts(ent, tw, d, 8)
    assert total + extra <= 1.2 * rows.size / 16
    assert extra <= 0.05 * total


def test_cols_encode_duplicates_and_long_lists():
    lib = _lib.load()
    rows = np.array([3, 3, 5, 0, 9], np.int64)
    cols = np.array([1, 1, 1, 0, 1], np.int64)
    neg = np.array([0, 1, 0, 1, 0], bool)
    ent, colmap, tw, maxp = cols_encode(lib, _lib.SK_F64, rows, cols, neg, 10, 2)
    got, _ = _decode(ent, colmap, tw, 10, 8)
    assert got == sorted(zip(rows.tolist(), cols.tolist(), neg.astype(int).tolist()))
    # a column longer than 128 entries has no single-pass encoding
    r = np.arange(200, dtype=np.int64)
    assert cols_encode(lib, _lib.SK_F64, r, np.zeros(200, np.int64), np.zeros(200, bool), 200, 1) is None


def test_cols_encode_rejects_bad_indices():
    lib = _lib.load()
    with pytest.raises(ValueError, match="index out of range"):
        cols_encode(lib, _lib.SK_F64, np.array([5]), np.array([0]), np.array([False]), 4, 2)
