"""Pins for oracle.seedtable (Fig. 1; bucketing DESIGN.md R21) -- CPU only.

  * the fingerprint is the top 32 bits of the 2k-bit key (explicit values);
  * the table equals a construction with Python's stable `sorted` by bucket;
  * offsets: offsets[0] = 0, offsets[-1] = M, non-decreasing, = cumsum of np.bincount;
  * partition property: concatenating every bucket's slice gives all entries in
    (bucket, input order); multiset(entries) = multiset(input);
  * the Fig. 1 / SPEC S:L318 style lookup on a raw k=2 table.
"""
import numpy as np
import pytest

import oracle as O


def test_fingerprint_values():
    assert O.fingerprint(0x3FFFFFFFFF, 19) == 0xFFFFFFFF
    assert O.fingerprint(0x1DF06F29BC, 19) == 0x1DF06F29BC >> 6
    assert O.fingerprint(0x3FF06F15, 15) == (0x3FF06F15 << 2) & 0xFFFFFFFF
    assert O.fingerprint(0xFFFF, 8) == 0xFFFF0000
    assert O.fingerprint(1, 16) == 1


@pytest.mark.parametrize("k,bits", [(15, 24), (19, 24), (15, 16), (8, 12), (19, 8)])
def test_against_sorted(k, bits):
    rng = np.random.default_rng(k * 100 + bits)
    m = 20000
    key = rng.integers(0, 1 << (2 * k), size=m, dtype=np.uint64)
    pos = np.sort(rng.choice(10 ** 9, size=m, replace=False)).astype(np.uint64)
    offsets, fp, pos_out = O.seedtable(key, pos, k, bits)
    fps = [O.fingerprint(int(x), k) for x in key]
    bk = [f >> (32 - bits) for f in fps]
    order = sorted(range(m), key=lambda e: bk[e])          # stable
    assert pos_out.tolist() == [int(pos[e]) for e in order]
    assert fp.tolist() == [fps[e] for e in order]
    cnt = np.bincount(np.array(bk), minlength=1 << bits)
    assert offsets[0] == 0 and offsets[-1] == m
    assert np.array_equal(offsets[1:], np.cumsum(cnt).astype(np.uint64))
    # partition property: bucket b's slice holds exactly its entries, ascending pos
    for b in rng.choice(1 << bits, size=50):
        sl = pos_out[offsets[b]: offsets[b + 1]]
        assert np.all(np.diff(sl.astype(np.int64)) > 0)
        assert sorted(sl.tolist()) == sorted(int(pos[e]) for e in range(m) if bk[e] == b)
    assert sorted(pos_out.tolist()) == sorted(pos.tolist())


def test_raw_k2_lookup_like_fig1():
    # records [(CT,3),(CG,5),(CT,0)], k=2; with bits = 2k = 4 the buckets are the
    # 16 seeds in lexicographic order, so the table is Fig. 1's pointer + position table.
    CT, CG = 0b0111, 0b0110
    key = np.array([CT, CG, CT], np.uint64)
    pos = np.array([3, 5, 0], np.uint64)
    offsets, fp, pos_out = O.seedtable(key, pos, 2, 4)
    assert pos_out[offsets[CG]: offsets[CG + 1]].tolist() == [5]
    assert sorted(pos_out[offsets[CT]: offsets[CT + 1]].tolist()) == [0, 3]
    assert offsets.tolist() == [0] * 7 + [1] + [3] * 9


def test_empty_and_errors():
    offsets, fp, pos_out = O.seedtable(np.zeros(0, np.uint64), np.zeros(0, np.uint64), 15, 10)
    assert offsets.sum() == 0 and len(pos_out) == 0
    with pytest.raises(ValueError):
        O.seedtable(np.zeros(1, np.uint64), np.zeros(1, np.uint64), 5, 12)  # bits > 2k
