"""Pins for oracle.lookup (seed lookup, Fig. 1 / PAPER.md L63-65 "lookups to 'CG' and 'CT'",
SURVEY NEXT f1; reading DESIGN.md R30) -- CPU only.

  * the "ACGTACGT" table (k=3, w=2, raw 6-bit keys, direct index) gives
    ACG -> [0, 4]; a seed never stored -> [];
  * a Python dict {seed: [positions]} built straight from the records (exact when 2k <= 32);
  * for 2k > 32: hits are exactly the records whose key shares the top 32 bits (brute force);
  * partition property: looking up every stored seed once, in sorted order, reproduces the
    position table.
"""
import numpy as np
import pytest

import oracle as O


def _dict_hits(key, pos):
    d = {}
    for kk, pp in zip(key.tolist(), pos.tolist()):
        d.setdefault(kk, []).append(pp)
    return d


def test_spec_acgtacgt_example():
    # minimizers of "ACGTACGT", k=3, w=2 with raw keys: (ACG,0) (CGT,1) (GTA,2) (ACG,4)
    key, pos = O.mz(b"ACGTACGT", 3, 2, keymode=O.KEY_RAW)
    assert list(zip(key.tolist(), pos.tolist())) == [(0b000110, 0), (0b011011, 1), (0b101100, 2), (0b000110, 4)]
    off, fp, pt = O.seedtable(key, pos, 3, 6)          # direct index: bits = 2k
    acg, tta = 0b000110, 0b111100
    ho, hp = O.lookup(np.array([acg, tta], np.uint64), 3, 6, off, fp, pt)
    assert hp[int(ho[0]):int(ho[1])].tolist() == [0, 4]
    assert hp[int(ho[1]):int(ho[2])].tolist() == []


@pytest.mark.parametrize("k,bits", [(15, 24), (12, 24), (8, 16), (3, 6)])
def test_exact_seed_hits_vs_dict(k, bits):
    """2k <= 32: the fingerprint is the whole key, hits = every stored position of the seed."""
    rng = np.random.default_rng(k * 7 + bits)
    m = 30_000
    key = rng.integers(0, min(1 << (2 * k), 5000), size=m, dtype=np.uint64)   # many repeats
    pos = np.sort(rng.choice(10 ** 8, size=m, replace=False)).astype(np.uint64)
    off, fp, pt = O.seedtable(key, pos, k, bits)
    q = np.concatenate([key[rng.integers(0, m, size=2000)], rng.integers(0, 1 << (2 * k), size=500,
                                                                          dtype=np.uint64)])
    ho, hp = O.lookup(q, k, bits, off, fp, pt)
    d = _dict_hits(key, pos)
    assert ho[0] == 0 and np.all(ho[1:] >= ho[:-1])
    for i, x in enumerate(q.tolist()):
        assert hp[int(ho[i]):int(ho[i + 1])].tolist() == d.get(x, []), i


def test_wide_keys_match_on_fingerprint():
    """2k > 32 (k=19): hits are the records whose key agrees on its top 32 bits."""
    k, bits = 19, 24
    rng = np.random.default_rng(3)
    m = 20_000
    base = rng.integers(0, 1 << 32, size=300, dtype=np.uint64)
    key = (base[rng.integers(0, 300, size=m)] << np.uint64(6)) | rng.integers(0, 64, size=m, dtype=np.uint64)
    pos = np.arange(m, dtype=np.uint64) * 3
    off, fp, pt = O.seedtable(key, pos, k, bits)
    q = key[rng.integers(0, m, size=400)]
    ho, hp = O.lookup(q, k, bits, off, fp, pt)
    for i, x in enumerate(q.tolist()):
        want = [int(p) for kk, p in zip(key.tolist(), pos.tolist()) if (kk >> 6) == (x >> 6)]
        assert hp[int(ho[i]):int(ho[i + 1])].tolist() == want


def test_partition_property():
    k, bits = 12, 20
    rng = np.random.default_rng(9)
    key = rng.integers(0, 1 << (2 * k), size=10_000, dtype=np.uint64)
    pos = np.sort(rng.choice(10 ** 7, size=10_000, replace=False)).astype(np.uint64)
    off, fp, pt = O.seedtable(key, pos, k, bits)
    seeds = np.unique(key)          # ascending key = ascending bucket, then fingerprint
    ho, hp = O.lookup(seeds, k, bits, off, fp, pt)
    assert int(ho[-1]) == len(key)
    # inside a bucket the table keeps input (position) order; per seed the hits ascend
    order = np.lexsort((pos, key))
    assert np.array_equal(hp, pos[order])
    assert np.array_equal(np.sort(hp), np.sort(pt))
