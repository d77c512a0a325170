"""MSDT serialization (SPEC S:L356 layout) -- CPU only: round trips of a direct
(Fig. 1, 4^k pointers) and a hashed table, the SPEC "ACGTACGT" entries, rejected headers."""
import struct

import numpy as np
import pytest

import oracle as O

M = pytest.importorskip("paper_1811_10074_b200.msdt")


def test_direct_spec_example(tmp_path):
    key, pos = O.mz(b"ACGTACGT", 3, 2, keymode=O.KEY_RAW)
    off, fp, pt = O.seedtable(key, pos, 3, 6)                 # direct index: bits = 2k
    p = tmp_path / "t.msdt"
    M.save(str(p), off, fp, pt, 3, 2, M.MODE_DIRECT)
    t = M.load(str(p))
    assert (t["mode"], t["k"], t["w"]) == (M.MODE_DIRECT, 3, 2)
    assert np.array_equal(t["offsets"], off)
    acg, cgt, gta = 0b000110, 0b011011, 0b101100
    assert list(zip(t["seeds"].tolist(), t["pos"].tolist())) == [(acg, 0), (acg, 4), (cgt, 1), (gta, 2)]
    raw = p.read_bytes()
    assert raw[:4] == b"MSDT" and struct.unpack_from("<I", raw, 4)[0] == 1
    assert len(raw) == 20 + 8 * (4 ** 3 + 1) + 16 * 4


@pytest.mark.parametrize("k", [2, 8, 12])
def test_direct_round_trip(tmp_path, k):
    rng = np.random.default_rng(k)
    key = rng.integers(0, 4 ** k, size=5000, dtype=np.uint64)
    pos = np.sort(rng.choice(10 ** 7, size=5000, replace=False)).astype(np.uint64)
    off, fp, pt = O.seedtable(key, pos, k, 2 * k)
    M.save(str(tmp_path / "d.msdt"), off, fp, pt, k, 10, M.MODE_DIRECT)
    t = M.load(str(tmp_path / "d.msdt"))
    assert np.array_equal(t["offsets"], off) and np.array_equal(t["pos"], pt)
    # every entry's seed is its bucket in the pointer table
    bucket = np.repeat(np.arange(4 ** k, dtype=np.uint64), np.diff(off.astype(np.int64)))
    assert np.array_equal(t["seeds"], bucket)


def test_hashed_round_trip_and_rejects(tmp_path):
    rng = np.random.default_rng(3)
    key = rng.integers(0, 1 << 38, size=3000, dtype=np.uint64)
    pos = np.arange(3000, dtype=np.uint64) * 9
    off, fp, pt = O.seedtable(key, pos, 19, 24)
    p = tmp_path / "h.msdt"
    M.save(str(p), off, fp, pt, 19, 10, M.MODE_HASHED)
    t = M.load(str(p))
    o = np.argsort(fp, kind="stable")
    assert t["offsets"] is None and np.array_equal(t["seeds"], fp[o].astype(np.uint64)) and np.array_equal(t["pos"], pt[o])
    # SPEC's sorted-hash layout: seeds non-decreasing, positions ascending within a seed, and the
    # entries are exactly the (fingerprint, position) pairs of the records
    sd, ps = t["seeds"], t["pos"]
    assert bool(np.all(sd[1:] >= sd[:-1]))
    same = sd[1:] == sd[:-1]
    assert bool(np.all(ps[1:][same] > ps[:-1][same]))
    fpk = np.array([O.fingerprint(int(x), 19) for x in key], dtype=np.uint64)
    assert sorted(zip(sd.tolist(), ps.tolist())) == sorted(zip(fpk.tolist(), pos.tolist()))
    # binary search of the seed column finds every record
    for j in range(0, 3000, 97):
        lo, hi = np.searchsorted(sd, fpk[j], "left"), np.searchsorted(sd, fpk[j], "right")
        assert pos[j] in ps[lo:hi]
    raw = bytearray(p.read_bytes())
    bad = tmp_path / "bad.msdt"
    bad.write_bytes(b"XSDT" + raw[4:])
    with pytest.raises(ValueError):
        M.load(str(bad))
    raw[4:8] = struct.pack("<I", 2)
    bad.write_bytes(bytes(raw))
    with pytest.raises(ValueError):
        M.load(str(bad))
    with pytest.raises(ValueError):
        M.save(str(p), off, fp, pt, 19, 10, M.MODE_DIRECT)     # not a direct-index table
