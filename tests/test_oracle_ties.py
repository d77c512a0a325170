"""Pins for orc_mz_ties, the minimap2-compatible minimizer variant (R35) --
CPU only.  The reading: all tied minima of every window are records, a run of present k-mers
shorter than w is one window (the end rule), symmetric k-mers (canonical modes) are never
selected.  Pinned against things other than itself:

  * hand examples whose answers follow from the reading by inspection (homopolymers, N-split
    short runs, a palindromic 2-mer);
  * a pure-Python brute force written from the reading with string slicing, int() codes and
    Python sets, on tiny inputs over small alphabets (many ties), with N runs and reads;
  * the Fig. 2 oracle: with no repeated key inside any window, no N and n >= k+w-1, all-ties
    selection is exactly the leftmost-argmin selection, so the two outputs are equal;
  * containment: every Fig. 2 record (leftmost argmin of a valid window) is a tied minimum of
    the same window, so orc_mz's set is a subset of orc_mz_ties' set on any input.
"""
import numpy as np
import pytest

import oracle as O

COMP = {"A": "T", "C": "G", "G": "C", "T": "A"}


def _code(s):
    return int(s.translate(str.maketrans("ACGT", "0123")), 4)


def _brute(seq, k, w, keymode, read_off=None):
    s = seq.upper()
    n = len(s)
    starts = set(read_off[1:-1]) if read_off is not None else set()
    canon = keymode in (O.KEY_CANON, O.KEY_CANON_RAW)
    hashed = keymode in (O.KEY_HASH, O.KEY_CANON)
    key, sym = {}, set()
    for q in range(n - k + 1):
        km = s[q:q + k]
        if any(ch not in "ACGT" for ch in km) or any(q < r <= q + k - 1 for r in starts):
            continue
        c = _code(km)
        if canon:
            rc = _code("".join(COMP[ch] for ch in reversed(km)))
            if rc == c:
                sym.add(q)
            c = min(c, rc)
        key[q] = O.hash_(c, 2 * k) if hashed else c
    runs, q = [], 0
    while q < n - k + 1:
        if q not in key:
            q += 1
            continue
        a = q
        while q in key:
            q += 1
        runs.append((a, q))
    sel = set()
    for a, b in runs:
        ww = min(w, b - a)
        for i in range(a, b - ww + 1):
            cand = [p for p in range(i, i + ww) if p not in sym]
            if cand:
                mn = min(key[p] for p in cand)
                sel |= {p for p in cand if key[p] == mn}
    return [(key[p], p) for p in sorted(sel)]


def _pairs(kp):
    return [(int(a), int(b)) for a, b in zip(*kp)]


def test_hand_examples():
    # homopolymer, raw keys: every k-mer ties with every other -> every position
    assert [p for _, p in _pairs(O.mz_ties(b"AAAAAAAA", 2, 3, keymode=O.KEY_RAW))] == list(range(7))
    # k=1 raw, w=10, "ACGT" N "AC": two short runs, each contributes its A
    assert _pairs(O.mz_ties(b"ACGTNAC", 1, 10, keymode=O.KEY_RAW)) == [(0, 0), (0, 5)]
    # canonical raw k=2 on ACGT: AC -> min(AC,GT)=1, CG symmetric (skipped), GT -> 1: {0, 2}
    assert _pairs(O.mz_ties(b"ACGT", 2, 3, keymode=O.KEY_CANON_RAW)) == [(1, 0), (1, 2)]
    # a sequence shorter than k has no k-mers
    assert _pairs(O.mz_ties(b"ACG", 4, 2)) == []
    # all N: nothing
    assert _pairs(O.mz_ties(b"NNNNNNNN", 3, 2)) == []
    # read boundary splits the runs: reads "CCA" | "CA", k=1, w=5 raw -> A of each read
    assert _pairs(O.mz_ties(b"CCACA", 1, 5, keymode=O.KEY_RAW, read_off=[0, 3, 5])) == [(0, 2), (0, 4)]
    # pos_base shifts positions only
    assert _pairs(O.mz_ties(b"ACGTNAC", 1, 10, keymode=O.KEY_RAW, pos_base=100)) == [(0, 100), (0, 105)]


@pytest.mark.parametrize("keymode", [O.KEY_HASH, O.KEY_RAW, O.KEY_CANON, O.KEY_CANON_RAW])
def test_brute_force_tiny(keymode):
    rng = np.random.default_rng(35 + keymode)
    for trial in range(150):
        alpha = ["AC", "ACGT", "ACGTN", "AAAC"][trial % 4]
        n = int(rng.integers(1, 40))
        seq = "".join(alpha[i] for i in rng.integers(0, len(alpha), n))
        k = int(rng.integers(1, 6))
        w = int(rng.integers(1, 8))
        ro = None
        if trial % 3 == 0 and n > 2:
            cuts = sorted(set(int(c) for c in rng.integers(1, n, 2)))
            ro = [0] + cuts + [n]
        got = _pairs(O.mz_ties(seq.encode(), k, w, keymode=keymode, read_off=ro))
        assert got == _brute(seq, k, w, keymode, ro), (seq, k, w, ro)


def test_equals_fig2_without_ties():
    """Random 19-mers under the 38-bit hash: no repeated key in any window of 10 (checked), no N
    -> every window has a unique minimum, and the all-ties set is the Fig. 2 set."""
    rng = np.random.default_rng(7)
    seq = bytes(np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, 20000)])
    k, w = 19, 10
    kt, pt = O.mz_ties(seq, k, w)
    km, pm = O.mz(seq, k, w)
    codes = O.encode(seq)[0]
    keys = O.hash_array(np.array([O.kmer(codes, i, k) for i in range(len(seq) - k + 1)], np.uint64), 2 * k)
    win = np.lib.stride_tricks.sliding_window_view(keys, w)
    assert all(len(set(r.tolist())) == w for r in win)
    np.testing.assert_array_equal(kt, km)
    np.testing.assert_array_equal(pt, pm)


@pytest.mark.parametrize("k,w", [(3, 5), (5, 10), (15, 10)])
def test_contains_fig2(k, w):
    rng = np.random.default_rng(k * 100 + w)
    alpha = np.frombuffer(b"ACGTN", np.uint8)
    p = [0.3, 0.3, 0.2, 0.19, 0.01]
    seq = bytes(alpha[rng.choice(5, 30000, p=p)])
    ro = np.array([0, 7000, 7001, 19000, 30000], np.uint64)
    for km in (O.KEY_HASH, O.KEY_RAW):
        kt, pt = O.mz_ties(seq, k, w, read_off=ro, keymode=km)
        kf, pf = O.mz(seq, k, w, read_off=ro, keymode=km)
        ties = set(zip(pt.tolist(), kt.tolist()))
        assert set(zip(pf.tolist(), kf.tolist())) <= ties
        assert np.all(np.diff(pt.astype(np.int64)) > 0)
