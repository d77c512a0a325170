"""Pins for canonical (strand-symmetric) keys, NEXT f4 (R32) -- CPU only.

  * reverse complements computed by hand: ACG -> CGT, AAAA -> TTTT, ACGT -> ACGT (palindrome);
  * involution: rc(rc(x)) = x on random k-mers; canonical(x) = canonical(rc(x));
  * canonical RAW keys equal min(code, rc code) built with Python string operations;
  * strand symmetry: the canonical minimizers of S and of revcomp(S) are mirror images
    (position p <-> n - k - p, same key) when no window holds a repeated key.
"""
import numpy as np
import pytest

import oracle as O

COMP = {ord("A"): "T", ord("C"): "G", ord("G"): "C", ord("T"): "A"}


def _code(s):
    c = 0
    for ch in s:
        c = c * 4 + "ACGT".index(ch)
    return c


def _rc(s):
    return "".join(COMP[ord(ch)] for ch in reversed(s))


def _codes(s):
    return np.frombuffer(s.encode(), np.uint8).copy(), O.encode(s.encode())[0]


@pytest.mark.parametrize("s,rc", [("ACG", "CGT"), ("AAAA", "TTTT"), ("ACGT", "ACGT"), ("GATTACA", "TGTAATC")])
def test_hand_reverse_complements(s, rc):
    codes = O.encode(s.encode())[0]
    assert O.kmer_rc(codes, 0, len(s)) == _code(rc)
    assert _rc(s) == rc


def test_involution_and_canonical_symmetry():
    rng = np.random.default_rng(32)
    for k in (1, 2, 5, 15, 19, 31):
        for _ in range(200):
            s = "".join("ACGT"[x] for x in rng.integers(0, 4, size=k))
            c, r = O.kmer(O.encode(s.encode())[0], 0, k), O.kmer_rc(O.encode(s.encode())[0], 0, k)
            rs = _rc(s)
            assert O.kmer_rc(O.encode(rs.encode())[0], 0, k) == c          # rc(rc(x)) = x
            assert r == _code(rs)
            assert min(c, r) == min(_code(rs), _code(s))                    # canonical(x) = canonical(rc x)


def test_canonical_raw_keys_are_min_of_strands():
    rng = np.random.default_rng(7)
    s = "".join("ACGT"[x] for x in rng.integers(0, 4, size=3000))
    k, w = 9, 1                                                             # w = 1: every k-mer
    key, pos = O.mz(s.encode(), k, w, keymode=O.KEY_CANON_RAW)
    assert len(pos) == len(s) - k + 1
    for p_, kk in zip(pos.tolist(), key.tolist()):
        km = s[p_:p_ + k]
        assert kk == min(_code(km), _code(_rc(km)))


@pytest.mark.parametrize("k,w", [(15, 10), (19, 10), (17, 5)])
def test_strand_symmetry(k, w):
    rng = np.random.default_rng(k * 100 + w)
    n = 20_000
    s = "".join("ACGT"[x] for x in rng.integers(0, 4, size=n))
    r = _rc(s)
    ks, ps = O.mz(s.encode(), k, w, keymode=O.KEY_CANON)
    kr, pr = O.mz(r.encode(), k, w, keymode=O.KEY_CANON)
    # every canonical k-mer key of S, with its position; no repeated key inside any window
    kall, pall = O.mz(s.encode(), k, 1, keymode=O.KEY_CANON)
    for i in range(0, n - k - w + 2):
        assert len(set(kall[i:i + w].tolist())) == w
    assert sorted(zip(ks.tolist(), ps.tolist())) == sorted(zip(kr.tolist(), (n - k - pr).tolist()))
