"""Pins for oracle.hash_ (H_b, R5) -- CPU only.

  * external test vectors written down in SURVEY.md Sec. 8(c) (golden/hash_vectors.json);
  * the published shift/add form of Thomas Wang's 64-bit integer mix as used by
    minimap2 (restated here: ~x + (x << 21), x ^ x >> 24, x + (x << 3) + (x << 8),
    x ^ x >> 14, x + (x << 2) + (x << 4), x ^ x >> 28, x + (x << 31), each masked);
  * exhaustive bijectivity of H_b for b <= 20 (every step of the mix is a bijection);
  * inverse round trip (orc_unhash) and the inverse multipliers listed in SURVEY.md.
"""
import numpy as np
import pytest

import oracle as O
from conftest import golden


def wang_shift_add(x: int, b: int) -> int:
    m = (1 << b) - 1
    x &= m
    x = ((~x) + (x << 21)) & m
    x = x ^ (x >> 24)
    x = (x + (x << 3) + (x << 8)) & m
    x = x ^ (x >> 14)
    x = (x + (x << 2) + (x << 4)) & m
    x = x ^ (x >> 28)
    x = (x + (x << 31)) & m
    return x


def test_survey_vectors():
    g = golden("hash_vectors.json")
    for v in g["vectors"]:
        assert O.hash_(int(v["x"], 16), v["b"]) == int(v["h"], 16), v
    kv = g["kmer_vector"]
    codes, valid = O.encode(kv["seq"])
    assert valid.all()
    code = O.kmer(codes, 0, kv["k"])
    assert code == int(kv["code"], 16)
    assert O.hash_(code, 2 * kv["k"]) == int(kv["h30"], 16)


def test_inverse_multipliers_listed():
    g = golden("hash_vectors.json")["inverse_multipliers"]
    for b, d in g.items():
        m = (1 << int(b)) - 1
        for a, inv in d.items():
            assert (int(a) * int(inv, 16)) & m == 1


@pytest.mark.parametrize("b", [2, 8, 30, 38, 44, 62])
def test_matches_published_shift_add_form(b):
    rng = np.random.default_rng(b)
    xs = [0, 1, 2, (1 << b) - 1, (1 << (b - 1))] + [int(v) for v in rng.integers(0, 1 << min(b, 63), size=2000, dtype=np.uint64)]
    for x in xs:
        x &= (1 << b) - 1
        assert O.hash_(x, b) == wang_shift_add(x, b), (b, x)


@pytest.mark.parametrize("b", [2, 4, 8, 12, 16, 20])
def test_bijective_exhaustive(b):
    x = np.arange(1 << b, dtype=np.uint64)
    h = O.hash_array(x, b)
    assert h.max() < (1 << b)
    assert len(np.unique(h)) == (1 << b)


@pytest.mark.parametrize("b", [6, 24, 30, 38, 50, 62])
def test_inverse_round_trip(b):
    rng = np.random.default_rng(1000 + b)
    xs = [0, 1, (1 << b) - 1] + [int(v) & ((1 << b) - 1) for v in rng.integers(0, 2 ** 63, size=3000, dtype=np.uint64)]
    for x in xs:
        assert O.unhash(O.hash_(x, b), b) == x


def test_hash_array_matches_scalar():
    x = np.arange(0, 5000, 7, dtype=np.uint64)
    h = O.hash_array(x, 38)
    assert all(int(h[i]) == O.hash_(int(x[i]), 38) for i in range(len(x)))
