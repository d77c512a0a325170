"""Pins for oracle.slsum / oracle.prefix (Eq. 1, Eq. 2 of PAPER.md) -- CPU only.

The oracle is checked against things other than itself:
  * SPEC.md worked examples (tests/golden/spec_examples.json);
  * the closed form of the u32-add sliding sum as a difference of prefix sums
    computed by numpy.cumsum (exact mod 2^32);
  * numpy sliding_window_view(...).min/max (a library routine);
  * float32 add vs math.fsum within the rounding-error bound of a w-term sum;
  * the affine operator by EVALUATING the composed maps on test points
    (function-application semantics, not the coefficient formula);
  * w = 1 is the identity; w = n gives the full fold (= last prefix sum).
"""
import math

import numpy as np
import pytest
from numpy.lib.stride_tricks import sliding_window_view

import oracle as O
from conftest import golden

OPS = {"min_u32": O.MIN_U32, "max_u32": O.MAX_U32, "add_u32": O.ADD_U32}


def test_spec_examples_slsum():
    g = golden("spec_examples.json")
    for ex in g["slsum"]:
        y = O.slsum(OPS[ex["op"]], ex["w"], np.array(ex["x"], np.uint32))
        assert y.tolist() == ex["y"], ex["line"]


def test_spec_examples_prefix_suffix():
    g = golden("spec_examples.json")
    for ex in g["prefix"]:
        assert O.prefix(OPS[ex["op"]], np.array(ex["x"], np.uint32)).tolist() == ex["y"], ex["line"]
    for ex in g["suffix"]:
        # suffix folds = prefix of the reversed sequence, reversed (valid for commutative ops)
        x = np.array(ex["x"], np.uint32)
        # and, independently, each suffix as a one-window sliding sum with w = len(suffix)
        got = [int(O.slsum(OPS[ex["op"]], len(x) - i, x[i:])[0]) for i in range(len(x))]
        assert got == ex["y"], ex["line"]


@pytest.mark.parametrize("w", [1, 2, 3, 4, 7, 16, 33, 64, 255])
def test_add_u32_closed_form(w):
    rng = np.random.default_rng(w)
    x = rng.integers(0, 2 ** 32, size=5000, dtype=np.uint64).astype(np.uint32)
    ps = np.concatenate([np.zeros(1, np.uint64), np.cumsum(x.astype(np.uint64))])  # exact (< 2^45)
    want = ((ps[w:] - ps[:-w]) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    assert np.array_equal(O.slsum(O.ADD_U32, w, x), want)


@pytest.mark.parametrize("w", [1, 2, 5, 10, 17, 64, 100])
def test_min_max_vs_numpy(w):
    rng = np.random.default_rng(100 + w)
    for hi in (4, 2 ** 32):  # small alphabet forces ties
        x = rng.integers(0, hi, size=3000, dtype=np.uint64).astype(np.uint32)
        v = sliding_window_view(x, w)
        assert np.array_equal(O.slsum(O.MIN_U32, w, x), v.min(axis=1))
        assert np.array_equal(O.slsum(O.MAX_U32, w, x), v.max(axis=1))
        x64 = rng.integers(0, 2 ** 63, size=2000, dtype=np.uint64)
        assert np.array_equal(O.slsum(O.MIN_U64, w, x64), sliding_window_view(x64, w).min(axis=1))


@pytest.mark.parametrize("w", [1, 4, 16, 64, 256, 1024])
def test_add_f32_within_rounding_bound(w):
    rng = np.random.default_rng(7 + w)
    x = rng.standard_normal(4096).astype(np.float32)
    y = O.slsum(O.ADD_F32, w, x)
    xd = x.astype(np.float64)
    u = 2.0 ** -24
    for i in range(0, len(y), max(1, len(y) // 300)):
        exact = math.fsum(xd[i:i + w].tolist())
        bound = (w - 1) * u * float(np.abs(xd[i:i + w]).sum()) * 1.0001 + 1e-30
        assert abs(float(y[i]) - exact) <= bound, (i, w)
    if w == 1:
        assert np.array_equal(y, x)


def test_add_f32_is_strict_left_fold_in_float32():
    # the fold order matters in float32: (1e8 + 1) + -1e8 = 0 but 1 + (-1e8 + 1) ... differ
    x = np.array([1e8, 1.0, -1e8, 1.0], np.float32)
    y = O.slsum(O.ADD_F32, 3, x)
    left0 = np.float32(np.float32(x[0] + x[1]) + x[2])
    left1 = np.float32(np.float32(x[1] + x[2]) + x[3])
    assert y[0] == left0 and y[1] == left1


def _apply(a, b, t):
    return (a * t + b) & 0xFFFFFFFF


@pytest.mark.parametrize("w", [1, 2, 3, 5, 8, 13])
def test_affine_by_evaluation(w):
    rng = np.random.default_rng(w)
    n = 200
    x = rng.integers(0, 2 ** 32, size=(n, 2), dtype=np.uint64).astype(np.uint32)
    y = O.slsum(O.AFFINE_U32X2, w, x)
    assert y.shape == (n - w + 1, 2)
    for i in range(0, n - w + 1, 7):
        for t in (0, 1, 12345, 2 ** 32 - 1):
            # x_i (+) ... (+) x_{i+w-1} is the map t -> f_i(f_{i+1}(... f_{i+w-1}(t)))
            v = t
            for j in range(i + w - 1, i - 1, -1):
                v = _apply(int(x[j, 0]), int(x[j, 1]), v)
            assert _apply(int(y[i, 0]), int(y[i, 1]), t) == v


def test_affine_not_commutative_fixture():
    # guards against an oracle that silently reorders operands
    x = np.array([[2, 3], [5, 7]], np.uint32)
    y = O.slsum(O.AFFINE_U32X2, 2, x)
    assert y.tolist() == [[10, 17]]           # t -> 2(5t+7)+3
    y2 = O.slsum(O.AFFINE_U32X2, 2, x[::-1].copy())
    assert y2.tolist() == [[10, 22]]          # t -> 5(2t+3)+7


def test_degenerate_sizes():
    x = np.arange(5, dtype=np.uint32)
    assert O.slsum(O.ADD_U32, 6, x).shape == (0,)
    assert O.slsum(O.ADD_U32, 5, x).tolist() == [int(O.prefix(O.ADD_U32, x)[-1])]
    assert np.array_equal(O.slsum(O.MIN_U32, 1, x), x)
    assert O.slsum(O.MIN_U32, 3, np.zeros(0, np.uint32)).shape == (0,)
    with pytest.raises(ValueError):
        O.slsum(O.MIN_U32, 0, x)


def test_prefix_matches_cumsum_and_accumulate():
    rng = np.random.default_rng(3)
    x = rng.integers(0, 2 ** 32, size=1000, dtype=np.uint64).astype(np.uint32)
    assert np.array_equal(O.prefix(O.ADD_U32, x), (np.cumsum(x.astype(np.uint64)) & np.uint64(0xFFFFFFFF)).astype(np.uint32))
    assert np.array_equal(O.prefix(O.MIN_U32, x), np.minimum.accumulate(x))


# ---------------------------------------------------------------- concatenation
@pytest.mark.parametrize("sigma,w", [(4, 15), (4, 16), (20, 7), (20, 9), (256, 4), (256, 6), (3, 1)])
def test_concat_is_base_sigma_numeral(sigma, w):
    """k-mers "as a sliding sum ... string concatenation": folding (b, sigma) over
    w symbols gives the base-sigma numeral of the w-mer and sigma^w, mod 2^32.  Pinned to
    Python big-integer arithmetic (exact, then reduced)."""
    rng = np.random.default_rng(sigma * 100 + w)
    n = 300
    b = rng.integers(0, sigma, size=n, dtype=np.uint64).astype(np.uint32)
    x = np.stack([b, np.full(n, sigma, np.uint32)], axis=1)
    y = O.slsum(O.CONCAT_U32X2, w, x)
    for i in range(n - w + 1):
        v = sum(int(b[i + t]) * sigma ** (w - 1 - t) for t in range(w))
        assert int(y[i, 0]) == v % 2 ** 32
        assert int(y[i, 1]) == sigma ** w % 2 ** 32


def test_concat_dna_equals_kmer_codes():
    """For DNA (sigma = 4, k <= 16) the concatenation fold is the k-mer code of a2."""
    seq = b"ACGTTGCAACGGTACCATGCAAGT" * 5
    codes, valid = O.encode(seq)
    assert valid.all()
    x = np.stack([codes.astype(np.uint32), np.full(len(codes), 4, np.uint32)], axis=1)
    for k in (3, 11, 16):
        y = O.slsum(O.CONCAT_U32X2, k, x)
        assert [int(v) for v in y[:, 0]] == [O.kmer(codes, i, k) for i in range(len(seq) - k + 1)]


def test_concat_not_commutative_fixture():
    x = np.array([[1, 10], [2, 10]], np.uint32)     # "1" then "2" in base 10
    assert O.slsum(O.CONCAT_U32X2, 2, x).tolist() == [[12, 100]]
    assert O.slsum(O.CONCAT_U32X2, 2, x[::-1].copy()).tolist() == [[21, 100]]
