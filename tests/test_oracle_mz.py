"""Pins for oracle.encode / pack / kmer / mz (Sec. 2.4) -- CPU only.

  * Fig. 2 caption facts on a constructed instance;
  * SPEC.md worked examples (S:L227-229, S:L237-238, S:L307, S:L309 corrected);
  * a numpy brute force written from the definition with library primitives
    (k-mer codes as a weighted sum over sliding_window_view, window argmin via
    numpy argmin = first occurrence = leftmost, records = np.unique of the
    winners of valid windows) on random inputs with N's, segments, small alphabets;
  * exhaustive enumeration of all 4^8 strings as one segmented batch;
  * invariants (D3): positions strictly increasing, every valid window's winner stored;
  * the density statement of L85 (statistical band, golden/density.json);
  * shard partition (R25): concatenating window-range outputs = the full output.
"""
import itertools

import numpy as np
import pytest
from numpy.lib.stride_tricks import sliding_window_view

import oracle as O
from conftest import golden
from synthgen import host as G

ACGT = "ACGT"


def decode(code, k):
    return "".join(ACGT[(code >> (2 * (k - 1 - t))) & 3] for t in range(k))


# ------------------------------------------------------------ encode / pack / kmer
def test_spec_encode():
    for ex in golden("spec_examples.json")["encode"]:
        c, v = O.encode(ex["seq"])
        assert c.tolist() == ex["codes"] and v.astype(int).tolist() == ex["valid"], ex["line"]


def test_encode_all_bytes():
    s = np.arange(256, dtype=np.uint8)
    c, v = O.encode(s)
    ok = {ord(ch): i for i, ch in enumerate("ACGT")}
    ok.update({ord(ch): i for i, ch in enumerate("acgt")})
    for b in range(256):
        assert bool(v[b]) == (b in ok)
        assert int(c[b]) == ok.get(b, 0)


def test_pack_layout():
    s = G.c1_ascii(1000, seed=5)
    s[[3, 40, 999]] = ord("N")
    words, inval = O.pack(s)
    assert len(words) == 32 and len(inval) == 32
    c, v = O.encode(s)
    for i in range(1000):
        t, j = divmod(i, 32)
        assert (int(words[t]) >> (62 - 2 * j)) & 3 == c[i]
        assert ((int(inval[t]) >> j) & 1) == (0 if v[i] else 1)
    # tail bits of the last word are zero
    assert int(inval[-1]) >> 8 == 0 and int(words[-1]) & ((1 << 48) - 1) == 0


def test_spec_kmers():
    ex = golden("spec_examples.json")["kmers"]
    c, v = O.encode(ex[0]["seq"])
    assert [O.kmer(c, i, 3) for i in range(3)] == ex[0]["codes"]
    # only k-mers fully inside valid bases
    c, v = O.encode(ex[1]["seq"])
    k = ex[1]["k"]
    good = [i for i in range(len(v) - k + 1) if v[i:i + k].all()]
    assert good == ex[1]["pos"]


def test_kmer_round_trip_and_lexicographic():
    rng = np.random.default_rng(0)
    for k in (1, 2, 5, 15, 19, 31):
        s = "".join(rng.choice(list(ACGT), size=k))
        c, _ = O.encode(s)
        assert decode(O.kmer(c, 0, k), k) == s
    # MSB-first codes sort lexicographically (Fig. 1 lists seeds lexicographically)
    words = ["".join(p) for p in itertools.product(ACGT, repeat=3)]
    codes = [O.kmer(O.encode(wd)[0], 0, 3) for wd in words]
    assert codes == sorted(codes) and codes == list(range(64))


# ------------------------------------------------------------ brute force
def wang(x: np.ndarray, b: int) -> np.ndarray:
    """Published shift/add form of the Wang/minimap2 mix, vectorised (see test_oracle_hash)."""
    m = np.uint64((1 << b) - 1)
    x = x.astype(np.uint64) & m
    with np.errstate(over="ignore"):
        x = ((~x) + (x << np.uint64(21))) & m
        x = x ^ (x >> np.uint64(24))
        x = (x + (x << np.uint64(3)) + (x << np.uint64(8))) & m
        x = x ^ (x >> np.uint64(14))
        x = (x + (x << np.uint64(2)) + (x << np.uint64(4))) & m
        x = x ^ (x >> np.uint64(28))
        x = (x + (x << np.uint64(31))) & m
    return x


def brute_mz(seq: bytes, k: int, w: int, keymode=O.KEY_HASH, read_off=None):
    s = np.frombuffer(seq, np.uint8) & 0xDF          # upper-case letters
    n = len(s)
    if n < k + w - 1:
        return np.zeros(0, np.uint64), np.zeros(0, np.uint64)
    lut = np.zeros(256, np.int64) - 1
    for i, ch in enumerate(b"ACGT"):
        lut[ch] = i
    code = lut[s]
    valid = code >= 0
    code = np.where(valid, code, 0).astype(np.uint64)
    wts = (np.uint64(4) ** np.arange(k - 1, -1, -1, dtype=np.uint64))
    kc = (sliding_window_view(code, k) * wts).sum(axis=1, dtype=np.uint64)
    key = kc if keymode == O.KEY_RAW else wang(kc, 2 * k)
    span = k + w - 1
    seg = np.zeros(n, np.int64) if read_off is None else np.searchsorted(np.asarray(read_off), np.arange(n), side="right") - 1
    wv = sliding_window_view(valid, span).all(axis=1) & (seg[: n - span + 1] == seg[span - 1:])
    best = sliding_window_view(key, w).argmin(axis=1) + np.arange(len(key) - w + 1)
    best = best[: n - span + 1]
    p = np.unique(best[wv])
    return key[p], p.astype(np.uint64)


def test_fig2_caption_facts():
    g = golden("fig2_minimizers.json")
    key, pos = O.mz(g["seq"], g["k"], g["w"], keymode=O.KEY_RAW)
    assert pos.tolist() == g["stored_positions"]
    assert not set(g["dropped_positions"]) & set(pos.tolist())
    assert len(g["seq"]) - (g["k"] + g["w"] - 1) + 1 == g["n_windows"]
    # ('CTT', 2) is the minimizer of windows 1 and 2, stored once
    i = pos.tolist().index(g["shared"]["pos"])
    assert decode(int(key[i]), g["k"]) == g["shared"]["seed"]
    for wi in g["shared"]["windows"]:
        sub = g["seq"][wi: wi + g["k"] + g["w"] - 1]
        k2, p2 = O.mz(sub, g["k"], g["w"], keymode=O.KEY_RAW)
        assert p2.tolist() == [g["shared"]["pos"] - wi]


def test_spec_minimizer_examples():
    for ex in golden("spec_examples.json")["minimizers_raw"]:
        key, pos = O.mz(ex["seq"], ex["k"], ex["w"], keymode=O.KEY_RAW)
        assert pos.tolist() == ex["pos"], ex["line"]
        assert [decode(int(x), ex["k"]) for x in key] == ex["seeds"], ex["line"]


def test_w1_is_every_valid_kmer():
    s = G.c1_ascii(3000, seed=9)
    s[[10, 11, 500]] = ord("N")
    for k in (1, 3, 15):
        key, pos = O.mz(s, k, 1)
        c, v = O.encode(s)
        good = [i for i in range(len(s) - k + 1) if v[i:i + k].all()]
        assert pos.tolist() == good


def _random_seq(rng, n, alphabet=b"ACGT", pn=0.0, lower=0.0):
    s = np.frombuffer(alphabet, np.uint8)[rng.integers(0, len(alphabet), size=n)].copy()
    if pn:
        s[rng.random(n) < pn] = ord("N")
    if lower:
        m = rng.random(n) < lower
        s[m] = s[m] | 0x20
    return s


@pytest.mark.parametrize("keymode", [O.KEY_RAW, O.KEY_HASH])
def test_brute_force_random(keymode):
    rng = np.random.default_rng(11 + keymode)
    for trial in range(300):
        n = int(rng.integers(0, 120))
        k = int(rng.integers(1, 8))
        w = int(rng.integers(1, 12))
        alpha = [b"A", b"AC", b"ACGT"][trial % 3]
        s = _random_seq(rng, n, alpha, pn=0.05 if trial % 2 else 0.0, lower=0.1)
        ro = None
        if trial % 4 == 3 and n > 2:
            cuts = np.sort(rng.choice(np.arange(1, n), size=min(3, n - 1), replace=False))
            ro = np.concatenate([[0], cuts, [n]]).astype(np.uint64)
        want_k, want_p = brute_mz(s.tobytes(), k, w, keymode, ro)
        got_k, got_p = O.mz(s, k, w, read_off=ro, keymode=keymode)
        assert np.array_equal(got_p, want_p), (trial, n, k, w)
        assert np.array_equal(got_k, want_k), (trial, n, k, w)


def test_brute_force_larger_k():
    rng = np.random.default_rng(5)
    for k, w in [(15, 10), (19, 10), (31, 5), (16, 16), (21, 3)]:
        s = _random_seq(rng, 4000, pn=0.002)
        assert all(np.array_equal(a, b) for a, b in zip(O.mz(s, k, w), brute_mz(s.tobytes(), k, w)))


def test_exhaustive_4_pow_8_segmented():
    L = 8
    allw = np.array(list(itertools.product(range(4), repeat=L)), np.uint8)  # 65536 x 8
    seq = np.frombuffer(b"ACGT", np.uint8)[allw].reshape(-1)
    ro = np.arange(0, len(seq) + 1, L, dtype=np.uint64)
    for k in (1, 2, 3):
        for w in (1, 2, 3, 4):
            for keymode in (O.KEY_RAW, O.KEY_HASH):
                key, pos = O.mz(seq, k, w, read_off=ro, keymode=keymode)
                # per-string brute force, vectorised over all strings
                wts = (4 ** np.arange(k - 1, -1, -1)).astype(np.uint64)
                kc = (sliding_window_view(allw.astype(np.uint64), k, axis=1) * wts).sum(axis=2, dtype=np.uint64)
                kk = kc if keymode == O.KEY_RAW else wang(kc, 2 * k)
                best = sliding_window_view(kk, w, axis=1).argmin(axis=2) + np.arange(L - k - w + 2)
                rows = np.repeat(np.arange(len(allw)), best.shape[1])
                gp = np.unique(rows * L + best.reshape(-1))
                assert np.array_equal(pos, gp.astype(np.uint64)), (k, w, keymode)
                assert np.array_equal(key, kk.reshape(-1)[(gp // L) * kk.shape[1] + gp % L]), (k, w, keymode)


def test_invariants_and_winner_coverage():
    rng = np.random.default_rng(2)
    s = _random_seq(rng, 5000, b"AC", pn=0.01)
    k, w = 4, 6
    key, pos = O.mz(s, k, w, keymode=O.KEY_RAW)
    assert np.all(np.diff(pos.astype(np.int64)) > 0)
    # every valid window's leftmost winner is stored, and every stored pos wins some valid window
    _, want = brute_mz(s.tobytes(), k, w, O.KEY_RAW)
    assert np.array_equal(pos, want)


def test_shard_partition():
    rng = np.random.default_rng(3)
    s = _random_seq(rng, 3000, pn=0.01)
    k, w = 5, 4
    full_k, full_p = O.mz(s, k, w)
    nwin = len(s) - (k + w - 1) + 1
    for G_ in (2, 3, 5):
        cuts = [nwin * g // G_ for g in range(G_ + 1)]
        parts = [O.mz(s, k, w, win_lo=cuts[g], win_hi=cuts[g + 1]) for g in range(G_)]
        assert np.array_equal(np.concatenate([p[1] for p in parts]), full_p)
        assert np.array_equal(np.concatenate([p[0] for p in parts]), full_k)
        # halo rule (R25): shard g only needs bases [a-1, b+k+w-2)
        for g in range(G_):
            a, b = cuts[g], cuts[g + 1]
            lo = max(0, a - 1)
            sub = s[lo: b + k + w - 2]
            kk, pp = O.mz(sub, k, w, pos_base=lo, win_lo=a - lo)
            assert np.array_equal(pp, parts[g][1]) and np.array_equal(kk, parts[g][0])


def test_density_c1():
    g = golden("density.json")
    s = G.c1_ascii(1_000_000)
    key, pos = O.mz(s, 15, 10)
    nwin = len(s) - 24 + 1
    d = len(pos) / nwin
    lo, hi = g["bands"]["k15_uniform"]
    assert lo <= d <= hi, d
    gap = (int(pos[-1]) - int(pos[0])) / (len(pos) - 1)
    glo, ghi = g["spec_mean_gap_band"]
    assert glo <= gap <= ghi


def test_density_k19_gc41():
    g = golden("density.json")
    c3 = G.C3(n=2_000_000)
    s = c3.ascii()
    key, pos = O.mz(s, 19, 10)
    valid = s != ord("N")
    nwin = int(sliding_window_view(valid, 28).all(axis=1).sum())   # valid windows only
    d = len(pos) / nwin
    lo, hi = g["bands"]["k19_gc41"]
    assert lo <= d <= hi, d


def test_degenerate():
    assert O.mz("ACG", 3, 2)[1].size == 0           # n < k + w - 1
    assert O.mz("ACGT", 3, 2)[1].tolist() in ([0], [1])
    assert O.mz("NNNNNNNN", 3, 2)[1].size == 0
    with pytest.raises(ValueError):
        O.mz("ACGT", 0, 2)
    with pytest.raises(ValueError):
        O.mz("ACGT", 32, 2)
