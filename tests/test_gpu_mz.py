"""GPU parity: mz_encode / mz_extract_ex vs the oracle (Sec. 2.4, Fig. 2).
Bit-exact: every (hash, pos) record, in order, and the count."""
import itertools

import numpy as np
import pytest
import torch

import oracle as O
from synthgen import host as G

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1811_10074_b200")


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_mz(seq, k, w, *, path=0, packed=False, keymode=P.MZ_KEY_HASH, read_off=None, pos_base=0, win_lo=0,
           win_hi=P.U64_MAX, capacity=None):
    s = _dev(O.as_bytes(seq))
    ro = None if read_off is None else _dev(np.asarray(read_off, np.uint64))
    if packed:
        words, inval = P.mz_encode(s)
        h, p, c = P.mz_extract_ex(words, k, w, n=s.numel(), kind=P.MZ_IN_PACKED2, invalid=inval, read_off=ro,
                                  pos_base=pos_base, win_lo=win_lo, win_hi=win_hi, keymode=keymode,
                                  capacity=capacity, path=path)
    else:
        h, p, c = P.mz_extract_ex(s, k, w, read_off=ro, pos_base=pos_base, win_lo=win_lo, win_hi=win_hi,
                                  keymode=keymode, capacity=capacity, path=path)
    torch.cuda.synchronize()
    cnt = int(c.item())
    m = min(cnt, h.numel())
    return h[:m].cpu().numpy(), p[:m].cpu().numpy(), cnt


def _rand_seq(rng, n, alpha=b"ACGT", pn=0.0, lower=0.0, junk=0.0):
    s = np.frombuffer(alpha, np.uint8)[rng.integers(0, len(alpha), size=n)].copy()
    if pn:
        s[rng.random(n) < pn] = ord("N")
    if lower:
        m = rng.random(n) < lower
        s[m] |= 0x20
    if junk:
        m = rng.random(n) < junk
        s[m] = rng.integers(0, 256, size=int(m.sum()), dtype=np.uint8)
    return s


def _same(seq, k, w, **kw):
    want_k, want_p = O.mz(seq, k, w, read_off=kw.get("read_off"), keymode=kw.get("keymode", O.KEY_HASH),
                          pos_base=kw.get("pos_base", 0), win_lo=kw.get("win_lo", 0),
                          win_hi=kw.get("win_hi", 2 ** 64 - 1))
    got_k, got_p, cnt = gpu_mz(seq, k, w, **kw)
    assert cnt == len(want_p), (k, w, cnt, len(want_p))
    assert np.array_equal(got_p, want_p), (k, w)
    assert np.array_equal(got_k, want_k), (k, w)


# ------------------------------------------------------------------ encode
def test_encode_vs_oracle_pack():
    rng = np.random.default_rng(0)
    for n in (1, 31, 32, 33, 1000, 65_537, 1_000_003):
        s = _rand_seq(rng, n, pn=0.01, lower=0.2, junk=0.01)
        words, inval = P.mz_encode(_dev(s))
        ow, oi = O.pack(s)
        assert np.array_equal(words.cpu().numpy(), ow), n
        assert np.array_equal(inval.cpu().numpy(), oi), n


# ------------------------------------------------------------------ extraction
@pytest.mark.parametrize("path", [0, 1])
@pytest.mark.parametrize("k,w", [(15, 10), (19, 10), (1, 1), (2, 3), (3, 3), (5, 1), (8, 7), (12, 16), (16, 5),
                                 (17, 9), (21, 11), (25, 4), (26, 6), (31, 8), (15, 17), (11, 64), (19, 100)])
def test_random_vs_oracle(k, w, path):
    rng = np.random.default_rng(1000 * k + w + 7 * path)
    for n, pn in [(k + w - 2, 0), (k + w - 1, 0), (k + w, 0), (5000, 0.0), (40_000, 0.002), (123_457, 0.0005)]:
        s = _rand_seq(rng, n, pn=pn, lower=0.05)
        _same(s, k, w, path=path)
        if n >= 5000:
            _same(s, k, w, path=path, packed=True)
            _same(s, k, w, path=path, keymode=P.MZ_KEY_RAW)


@pytest.mark.parametrize("path", [0, 1])
@pytest.mark.parametrize("keymode", [P.MZ_KEY_CANON, P.MZ_KEY_CANON_RAW])
@pytest.mark.parametrize("k,w", [(15, 10), (19, 10), (1, 1), (2, 3), (4, 5), (8, 7), (16, 5), (17, 9), (26, 6),
                                 (31, 8), (11, 64)])
def test_canonical_vs_oracle(k, w, keymode, path):
    """Canonical (strand-symmetric) keys, NEXT f4 (R32), vs the oracle."""
    rng = np.random.default_rng(77 * k + w + path + keymode)
    for n, pn in [(k + w - 1, 0), (5000, 0.0), (60_000, 0.002)]:
        s = _rand_seq(rng, n, pn=pn, lower=0.05)
        _same(s, k, w, path=path, keymode=keymode)
        if n >= 5000:
            _same(s, k, w, path=path, keymode=keymode, packed=True)
    c4 = G.C4(nreads=60, tlen=1 << 20)
    ro = c4.read_off.astype(np.uint64)
    _same(c4.ascii_range(0, c4.n), k, w, path=path, keymode=keymode, read_off=ro)


@pytest.mark.parametrize("path", [0, 1])
def test_ties_small_alphabets(path):
    rng = np.random.default_rng(3)
    for alpha in (b"A", b"AC", b"ACG"):
        for k, w in [(3, 3), (4, 10), (15, 10), (2, 16), (6, 33)]:
            s = _rand_seq(rng, 30_000, alpha)
            _same(s, k, w, path=path, keymode=P.MZ_KEY_RAW)
            _same(s, k, w, path=path)


@pytest.mark.parametrize("path", [0, 1])
def test_repeats_tie_stress(path):
    # C3 recipe with homopolymer / di- / tri-nucleotide repeat runs (SURVEY.md 8(d) tie-stress)
    rng = np.random.default_rng(4)
    s = G.C3(n=300_000).ascii()
    for unit in (b"A", b"AC", b"CAG", b"T"):
        for _ in range(20):
            st = int(rng.integers(0, len(s) - 2000))
            L = int(rng.integers(10, 1500))
            rep = np.frombuffer(unit * (L // len(unit) + 1), np.uint8)[:L]
            s[st: st + L] = rep
    for k, w in [(15, 10), (19, 10), (5, 4)]:
        _same(s, k, w, path=path)


@pytest.mark.parametrize("path", [0, 1])
def test_segments_reads(path):
    rng = np.random.default_rng(5)
    n = 200_000
    s = _rand_seq(rng, n, pn=0.001)
    cuts = np.sort(rng.choice(np.arange(1, n), size=300, replace=False))
    # some very short reads (shorter than k+w-1) and some empty ones
    cuts = np.concatenate([cuts, cuts[:20] + 1, cuts[20:25]])
    ro = np.concatenate([[0], np.sort(cuts), [n]]).astype(np.uint64)
    for k, w in [(15, 10), (19, 10), (3, 2), (7, 20)]:
        _same(s, k, w, path=path, read_off=ro)


@pytest.mark.parametrize("lens", [(900, 1100), (60, 140), (8192, 8192), (20000, 40000)])
def test_read_start_density(lens):
    """Read-start handling of the fast kernel: ~31 starts per super-tile (the shared-memory
    list's capacity edge), very short reads (list overflow -> global search), reads starting
    exactly on the 8 kbp blocks of the coarse read index, and long reads; N-runs mixed in.
    Bit-exact vs the oracle, ASCII and packed input."""
    rng = np.random.default_rng(lens[0])
    n = 400_003
    s = _rand_seq(rng, n, pn=0.0005)
    lo, hi = lens
    ln = rng.integers(lo, hi + 1, size=n // lo + 2)
    st = np.concatenate([[0], np.cumsum(ln)])
    st = st[st < n]
    ro = np.concatenate([st, [n]]).astype(np.uint64)
    for k, w in [(15, 10), (19, 10)]:
        _same(s, k, w, read_off=ro)
        _same(s, k, w, read_off=ro, packed=True)


def test_c4_like_batch():
    c4 = G.C4(nreads=300)
    s = c4.ascii_range(0, c4.n)
    ro = c4.read_off.astype(np.uint64)
    _same(s, 15, 10, read_off=ro)
    _same(s, 15, 10, read_off=ro, packed=True)


@pytest.mark.parametrize("path", [0, 1])
def test_shards_and_pos_base(path):
    rng = np.random.default_rng(6)
    s = _rand_seq(rng, 100_000, pn=0.001)
    k, w = 15, 10
    full_k, full_p = O.mz(s, k, w)
    nwin = len(s) - (k + w - 1) + 1
    for Gn in (2, 3, 8):
        cuts = [nwin * g // Gn for g in range(Gn + 1)]
        cuts = [c - c % 32 for c in cuts[:-1]] + [nwin]
        parts_k, parts_p = [], []
        for g in range(Gn):
            a, b = cuts[g], cuts[g + 1]
            lo = max(0, a - 1)
            sub = s[lo: b + k + w - 2]
            hk, hp, cnt = gpu_mz(sub, k, w, path=path, pos_base=lo, win_lo=a - lo)
            parts_k.append(hk)
            parts_p.append(hp)
        assert np.array_equal(np.concatenate(parts_p), full_p)
        assert np.array_equal(np.concatenate(parts_k), full_k)


def test_window_range_and_capacity():
    rng = np.random.default_rng(7)
    s = _rand_seq(rng, 50_000)
    _same(s, 15, 10, win_lo=1000, win_hi=20_000)
    _same(s, 15, 10, win_lo=0, win_hi=0)
    wk, wp = O.mz(s, 15, 10)
    hk, hp, cnt = gpu_mz(s, 15, 10, capacity=100)
    assert cnt == len(wp) and np.array_equal(hp, wp[:100]) and np.array_equal(hk, wk[:100])
    with pytest.raises(P.SlsumError) as e:
        P.mz_extract(_dev(s), 15, 10, capacity=100, out_hash=torch.empty(100, dtype=torch.uint64, device="cuda"),
                     out_pos=torch.empty(100, dtype=torch.uint64, device="cuda"))
    assert e.value.rc == P.SLSUM_ECAPACITY


def test_degenerate_and_errors():
    assert gpu_mz("ACGT", 3, 3)[2] == 0
    assert gpu_mz("NNNNNNNNNNNNNNNNNNNNNNNNNNNNNNNNNNN", 3, 3)[2] == 0
    for k, w in [(0, 3), (32, 3), (3, 0)]:
        with pytest.raises(P.SlsumError):
            gpu_mz("ACGTACGTACGT", k, w)


def test_fig2_and_spec_examples():
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig2_minimizers.json")))
    hk, hp, cnt = gpu_mz(g["seq"], g["k"], g["w"], keymode=P.MZ_KEY_RAW)
    assert hp.tolist() == g["stored_positions"]
    ex = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
    for e in ex["minimizers_raw"]:
        hk, hp, cnt = gpu_mz(e["seq"], e["k"], e["w"], keymode=P.MZ_KEY_RAW)
        assert hp.tolist() == e["pos"]


def test_exhaustive_4_pow_8():
    L = 8
    allw = np.array(list(itertools.product(range(4), repeat=L)), np.uint8)
    seq = np.frombuffer(b"ACGT", np.uint8)[allw].reshape(-1).copy()
    ro = np.arange(0, len(seq) + 1, L, dtype=np.uint64)
    for k in (1, 2, 3):
        for w in (1, 2, 3, 4):
            for km in (P.MZ_KEY_RAW, P.MZ_KEY_HASH, P.MZ_KEY_CANON, P.MZ_KEY_CANON_RAW):
                for path in (0, 1):
                    _same(seq, k, w, read_off=ro, keymode=km, path=path)


def test_c1_full():
    s = G.c1_ascii(1_000_000)
    for path in (0, 1):
        _same(s, 15, 10, path=path)
        _same(s, 15, 10, path=path, packed=True)


def test_c3_full_size_sampled():
    """C3 at full size (3.1 Gbp, k=19, w=10) in the launch configuration bench.py times:
    sampled position ranges vs the oracle run on the matching sub-sequence (R25 halo rule)."""
    from synthgen import device as D
    k, w = 19, 10
    c3 = G.C3()
    seq = D.c3_ascii(c3)
    n = c3.n
    nwin = n - (k + w - 1) + 1
    cap = int(0.25 * nwin)
    h, p, c = P.mz_extract_ex(seq, k, w, capacity=cap)
    torch.cuda.synchronize()
    cnt = int(c.item())
    assert cnt <= cap
    dens = cnt / nwin
    assert 0.176 < dens < 0.186, dens
    p = p[:cnt].view(torch.int64)   # positions < 2^63: the int64 view orders them correctly
    h = h[:cnt]
    assert bool((p[1:] > p[:-1]).all())
    rng = np.random.default_rng(19)
    starts = [0, nwin - 50_000] + [int(x) for x in rng.integers(0, nwin - 50_000, size=12)]
    # include a range that straddles an N-run
    iv = c3.intervals[len(c3.intervals) // 2]
    starts.append(int(iv[0]) - 20_000)
    for a in starts:
        b = a + 50_000
        lo = max(0, a - 1)
        sub = c3.ascii(lo, b + k + w - 2 - lo)
        ok, op_ = O.mz(sub, k, w, pos_base=lo, win_lo=a - lo)
        sel = (op_ >= a + w - 1) & (op_ < b)
        lo_i = int(torch.searchsorted(p, torch.tensor([a + w - 1], dtype=torch.int64, device="cuda")).item())
        hi_i = int(torch.searchsorted(p, torch.tensor([b], dtype=torch.int64, device="cuda")).item())
        assert np.array_equal(p[lo_i:hi_i].cpu().numpy().astype(np.uint64), op_[sel]), a
        assert np.array_equal(h[lo_i:hi_i].cpu().numpy(), ok[sel]), a
