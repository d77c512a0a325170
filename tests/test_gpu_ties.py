"""GPU parity: mz_extract_ties (minimap2-compatible minimizers, R35) vs
orc_mz_ties, through the C ABI.  Bit-exact: the count and every (hash, pos) record in order.
Inputs: small alphabets and homopolymer stretches (ties everywhere), N runs (short runs and the
end rule), reads, canonical even k (symmetric k-mers), sizes spanning several 8192-position
blocks with a ragged tail, ASCII and packed input, w from 1 to 300, and the degenerate cases."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1811_10074_b200")


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _gpu(seq, k, w, *, keymode=P.MZ_KEY_HASH, read_off=None, pos_base=0, packed=False, capacity=None,
         items=False):
    s = _dev(O.as_bytes(seq))
    ro = None if read_off is None else _dev(np.asarray(read_off, np.uint64))
    nk = max(0, s.numel() - k + 1)
    cap = nk if capacity is None else capacity
    it = torch.empty(max(1, cap), dtype=torch.uint64, device="cuda") if items else None
    if packed:
        words, inval = P.mz_encode(s)
        h, p, c = P.mz_extract_ties(words, k, w, n=s.numel(), kind=P.MZ_IN_PACKED2, invalid=inval, read_off=ro,
                                    pos_base=pos_base, keymode=keymode, capacity=cap, out_items=it)
    else:
        h, p, c = P.mz_extract_ties(s, k, w, read_off=ro, pos_base=pos_base, keymode=keymode, capacity=cap,
                                    out_items=it)
    torch.cuda.synchronize()
    cnt = int(c.item())
    m = min(cnt, cap)
    out = (h[:m].cpu().numpy(), p[:m].cpu().numpy(), cnt)
    return out + ((it[:m].cpu().numpy(),) if items else ())


def _seq(rng, n, alpha=b"ACGT", pn=0.0, nrun=0):
    s = np.frombuffer(alpha, np.uint8)[rng.integers(0, len(alpha), size=n)].copy()
    if pn:
        s[rng.random(n) < pn] = ord("N")
    for _ in range(nrun):
        a = int(rng.integers(0, n))
        s[a:a + int(rng.integers(1, 60))] = ord("N")
    return s


def _same(seq, k, w, **kw):
    wk, wp = O.mz_ties(seq, k, w, read_off=kw.get("read_off"), keymode=kw.get("keymode", O.KEY_HASH),
                       pos_base=kw.get("pos_base", 0))
    gk, gp, cnt = _gpu(seq, k, w, **kw)
    assert cnt == len(wp), (k, w, cnt, len(wp))
    assert np.array_equal(gp, wp), (k, w)
    assert np.array_equal(gk, wk), (k, w)


@pytest.mark.parametrize("k,w", [(1, 1), (2, 3), (3, 5), (5, 10), (8, 16), (15, 10), (16, 7), (19, 10), (21, 50),
                                 (31, 100), (12, 300)])
def test_random_with_n_runs(k, w):
    rng = np.random.default_rng(k * 1000 + w)
    _same(_seq(rng, 50_001, pn=0.002, nrun=20), k, w)


@pytest.mark.parametrize("keymode", [P.MZ_KEY_HASH, P.MZ_KEY_RAW, P.MZ_KEY_CANON, P.MZ_KEY_CANON_RAW])
@pytest.mark.parametrize("alpha", [b"AC", b"AAAC", b"ACGT"])
def test_ties_heavy_alphabets(keymode, alpha):
    rng = np.random.default_rng(len(alpha) * 10 + keymode)
    for k, w in [(2, 4), (4, 8), (6, 5), (10, 12)]:
        _same(_seq(rng, 30_017, alpha=alpha, pn=0.001), k, w, keymode=keymode)


def test_homopolymer_every_position():
    seq = b"A" * 20_000
    gk, gp, cnt = _gpu(seq, 5, 7, keymode=P.MZ_KEY_RAW)
    assert cnt == 20_000 - 4 and np.array_equal(gp, np.arange(cnt, dtype=np.uint64)) and not gk.any()


@pytest.mark.parametrize("packed", [False, True])
def test_reads_and_pos_base(packed):
    rng = np.random.default_rng(11)
    n = 40_000
    cuts = np.sort(rng.choice(np.arange(1, n), 300, replace=False))
    ro = np.concatenate([[0], cuts, [n]]).astype(np.uint64)  # many reads shorter than k + w - 1
    seq = _seq(rng, n, pn=0.003)
    for k, w in [(15, 10), (19, 10), (4, 30)]:
        _same(seq, k, w, read_off=ro, pos_base=123_456_789_000, packed=packed)


def test_short_sequences_and_degenerate():
    rng = np.random.default_rng(3)
    for n in [1, 2, 5, 18, 19, 20, 27, 28, 29, 40]:
        _same(_seq(rng, n), 19, 10)
        _same(_seq(rng, n, alpha=b"ACN"), 3, 4, keymode=P.MZ_KEY_RAW)
    _same(b"N" * 5000, 5, 3)
    _same(b"ACGTN" * 3000, 4, 10, keymode=P.MZ_KEY_CANON)        # every run is 1 k-mer long
    gk, gp, cnt = _gpu(b"ACG", 5, 3)
    assert cnt == 0


def test_capacity_overflow_and_items():
    rng = np.random.default_rng(5)
    seq = _seq(rng, 20_000)
    wk, wp = O.mz_ties(seq, 15, 10)
    gk, gp, cnt, it = _gpu(seq, 15, 10, capacity=100, items=True)
    assert cnt == len(wp) and len(gp) == 100
    assert np.array_equal(gp, wp[:100]) and np.array_equal(gk, wk[:100])
    want_it = ((wk[:100] << np.uint64(2)) << np.uint64(32)) | (wp[:100] & np.uint64(0xFFFFFFFF))
    assert np.array_equal(it, want_it)  # fp = key << (32 - 2k) for 2k < 32 (R21)


def test_c3_shape_sample_block_boundaries():
    """A 2 Mbp C1-shaped sample (synthgen: uniform ACGT) at k=19, w=10: 245 mark blocks, every record."""
    from synthgen import host as G
    _same(G.c1_ascii(2_000_000), 19, 10)


def test_rejects_shard_range_and_hist():
    s = _dev(np.frombuffer(b"ACGT" * 100, np.uint8))
    mi = P._lib.MzIn(P.MZ_IN_ASCII, s.data_ptr(), None, 400, None, 0, 0, 5, P.U64_MAX)
    h = torch.empty(400, dtype=torch.uint64, device="cuda")
    c = torch.zeros(1, dtype=torch.uint64, device="cuda")
    mo = P._lib.MzOut(h.data_ptr(), h.data_ptr(), 400, c.data_ptr(), None, None, 0)
    import ctypes
    assert P._lib._mz_extract_ties(ctypes.byref(mi), 5, 4, 0, ctypes.byref(mo), None, 0, None) == -2
    mi.win_lo = 0
    mo.hist = c.data_ptr()
    assert P._lib._mz_extract_ties(ctypes.byref(mi), 5, 4, 0, ctypes.byref(mo), None, 0, None) == -1
