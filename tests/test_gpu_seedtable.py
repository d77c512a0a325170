"""GPU parity: seedtable_build and the multi-GPU phases (count / partition / finalize) vs
the oracle's seed table (Fig. 1; bucketing DESIGN.md R21).  Bit-exact."""
import numpy as np
import pytest
import torch

import oracle as O
from synthgen import host as G

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1811_10074_b200")


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_table(key, pos, k, bits, use_dm=False):
    kt, pt = _dev(key.astype(np.uint64)), _dev(pos.astype(np.uint64))
    m = len(key)
    if use_dm:
        dm = torch.tensor([m], dtype=torch.int64, device="cuda").view(torch.uint64)
        # capacity larger than the count: the device count must win
        kt = _dev(np.concatenate([key.astype(np.uint64), np.zeros(17, np.uint64)]))
        pt = _dev(np.concatenate([pos.astype(np.uint64), np.zeros(17, np.uint64)]))
        off, po, fp = P.seedtable_build(kt, pt, k, bits, m=kt.numel(), d_m=dm)
    else:
        off, po, fp = P.seedtable_build(kt, pt, k, bits)
    torch.cuda.synchronize()
    return off.cpu().numpy(), po[:m].cpu().numpy(), fp[:m].cpu().numpy()


def _cmp(key, pos, k, bits, **kw):
    wo, wf, wp = O.seedtable(key, pos, k, bits)
    go, gp, gf = gpu_table(key, pos, k, bits, **kw)
    assert np.array_equal(go, wo)
    assert np.array_equal(gp, wp)
    assert np.array_equal(gf, wf)


@pytest.mark.parametrize("k,bits", [(15, 24), (19, 24), (15, 16), (19, 8), (15, 1), (4, 8), (12, 20), (31, 30)])
def test_random_keys(k, bits):
    rng = np.random.default_rng(k * 31 + bits)
    for m in (1, 7, 4095, 4096, 4097, 100_003):
        key = rng.integers(0, 1 << (2 * k), size=m, dtype=np.uint64)
        pos = np.sort(rng.choice(10 ** 10, size=m, replace=False)).astype(np.uint64)
        _cmp(key, pos, k, bits)


@pytest.mark.parametrize("k,bits", [(15, 24), (19, 24), (19, 16), (15, 8), (12, 20)])
def test_random_keys_narrow_span(k, bits):
    """Positions spanning < 2^32 take the packed-item (narrow) radix path."""
    rng = np.random.default_rng(k * 131 + bits)
    for m in (1, 2047, 2048, 4097, 131_071, 131_073, 300_001):
        key = rng.integers(0, 1 << (2 * k), size=m, dtype=np.uint64)
        base = int(rng.integers(0, 1 << 40))
        pos = (np.uint64(base) + np.sort(rng.choice(min(1 << 32, 50 * m), size=m, replace=False))).astype(np.uint64)
        _cmp(key, pos, k, bits)
        _cmp(key, pos, k, bits, use_dm=True)


@pytest.mark.parametrize("span", [(1 << 32) - 1, 1 << 32])
def test_span_boundary(span):
    """Largest narrow span (2^32 - 1) and the smallest wide one."""
    rng = np.random.default_rng(span & 0xffff)
    m = 50_000
    key = rng.integers(0, 1 << 38, size=m, dtype=np.uint64)
    mid = np.sort(rng.choice(span - 1, size=m - 2, replace=False) + 1)
    pos = np.concatenate([[0], mid, [span]]).astype(np.uint64) + np.uint64(7)
    _cmp(key, pos, 19, 24)


def test_unsorted_positions_fall_back():
    """pos[0] and pos[m-1] are close but an inner position is 2^33 away: the first narrow
    pass detects it and the wide path redoes the sort (stable = input order inside a bucket)."""
    rng = np.random.default_rng(5)
    m = 200_000
    key = rng.integers(0, 1 << 30, size=m, dtype=np.uint64)
    pos = np.arange(m, dtype=np.uint64) * 5
    pos[m // 2] = np.uint64(1 << 33)
    _cmp(key, pos, 15, 24)
    pos2 = pos.copy()
    pos2[m // 3] = np.uint64(0)          # below pos[0]: also outside [pos0, pos0 + 2^32)
    pos2[0] = np.uint64(10)
    pos2[m // 2] = np.uint64(m)
    _cmp(key, pos2, 15, 24)


def test_unaligned_inputs():
    """Inputs 8 B off a 16 B boundary cannot be TMA-staged; the kernels load them directly."""
    rng = np.random.default_rng(11)
    for m, span in ((70_001, 10 ** 6), (70_001, 10 ** 11)):
        key = rng.integers(0, 1 << 38, size=m, dtype=np.uint64)
        pos = np.sort(rng.choice(span, size=m, replace=False)).astype(np.uint64)
        kt = _dev(np.concatenate([np.zeros(1, np.uint64), key]))[1:]
        pt = _dev(np.concatenate([np.zeros(1, np.uint64), pos]))[1:]
        assert kt.data_ptr() % 16 == 8
        off, po, fp = P.seedtable_build(kt, pt, 19, 24)
        wo, wf, wp = O.seedtable(key, pos, 19, 24)
        assert np.array_equal(off.cpu().numpy(), wo)
        assert np.array_equal(po[:m].cpu().numpy(), wp)
        assert np.array_equal(fp[:m].cpu().numpy(), wf)


def test_heavy_buckets_and_device_count():
    rng = np.random.default_rng(1)
    m = 300_000
    key = np.where(rng.random(m) < 0.6, np.uint64(12345), rng.integers(0, 1 << 30, size=m, dtype=np.uint64))
    pos = np.arange(m, dtype=np.uint64) * 3
    _cmp(key, pos, 15, 24)
    _cmp(key, pos, 15, 24, use_dm=True)
    _cmp(np.full(10_000, 7, np.uint64), np.arange(10_000, dtype=np.uint64), 15, 24)


def test_empty():
    off, po, fp = P.seedtable_build(torch.zeros(1, dtype=torch.uint64, device="cuda"),
                                    torch.zeros(1, dtype=torch.uint64, device="cuda"), 15, 12, m=0)
    assert int(off.view(torch.int64).abs().sum().item()) == 0


def test_c1_minimizers_table():
    s = G.c1_ascii(1_000_000)
    key, pos = O.mz(s, 15, 10)
    _cmp(key, pos, 15, 24)
    _cmp(key, pos, 15, 16)


@pytest.mark.parametrize("nranks", [1, 2, 4, 8])
def test_multi_rank_phases_emulated(nranks):
    """The C5 exchange with the NCCL collectives replaced by in-process slicing: ranks own
    contiguous shards of the minimizer list; count -> (sum) -> partition -> (all_to_all)
    -> finalize; the concatenated slices must equal the single-table oracle."""
    k, bits = 19, 24
    c3 = G.C3(n=3_000_000)
    key, pos = O.mz(c3.ascii(), k, 19 - 9)
    m = len(key)
    cuts = [m * g // nranks for g in range(nranks + 1)]
    counts = None
    sends = []
    for g in range(nranks):
        kt, pt = _dev(key[cuts[g]:cuts[g + 1]]), _dev(pos[cuts[g]:cuts[g + 1]])
        c = P.seedtable_count(kt, k, bits).view(torch.int32).to(torch.int64)
        counts = c if counts is None else counts + c
        sends.append(P.seedtable_partition(kt, pt, k, bits, nranks))
    gcounts = counts.to(torch.int32).view(torch.uint32)
    wo, wf, wp = O.seedtable(key, pos, k, bits)
    nbl = (1 << bits) // nranks
    all_off, all_pos, all_fp, base = [], [], [], 0
    for r in range(nranks):
        fps, poss = [], []
        for g in range(nranks):
            sf, sp, sc = sends[g]
            sc = sc.cpu().numpy().astype(np.int64)
            o = int(sc[:r].sum())
            fps.append(sf[o:o + sc[r]])
            poss.append(sp[o:o + sc[r]])
        rf = torch.cat([f.view(torch.int32) for f in fps]).view(torch.uint32)
        rp = torch.cat([q.view(torch.int64) for q in poss]).view(torch.uint64)
        mr = rf.numel()
        for gc in (gcounts, None):
            off, po, fp = P.seedtable_finalize(rf, rp, mr, gc, bits, r, nranks)
            offn = off.cpu().numpy()
            assert np.array_equal(offn + np.uint64(base), wo[r * nbl: (r + 1) * nbl + 1])
        all_pos.append(po[:mr].cpu().numpy())
        all_fp.append(fp[:mr].cpu().numpy())
        base += mr
    assert np.array_equal(np.concatenate(all_pos), wp)
    assert np.array_equal(np.concatenate(all_fp), wf)


@pytest.mark.parametrize("nranks,items,pos_base", [(2, False, 0), (4, False, 0), (8, False, 0), (2, True, 0),
                                                   (8, True, (1 << 32) - 1_000_000)])
def test_partition_p2p_emulated(nranks, items, pos_base):
    """The partition fused with the all-to-all (seedtable_partition_p2p, and _items from the
    packed items), with the ranks emulated in one process on one GPU: every sender writes
    straight into all owners' receive buffers (here plain device buffers; peer-mapped symmetric
    memory on a real box) at its base offsets; each owner then finalizes.  The concatenated
    slices must equal the oracle table (also across a multiple of 2^32 in the positions)."""
    k, bits = 19, 24
    c3 = G.C3(n=3_000_000)
    key, pos = O.mz(c3.ascii(), k, 10, pos_base=pos_base)
    m = len(key)
    cuts = [m * g // nranks for g in range(nranks + 1)]
    nbl = (1 << bits) // nranks
    shards, per_owner, gcounts = [], [], None
    for g in range(nranks):
        kt, pt = _dev(key[cuts[g]:cuts[g + 1]]), _dev(pos[cuts[g]:cuts[g + 1]])
        c = P.seedtable_count(kt, k, bits).view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        gcounts = c if gcounts is None else gcounts + c
        per_owner.append(c.view(nranks, nbl).sum(1).cpu().numpy())
        shards.append((kt, pt))
    cnt = np.stack(per_owner)                       # [sender, owner]
    recv = cnt.sum(0)
    bufs = [(torch.empty(max(1, int(recv[o])), dtype=torch.uint32, device="cuda"),
             torch.empty(max(1, int(recv[o])), dtype=torch.uint64, device="cuda")) for o in range(nranks)]
    for g, (kt, pt) in enumerate(shards):
        base = [int(cnt[:g, o].sum()) for o in range(nranks)]
        it = None
        if items:   # items as mz_extract_ex writes them: fp << 32 | pos mod 2^32 (from the oracle's records)
            kn, pn = key[cuts[g]:cuts[g + 1]], pos[cuts[g]:cuts[g + 1]]
            it = _dev((_fp_np(kn, k) << np.uint64(32)) | (pn & np.uint64(0xFFFFFFFF)))
        rc = P.seedtable_partition_p2p(kt, pt, k, bits, [b[0].data_ptr() for b in bufs],
                                       [b[1].data_ptr() for b in bufs], base, items=it)
        assert rc == P.SLSUM_OK
    torch.cuda.synchronize()
    gc32 = gcounts.to(torch.int32).view(torch.uint32)
    wo, wf, wp = O.seedtable(key, pos, k, bits)
    all_pos, all_fp, b0 = [], [], 0
    for r in range(nranks):
        mr = int(recv[r])
        off, po, fp = P.seedtable_finalize(bufs[r][0], bufs[r][1], mr, gc32, bits, r, nranks)
        assert np.array_equal(off.cpu().numpy() + np.uint64(b0), wo[r * nbl: (r + 1) * nbl + 1])
        all_pos.append(po[:mr].cpu().numpy())
        all_fp.append(fp[:mr].cpu().numpy())
        b0 += mr
    assert np.array_equal(np.concatenate(all_pos), wp)
    assert np.array_equal(np.concatenate(all_fp), wf)


def test_partition_p2p_rejects_wide_spans():
    kt = _dev(np.arange(100, dtype=np.uint64))
    pt = _dev((np.arange(100, dtype=np.uint64) * np.uint64(10 ** 9)))    # spans > 2^32
    b = torch.empty(100, dtype=torch.uint64, device="cuda")
    rc = P.seedtable_partition_p2p(kt, pt, 19, 24, [b.data_ptr()] * 2, [b.data_ptr()] * 2, [0, 0])
    assert rc == P.SLSUM_EUNSUPPORTED


def _fp_np(h, k):
    b = 2 * k
    h = h.astype(np.uint64)
    return (h >> np.uint64(b - 32)) if b >= 32 else (h << np.uint64(32 - b)) & np.uint64(0xFFFFFFFF)


@pytest.mark.parametrize("k,pos_base,path", [(19, 0, 0), (15, 0, 0), (19, (1 << 32) - 300_000, 0),
                                             (15, (1 << 33) + 5, 1), (22, 7, 0)])
def test_items_path_vs_oracle(k, pos_base, path):
    """mz_extract_ex's packed items (fp << 32 | pos mod 2^32) and seedtable_build_items: the
    items match their definition, and the table built from them equals the oracle's and
    seedtable_build's -- also when the positions cross a multiple of 2^32."""
    w, bits = 10, 24
    seq = G.C3(n=700_000).ascii(0, 600_000)
    st = torch.from_numpy(seq).cuda()
    cap = 200_000
    items = torch.empty(cap, dtype=torch.uint64, device="cuda")
    h, p, c = P.mz_extract_ex(st, k, w, pos_base=pos_base, capacity=cap, out_items=items, path=path)
    torch.cuda.synchronize()
    m = int(c.view(torch.int64).item())
    hk, pp = h[:m].cpu().numpy(), p[:m].cpu().numpy()
    it = items[:m].cpu().numpy()
    want_it = (_fp_np(hk, k) << np.uint64(32)) | (pp & np.uint64(0xFFFFFFFF))
    assert np.array_equal(it, want_it)
    wk, wp = O.mz(seq, k, w, pos_base=pos_base)
    assert np.array_equal(hk, wk) and np.array_equal(pp, wp)
    wo, wf, wpos = O.seedtable(wk, wp, k, bits)
    for d_m in (None, c):
        off, po, fp = P.seedtable_build_items(items, h, p, k, bits, m=(m if d_m is None else cap), d_m=d_m)
        torch.cuda.synchronize()
        assert np.array_equal(off.cpu().numpy(), wo)
        assert np.array_equal(po[:m].cpu().numpy(), wpos)
        assert np.array_equal(fp[:m].cpu().numpy(), wf)
        # the 32-bit position table: the same entries, positions mod 2^32
        off32, po32, fp32 = P.seedtable_build_items32(items, h, p, k, bits, m=(m if d_m is None else cap), d_m=d_m)
        torch.cuda.synchronize()
        assert np.array_equal(off32.cpu().numpy(), wo)
        assert np.array_equal(po32[:m].cpu().numpy(), (wpos & np.uint64(0xFFFFFFFF)).astype(np.uint32))
        assert np.array_equal(fp32[:m].cpu().numpy(), wf)


def _items_of(key, pos, k):
    return _dev((_fp_np(key, k) << np.uint64(32)) | (pos & np.uint64(0xFFFFFFFF)))


def _cmp_items(key, pos, k, bits, cap_extra=0):
    """seedtable_build_items / _items32 (and with a device count below the capacity) vs the oracle"""
    m = len(key)
    wo, wf, wpos = O.seedtable(key, pos, k, bits)
    kpad = np.concatenate([key, np.zeros(cap_extra, np.uint64)])
    ppad = np.concatenate([pos, np.full(cap_extra, pos[-1] if m else 0, np.uint64)])
    it, kt, pt = _items_of(kpad, ppad, k), _dev(kpad), _dev(ppad)
    dm = torch.tensor([m], dtype=torch.int64, device="cuda").view(torch.uint64) if cap_extra else None
    off, po, fp = P.seedtable_build_items(it, kt, pt, k, bits, m=m + cap_extra, d_m=dm)
    torch.cuda.synchronize()
    assert np.array_equal(off.cpu().numpy(), wo)
    assert np.array_equal(po[:m].cpu().numpy(), wpos)
    assert np.array_equal(fp[:m].cpu().numpy(), wf)
    off32, po32, fp32 = P.seedtable_build_items32(it, kt, pt, k, bits, m=m + cap_extra, d_m=dm)
    torch.cuda.synchronize()
    assert np.array_equal(off32.cpu().numpy(), wo)
    assert np.array_equal(po32[:m].cpu().numpy(), (wpos & np.uint64(0xFFFFFFFF)).astype(np.uint32))
    assert np.array_equal(fp32[:m].cpu().numpy(), wf)


@pytest.mark.parametrize("bits", [9, 12, 16, 17, 20, 23, 24])
def test_items_bit_widths(bits):
    """The packed-item path at 9..24 bucket bits (2 or 3 radix passes, a last digit of 1..8 bits):
    random keys, heavy repeats, and a device count below the capacity."""
    rng = np.random.default_rng(bits)
    k = 19
    m = 120_000
    key = rng.integers(0, 1 << 38, size=m, dtype=np.uint64)
    pos = np.cumsum(rng.integers(1, 40, size=m, dtype=np.uint64)) + np.uint64(1000)
    _cmp_items(key, pos, k, bits)
    heavy = np.where(rng.random(m) < 0.3, np.uint64(0x12345678), key)   # one bucket of ~36k entries
    _cmp_items(heavy, pos, k, bits, cap_extra=13)


def test_items_clustered_prefixes():
    """Runs of 4095, 4096, 4097, 8192 and 12289 entries sharing the top 16 bits of the key (a
    downsweep tile holds 4096 items) among random keys, and one bucket holding every entry; k=16
    so the fingerprint is the key (bits = 24)."""
    rng = np.random.default_rng(5)
    k, bits = 16, 24
    parts = [rng.integers(0, 1 << 32, size=20_000, dtype=np.uint64)]
    for pre, n in ((5, 4096), (9, 4097), (0xABCD, 8192), (0xFFFF, 12289), (0x8000, 4095)):
        parts.append((np.uint64(pre) << np.uint64(16)) | rng.integers(0, 1 << 16, size=n, dtype=np.uint64))
    key = np.concatenate(parts)
    key = key[rng.permutation(len(key))]
    pos = np.arange(len(key), dtype=np.uint64) * np.uint64(3)
    _cmp_items(key, pos, k, bits)
    # every entry of one bucket (one segment, one local digit)
    _cmp_items(np.full(9000, 0xABCDEF12, np.uint64), np.arange(9000, dtype=np.uint64), k, bits)


@pytest.mark.parametrize("npass_bits", [12, 16, 24, 30])
def test_items32_wide_spans_and_bit_widths(npass_bits):
    """seedtable_build_items32 when the positions span >= 2^32 (the wide path, narrowed to u32
    afterwards) and for 1, 2, 3 and 4 radix passes (the u64 scratch of the wide path's last pass
    is a separate buffer unless there are exactly 3 passes)."""
    k = 19
    rng = np.random.default_rng(npass_bits)
    m = 50_000
    key = rng.integers(0, 1 << 38, size=m, dtype=np.uint64)
    for step in (7, 200_003):                       # narrow span, then a span >= 2^32 (wide path)
        pos = (np.arange(m, dtype=np.uint64) * np.uint64(step) + np.uint64(12345))
        fpk = _fp_np(key, k)
        items = _dev((fpk << np.uint64(32)) | (pos & np.uint64(0xFFFFFFFF)))
        wo, wf, wpos = O.seedtable(key, pos, k, npass_bits)
        off, po, fp = P.seedtable_build_items32(items, _dev(key), _dev(pos), k, npass_bits)
        torch.cuda.synchronize()
        assert np.array_equal(off.cpu().numpy(), wo), step
        assert np.array_equal(po.cpu().numpy(), (wpos & np.uint64(0xFFFFFFFF)).astype(np.uint32)), step
        assert np.array_equal(fp.cpu().numpy(), wf), step


def _hist_oracle(wk, k, bits, cap):
    """The first radix pass's digit counts, from the ORACLE records: chunks of the radix chunk
    size for m = cap (at most 131072 entries, at least 4096, ~cap/296 rounded up to 4096
    between), digit = the low min(8, bits) bits of the bucket fp >> (32 - bits)."""
    want = (cap + 295) // 296
    chunk = min(131072, max(4096, (want + 4095) // 4096 * 4096))
    nch = (cap + chunk - 1) // chunk
    d = (_fp_np(wk, k) >> np.uint64(32 - bits)) & np.uint64((1 << min(8, bits)) - 1)
    c = np.arange(len(wk), dtype=np.uint64) // np.uint64(chunk)
    h = np.zeros((256, nch), dtype=np.int64)
    np.add.at(h, (d.astype(np.int64), c.astype(np.int64)), 1)
    return h.reshape(-1), nch


@pytest.mark.parametrize("k,bits,cap,path", [(19, 24, 200_000, 0), (19, 24, 40_000_000, 0), (15, 24, 40_000_000, 0),
                                             (15, 6, 150_000, 0), (19, 24, 150_000, 1), (19, 16, 40_000_000, 1),
                                             (19, 24, 60_000, 0)])
def test_fused_first_pass_histogram(k, bits, cap, path):
    """mz_extract_ex's fused first-pass histogram (mz_out.hist) equals the digit counts of the
    oracle's records per radix chunk, and seedtable_build_items_ex started from it equals the
    oracle table (Fig. 1).  cap = 40e6 takes 131072-entry chunks (a super-tile's
    records touch <= 2 chunks: the shared-memory path); cap = 200k / 150k takes 4096-entry chunks
    (records past the second chunk: the global-atomic path); cap = 60k < the count: only the
    first cap records are counted.  path 1: the generic kernel."""
    w = 10
    seq = G.C3(n=700_000).ascii(0, 600_000)
    st = torch.from_numpy(seq).cuda()
    items = torch.empty(cap, dtype=torch.uint64, device="cuda")
    hist = torch.full((P.seedtable_hist_words(cap, bits),), 0xDEAD, dtype=torch.uint32, device="cuda")
    h, p, c = P.mz_extract_ex(st, k, w, capacity=cap, out_items=items, out_hist=hist, hist_bits=bits, path=path)
    torch.cuda.synchronize()
    m = int(c.view(torch.int64).item())
    wk, wp = O.mz(seq, k, w)
    assert m == len(wk)
    mw = min(m, cap)
    want_h, nch = _hist_oracle(wk[:mw], k, bits, cap)
    assert hist.numel() == 256 * nch
    assert np.array_equal(hist.cpu().numpy().astype(np.int64), want_h)
    if m > cap:
        return
    wo, wf, wpos = O.seedtable(wk, wp, k, bits)
    for pos32 in (False, True):
        off, po, fp = P.seedtable_build_items_ex(items, h, p, k, bits, m=cap, d_m=c, hist=hist, pos32=pos32)
        torch.cuda.synchronize()
        assert np.array_equal(off.cpu().numpy(), wo)
        assert np.array_equal(fp[:m].cpu().numpy(), wf)
        gp = po[:m].cpu().numpy()
        assert np.array_equal(gp, (wpos & np.uint64(0xFFFFFFFF)).astype(np.uint32) if pos32 else wpos)
