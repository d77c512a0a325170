"""GPU parity: seedtable_lookup (Fig. 1 lookups; reading
DESIGN.md R30) vs the oracle's lookup.  Bit-exact CSR offsets and hit positions."""
import numpy as np
import pytest
import torch

import oracle as O
from synthgen import host as G

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1811_10074_b200")


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _gpu_lookup(key, pos, q, k, bits, **kw):
    off, po, fp = P.seedtable_build(_dev(key.astype(np.uint64)), _dev(pos.astype(np.uint64)), k, bits)
    ho, hp, tot = P.seedtable_lookup(_dev(q.astype(np.uint64)), k, bits, off, fp, po, **kw)
    torch.cuda.synchronize()
    t = int(tot.view(torch.int64).item())
    return ho.cpu().numpy(), hp.cpu().numpy(), t


@pytest.mark.parametrize("k,bits", [(15, 24), (19, 24), (12, 24), (8, 16), (3, 6), (31, 30)])
def test_random_vs_oracle(k, bits):
    rng = np.random.default_rng(k * 11 + bits)
    for m, nq in ((1, 1), (1000, 0), (5000, 3), (70_001, 10_007), (300_000, 100_001)):
        span = min(1 << (2 * k), max(64, m // 3))      # repeated seeds -> multi-hit queries
        key = rng.integers(0, span, size=m, dtype=np.uint64)
        if 2 * k > 32:   # wide keys: repeated top 32 bits (the fingerprint), random low bits
            lb = 2 * k - 32
            key = (key << np.uint64(lb)) | rng.integers(0, 1 << min(lb, 62), size=m, dtype=np.uint64)
        pos = np.sort(rng.choice(10 ** 9, size=m, replace=False)).astype(np.uint64)
        q = np.concatenate([key[rng.integers(0, m, size=nq // 2)],
                            rng.integers(0, 1 << (2 * k), size=nq - nq // 2, dtype=np.uint64)])
        wo, wf, wp = O.seedtable(key, pos, k, bits)
        ho_w, hp_w = O.lookup(q, k, bits, wo, wf, wp)
        ho, hp, t = _gpu_lookup(key, pos, q, k, bits)
        assert t == len(hp_w)
        assert np.array_equal(ho[: nq + 1], ho_w)
        assert np.array_equal(hp[:t], hp_w)


def test_spec_example():
    key, pos = O.mz(b"ACGTACGT", 3, 2, keymode=O.KEY_RAW)
    q = np.array([0b000110, 0b111100], np.uint64)         # ACG, TTA
    ho, hp, t = _gpu_lookup(key, pos, q, 3, 6)
    assert hp[int(ho[0]):int(ho[1])].tolist() == [0, 4]
    assert int(ho[2]) == int(ho[1]) == t == 2


def test_device_count_and_capacity():
    rng = np.random.default_rng(5)
    k, bits, m = 15, 20, 50_000
    key = rng.integers(0, 3000, size=m, dtype=np.uint64)
    pos = np.arange(m, dtype=np.uint64) * 7
    q = key[rng.integers(0, m, size=20_000)]
    wo, wf, wp = O.seedtable(key, pos, k, bits)
    ho_w, hp_w = O.lookup(q[:12_345], k, bits, wo, wf, wp)
    off, po, fp = P.seedtable_build(_dev(key), _dev(pos), k, bits)
    qt = _dev(q)
    dn = torch.tensor([12_345], dtype=torch.int64, device="cuda").view(torch.uint64)
    cap = len(hp_w) // 2
    ho, hp, tot = P.seedtable_lookup(qt, k, bits, off, fp, po, d_nq=dn, hit_cap=cap)
    torch.cuda.synchronize()
    assert int(tot.view(torch.int64).item()) == len(hp_w)
    assert np.array_equal(ho[:12_346].cpu().numpy(), ho_w)
    assert np.array_equal(hp[:cap].cpu().numpy(), hp_w[:cap])   # ordered prefix up to the capacity


def test_reads_against_template_end_to_end():
    """The f1 workload in miniature: table of a template's minimizers (k=15, w=10), queries =
    minimizers of noisy reads cut from it (C4 recipe); the GPU pipeline mz -> seed table ->
    mz(reads) -> lookup equals the oracle's, hit for hit."""
    k, w, bits = 15, 10, 24
    c4 = G.C4(nreads=400, tlen=1 << 22)
    tmpl = G.c1_ascii(1 << 22, seed=c4.seed_t)            # the template: uniform bases, stream seed_t
    reads = c4.ascii_range(0, c4.n)
    ro = c4.read_off.astype(np.uint64)
    tk, tp = O.mz(tmpl, k, w)
    rk, rp = O.mz(reads, k, w, read_off=ro)
    wo, wf, wp = O.seedtable(tk, tp, k, bits)
    ho_w, hp_w = O.lookup(rk, k, bits, wo, wf, wp)
    # GPU pipeline, every step through the library
    th, tpp, tc = P.mz_extract_ex(_dev(tmpl), k, w)
    rh, rpp, rc = P.mz_extract_ex(_dev(reads), k, w, read_off=_dev(ro))
    torch.cuda.synchronize()
    mt, mr = int(tc.item()), int(rc.item())
    off, po, fp = P.seedtable_build(th[:mt], tpp[:mt], k, bits)
    ho, hp, tot = P.seedtable_lookup(rh[:mr], k, bits, off, fp, po)
    torch.cuda.synchronize()
    assert mr == len(rk) and np.array_equal(rh[:mr].cpu().numpy(), rk)
    assert np.array_equal(ho.cpu().numpy(), ho_w)
    assert np.array_equal(hp[: len(hp_w)].cpu().numpy(), hp_w)
    assert int(tot.view(torch.int64).item()) > mr // 10    # reads do hit their template


@pytest.mark.parametrize("k,bits", [(15, 24), (19, 24), (15, 28), (8, 16)])
def test_sorted_lookup_large_batches(k, bits):
    """Batches of >= 2^20 queries take the sorted lookup (queries radix-sorted by bucket, then
    served in bucket order, results at their own index): the CSR equals the oracle's, with
    repeated queries, hitless ones and multi-hit seeds."""
    rng = np.random.default_rng(k * 7 + bits)
    m, nq = 400_000, (1 << 20) + 12_345
    span = min(1 << (2 * k), 150_000)
    key = rng.integers(0, span, size=m, dtype=np.uint64)
    if 2 * k > 32:
        lb = 2 * k - 32
        key = (key << np.uint64(lb)) | rng.integers(0, 1 << lb, size=m, dtype=np.uint64)
    pos = np.sort(rng.choice(10 ** 9, size=m, replace=False)).astype(np.uint64)
    q = np.concatenate([key[rng.integers(0, m, size=nq // 2)],
                        rng.integers(0, 1 << (2 * k), size=nq - nq // 2, dtype=np.uint64)])
    wo, wf, wp = O.seedtable(key, pos, k, bits)
    ho_w, hp_w = O.lookup(q, k, bits, wo, wf, wp)
    for kw in ({}, {"hit_cap": len(hp_w) // 2}):
        ho, hp, t = _gpu_lookup(key, pos, q, k, bits, **kw)
        assert t == len(hp_w)
        assert np.array_equal(ho[: nq + 1], ho_w)
        c = kw.get("hit_cap", t)
        assert np.array_equal(hp[:c], hp_w[:c])


@pytest.mark.parametrize("pos_hi", [0, 1 << 33])
def test_sorted_lookup_single_hit_positions(pos_hi):
    """The sorted lookup's count step carries a single-hit query's POSITION to the emit (read in
    bucket order); a position >= 2^32 does not fit the packed item, so such queries are counted
    again in query order and their position read there.  Hits equal the oracle's either way."""
    k, bits = 15, 24
    rng = np.random.default_rng(3 + pos_hi % 7)
    m, nq = 300_000, (1 << 20) + 99
    key = rng.integers(0, 1 << 30, size=m, dtype=np.uint64)          # mostly distinct: single hits
    key[: m // 10] = key[m // 10: 2 * (m // 10)]                     # and some doubles
    pos = np.sort(rng.choice(10 ** 9, size=m, replace=False)).astype(np.uint64) + np.uint64(pos_hi)
    q = np.concatenate([key[rng.integers(0, m, size=nq - 5000)], rng.integers(0, 1 << 30, size=5000, dtype=np.uint64)])
    wo, wf, wp = O.seedtable(key, pos, k, bits)
    ho_w, hp_w = O.lookup(q, k, bits, wo, wf, wp)
    ho, hp, t = _gpu_lookup(key, pos, q, k, bits)
    assert t == len(hp_w)
    assert np.array_equal(ho[: nq + 1], ho_w)
    assert np.array_equal(hp[:t], hp_w)


def test_sorted_lookup_multi_hit_side_overflow():
    """The sorted lookup's count step copies the positions of 2..14-hit queries to a side array
    of nq entries; here every query has ~10 hits, so the array fills after ~nq/10 queries and the
    rest are recounted and scanned in query order.  Hits equal the oracle's either way."""
    k, bits = 15, 24
    rng = np.random.default_rng(77)
    m, nq = 400_000, (1 << 20) + 3
    key = rng.integers(0, 40_000, size=m, dtype=np.uint64)      # each key ~10 times
    pos = np.sort(rng.choice(10 ** 9, size=m, replace=False)).astype(np.uint64)
    q = key[rng.integers(0, m, size=nq)]
    wo, wf, wp = O.seedtable(key, pos, k, bits)
    ho_w, hp_w = O.lookup(q, k, bits, wo, wf, wp)
    ho, hp, t = _gpu_lookup(key, pos, q, k, bits)
    assert t == len(hp_w)
    assert np.array_equal(ho[: nq + 1], ho_w)
    assert np.array_equal(hp[:t], hp_w)


@pytest.mark.parametrize("span", [1000, 20])
def test_sorted_lookup_heavy_repeats(span):
    """The sorted lookup's packed per-query result carries hit counts up to 14; queries with 15
    or more hits (here every key occurs ~400 or ~20000 times) are counted again in query order.
    The CSR still equals the oracle's (Fig. 1 lookups; R30)."""
    k, bits = 15, 24
    rng = np.random.default_rng(span)
    m, nq = 400_000, (1 << 20) + 7
    key = rng.integers(0, span, size=m, dtype=np.uint64)
    pos = np.sort(rng.choice(10 ** 9, size=m, replace=False)).astype(np.uint64)
    q = np.concatenate([key[rng.integers(0, m, size=nq - 1000)], rng.integers(0, 1 << 30, size=1000, dtype=np.uint64)])
    wo, wf, wp = O.seedtable(key, pos, k, bits)
    npre = 64 if span < 100 else 4096                      # the oracle on a prefix (the hits are many)
    ho_w, hp_w = O.lookup(q[:npre], k, bits, wo, wf, wp)
    ho, hp, t = _gpu_lookup(key, pos, q, k, bits, hit_cap=0)
    assert np.array_equal(ho[: npre + 1], ho_w)
    # every query's count, by the definition: the entries of the table whose key equals it
    cnt = np.bincount(key.astype(np.int64), minlength=span)
    qs = q.astype(np.int64)
    want = np.where(qs < span, cnt[np.minimum(qs, span - 1)], 0)
    assert np.array_equal(np.diff(ho[: nq + 1].astype(np.int64)), want)
