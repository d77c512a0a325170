"""GPU parity at BASELINE.json's full sizes, in exactly the launch configuration bench.py
times (encode -> PACKED2 + invalid bitmap -> mz_extract_ex with the device count ->
seedtable_build with d_m), checked on sampled outputs the oracle computes one by one and by
properties that hold at any size (R3, R21, R25).

C3: 3.1 Gbp, k=19, w=10, 2^24 buckets (configs[2] and [4]); C4: 1M reads, k=15, w=10
(configs[3]).  The oracle never sees a CUDA result: it is run on sub-sequences regenerated on
the host from the same seeded recipe."""
import numpy as np
import pytest
import torch

import oracle as O
from synthgen import host as G

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1811_10074_b200")


def _bench_path(seq, n, k, w, cap, read_off=None, items=None):
    """bench.py's step: mz_encode + mz_extract_ex(PACKED2, invalid bitmap, d_count[, items])."""
    nw = (n + 31) // 32
    words = torch.empty(nw + 1, dtype=torch.uint64, device="cuda")
    inval = torch.empty(nw + 1, dtype=torch.uint32, device="cuda")
    P.mz_encode(seq, words, inval)
    h, p, c = P.mz_extract_ex(words, k, w, n=n, kind=P.MZ_IN_PACKED2, invalid=inval, read_off=read_off,
                              capacity=cap, out_items=items)
    return words, inval, h, p, c


def _fp(key, k):
    b = 2 * k
    return (key >> np.uint64(b - 32)).astype(np.uint32) if b >= 32 else (key << np.uint64(32 - b)).astype(np.uint32)


def test_c3_bench_path_and_table_full_size_sampled():
    from synthgen import device as D
    k, w, bits = 19, 10, 24
    c3 = G.C3()
    n = c3.n
    seq = D.c3_ascii(c3)
    nwin = n - (k + w - 1) + 1
    cap = int(0.25 * nwin) + 1024            # bench.py's capacity rule
    items = torch.empty(cap, dtype=torch.uint64, device="cuda")
    _, _, h, p, c = _bench_path(seq, n, k, w, cap, items=items)
    del seq
    # seed table as bench.py builds it: from the packed items, capacity-sized inputs, device count
    offsets, pos_out, fp_out = P.seedtable_build_items(items, h, p, k, bits, m=cap, d_m=c)
    del items
    torch.cuda.synchronize()
    m = int(c.item())
    assert m <= cap and 0.176 < m / nwin < 0.186
    pi = p[:m].view(torch.int64)
    assert bool((pi[1:] > pi[:-1]).all())
    # ---- sampled minimizer ranges vs the oracle (R25 halo rule), incl. one across an N-run
    rng = np.random.default_rng(1903)
    starts = [0, nwin - 40_000] + [int(x) for x in rng.integers(0, nwin - 40_000, size=10)]
    iv = c3.intervals[len(c3.intervals) // 3]
    starts.append(int(iv[0]) - 15_000)
    samples = []
    for a in starts:
        b = a + 40_000
        lo = max(0, a - 1)
        sub = c3.ascii(lo, b + k + w - 2 - lo)
        ok, op_ = O.mz(sub, k, w, pos_base=lo, win_lo=a - lo)
        sel = (op_ >= a + w - 1) & (op_ < b)
        li = int(torch.searchsorted(pi, torch.tensor([a + w - 1], dtype=torch.int64, device="cuda")).item())
        hi = int(torch.searchsorted(pi, torch.tensor([b], dtype=torch.int64, device="cuda")).item())
        assert np.array_equal(pi[li:hi].cpu().numpy().astype(np.uint64), op_[sel]), a
        assert np.array_equal(h[li:hi].cpu().numpy(), ok[sel]), a
        samples.append((ok[sel], op_[sel]))
    # ---- table properties at full size
    off = offsets.view(torch.int64)
    assert int(off[0].item()) == 0 and int(off[-1].item()) == m
    assert bool((off[1:] >= off[:-1]).all())
    fpt = fp_out[:m].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    bucket = fpt >> (32 - bits)
    nz = torch.nonzero(off[1:] > off[:-1]).flatten()        # non-empty buckets
    expect_b = torch.repeat_interleave(nz, (off[1:] - off[:-1])[nz])
    assert torch.equal(bucket, expect_b)                      # every entry sits in its bucket
    pt = pos_out[:m].view(torch.int64)
    same_b = bucket[1:] == bucket[:-1]
    assert bool((pt[1:] > pt[:-1])[same_b].all())             # ascending positions inside a bucket
    # the table is a permutation of the (fp, pos) records
    order = torch.argsort(pt)
    assert torch.equal(pt[order], pi)
    assert torch.equal(fpt[order], (h[:m].view(torch.int64) >> (2 * k - 32)) & 0xFFFFFFFF)
    del order, same_b, expect_b
    # ---- the oracle's sampled records are found, exactly, in their oracle-computed buckets
    offn = off.cpu().numpy()
    for ok, op_ in samples:
        f = _fp(ok, k)
        for j in rng.integers(0, len(op_), size=min(200, len(op_))):
            bkt = int(f[j]) >> (32 - bits)
            sl = slice(int(offn[bkt]), int(offn[bkt + 1]))
            bp = pt[sl].cpu().numpy()
            i = int(np.searchsorted(bp, np.int64(op_[j])))
            assert i < len(bp) and bp[i] == np.int64(op_[j])
            assert int(fpt[sl][i].item()) == int(f[j])


def test_c4_bench_path_full_size_sampled():
    from synthgen import device as D
    k, w = 15, 10
    c4 = G.C4()
    n = c4.n
    seq = D.c4_ascii(c4)
    ro = torch.from_numpy(c4.read_off.astype(np.int64)).cuda().view(torch.uint64)
    cap = int(0.21 * n) + 1024               # bench.py --config c4 capacity rule
    _, _, h, p, c = _bench_path(seq, n, k, w, cap, read_off=ro)
    torch.cuda.synchronize()
    del seq
    m = int(c.item())
    assert m <= cap
    pi = p[:m].view(torch.int64)
    assert bool((pi[1:] > pi[:-1]).all())
    rng = np.random.default_rng(1904)
    reads = [0, c4.nreads - 1] + [int(r) for r in rng.integers(0, c4.nreads, size=40)]
    for r in reads:
        a, b = int(c4.read_off[r]), int(c4.read_off[r + 1])
        ok, op_ = O.mz(c4.read_ascii(r), k, w, pos_base=a)
        li = int(torch.searchsorted(pi, torch.tensor([a], dtype=torch.int64, device="cuda")).item())
        hi = int(torch.searchsorted(pi, torch.tensor([b], dtype=torch.int64, device="cuda")).item())
        assert np.array_equal(pi[li:hi].cpu().numpy().astype(np.uint64), op_), r
        assert np.array_equal(h[li:hi].cpu().numpy(), ok), r


@pytest.mark.parametrize("w", [16, 100, 1024])
def test_slsum_beyond_2_32_elements(w):
    """64-bit indexing of the sliding-sum kernels: n = 2^32 + 4099 u32 elements (16 GiB in,
    16 GiB out), GENERIC and COMMUTATIVE paths, outputs sampled around the 2^32 boundary and
    at the end vs the oracle on the same elements (regenerated on the host)."""
    from synthgen import device as D
    import paper_1811_10074_b200 as P
    n = (1 << 32) + 4099
    x = D.c2_u32(n)
    idx = np.array([0, (1 << 32) - w - 3, (1 << 32) - w + 1, (1 << 32) - 1, 1 << 32, n - w - 7, n - w], np.int64)
    it = torch.from_numpy(idx).cuda()
    for path in (P.SLSUM_PATH_GENERIC, P.SLSUM_PATH_COMMUTATIVE):
        y = P.slsum_run(P.SLSUM_MIN_U32, w, x, path=path)
        assert y.numel() == n - w + 1
        ys = y.view(torch.int32)[it].cpu().numpy().view(np.uint32)
        for j, i in enumerate(idx):
            assert ys[j] == O.slsum(O.MIN_U32, w, G.c2_u32(w, lo=int(i)))[0], (path, int(i))
        del y
    del x
    torch.cuda.empty_cache()
