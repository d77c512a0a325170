"""The chunking that the full-size GPU parity tests (tests/test_gpu_fullsize.py) rely on, checked
on the oracle alone (CPU): per-chunk oracle runs with the R25 halo concatenate to the whole-input
minimizer list, and per-chunk oracle tables, placed bucket by bucket after the earlier chunks'
entries, reproduce the whole-input table slot for slot (Fig. 1 L63-65;
DESIGN.md R21, R25)."""
import numpy as np

import oracle as O
from synthgen import host as G
from _chunked import ordered, table_compare_chunk


def _whole_and_chunked(seq, k, w, bits, step, pos_base=0):
    key, pos = O.mz(seq, k, w, pos_base=pos_base)
    off, fp, tp = O.seedtable(key, pos, k, bits)
    n = len(seq)
    nwin = n - (k + w - 1) + 1
    chunks = [(a, min(nwin, a + step)) for a in range(0, nwin, step)]

    def gen(a, b):
        lo = max(0, a - 1)
        return seq[lo:b + k + w - 2]

    def orc(sub, a, b):
        lo = max(0, a - 1)
        kk, pp = O.mz(sub, k, w, pos_base=pos_base + lo, win_lo=a - lo, win_hi=b - lo, cap=16)
        return kk, pp, O.seedtable(kk, pp, k, bits)

    return key, pos, (off, fp, tp), chunks, gen, orc


def test_chunked_oracle_reproduces_whole_list_and_table():
    c3 = G.C3(n=2_000_000, mean_run=3_000.0, n_frac=0.03)
    seq = c3.ascii()
    for k, w, bits, step in ((19, 10, 16, 137_111), (15, 10, 12, 50_000), (5, 3, 10, 70_001)):
        key, pos, (off, fp, tp), chunks, gen, orc = _whole_and_chunked(seq, k, w, bits, step, pos_base=7)
        offh = off.view(np.int64)
        cursor = np.zeros(1 << bits, np.int64)
        cum = 0
        for (a, b), (kk, pp, tab) in ordered(chunks, gen, orc):
            assert np.array_equal(pp, pos[cum:cum + len(pp)]) and np.array_equal(kk, key[cum:cum + len(kk)])
            cum += len(pp)
            table_compare_chunk(tab, offh, cursor, lambda i: (tp[i], fp[i]), len(tp))
        assert cum == len(pos)
        assert np.array_equal(cursor, np.diff(offh))


def test_table_compare_detects_a_swapped_entry():
    c3 = G.C3(n=300_000, mean_run=3_000.0, n_frac=0.03)
    seq = c3.ascii()
    key, pos, (off, fp, tp), chunks, gen, orc = _whole_and_chunked(seq, 19, 10, 12, 40_000)
    bad = tp.copy()
    bad[[100, 101]] = bad[[101, 100]]
    offh = off.view(np.int64)
    cursor = np.zeros(1 << 12, np.int64)
    try:
        for _, (kk, pp, tab) in ordered(chunks, gen, orc):
            table_compare_chunk(tab, offh, cursor, lambda i: (bad[i], fp[i]), len(bad))
    except AssertionError:
        return
    raise AssertionError("a swapped table entry went undetected")
