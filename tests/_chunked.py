"""Chunked oracle runs for the full-size parity tests (test infrastructure).

The oracle (`oracle/`) is run over consecutive chunks of a full-size workload, each chunk's
input regenerated on the host from the seeded recipe (`synthgen.host`), so no oracle input
ever comes from the device.  Input generation runs on a small thread pool (numpy releases the
GIL), the oracle calls run one at a time on a single worker (each one uses every core through
OpenMP), and the caller compares chunk i while the oracle computes chunk i+1.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np


def par_concat(fn, lo: int, hi: int, pieces: int, pool: ThreadPoolExecutor) -> np.ndarray:
    """fn(a, b) over `pieces` sub-ranges of [lo, hi) on `pool`, concatenated in order."""
    cuts = np.linspace(lo, hi, pieces + 1).astype(np.int64)
    futs = [pool.submit(fn, int(a), int(b)) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
    parts = [f.result() for f in futs]
    return parts[0] if len(parts) == 1 else np.concatenate(parts)


def ordered(chunks, gen, orc, ahead: int = 3, gen_threads: int | None = None):
    """Yield (chunk, orc(gen(*chunk), *chunk)) in chunk order, pipelined."""
    gen_threads = gen_threads or max(2, min(8, (os.cpu_count() or 4) // 2))
    with ThreadPoolExecutor(gen_threads) as gp, ThreadPoolExecutor(1) as op:
        gf = {}

        def sched(i):
            if i < len(chunks) and i not in gf:
                gf[i] = gp.submit(gen, *chunks[i])

        for i in range(ahead):
            sched(i)
        of = {}
        for i in range(len(chunks)):
            sched(i + ahead)
            f = gf[i]
            of[i] = op.submit(lambda f=f, c=chunks[i]: orc(f.result(), *c))
            if i >= 1:
                yield chunks[i - 1], of.pop(i - 1).result()
                gf.pop(i - 1, None)
        if chunks:
            yield chunks[-1], of.pop(len(chunks) - 1).result()


def table_compare_chunk(tab, offh: np.ndarray, cursor: np.ndarray, gather, m: int) -> None:
    """Check one chunk's oracle table (the chunk's records bucketed in input order, Fig. 1)
    against a whole-input table given by its offsets `offh` and `gather(idx) -> (pos, fp)`.

    Chunks come in position order, so inside bucket b this chunk's entries sit right after the
    earlier chunks' entries: at offh[b] + cursor[b] + j.  `offh` only indexes the gather; the
    caller checks at the end that cursor equals np.diff(offh) and offh[0] == 0, which makes every
    slot of the table compared exactly once (and the offsets equal to the oracle's)."""
    coff, cfp, cpos = tab
    co = coff.view(np.int64)
    cnt_b = np.diff(co)
    mc = len(cpos)
    if mc:
        bk = np.repeat(np.arange(len(cnt_b), dtype=np.int64), cnt_b)
        idx = offh[bk] + cursor[bk] + (np.arange(mc, dtype=np.int64) - co[bk])
        np.clip(idx, 0, max(0, m - 1), out=idx)   # a wrong offset fails the comparison, not the gather
        gp, gf = gather(idx)
        assert np.array_equal(gp, cpos), "seed-table positions differ"
        assert np.array_equal(gf, cfp), "seed-table fingerprints differ"
    cursor += cnt_b
