"""Seeded synthetic inputs, host side (numpy).

This module is the ONLY code shared by the oracle (`oracle/`) and the CUDA path
(`paper_1811_10074_b200/`).  It holds none of the method's arithmetic: no
k-mer codes, no hash, no window minimum, no seed table.  It only draws bases
and numbers.

Every draw is counter-based: value number `i` of a stream is
``mix64(seed, i)`` (the SplitMix64 output function applied to
``seed + (i+1)*0x9E3779B97F4A7C15``).  Any sub-range of any stream can
therefore be generated independently -- the oracle can regenerate the bases of
a sample window of a 3.1 Gbp input without generating the other 3.1e9 bases,
and `synthgen/csrc/synthgen.cu` produces bit-identical bytes on the device
(checked by `tests/test_gpu_synthgen.py`).

Recipes (DESIGN.md "Input recipe" restates them with the config they serve):

* uniform DNA (C1, C4 template): code_i = mix64(seed, i) >> 62 (A,C,G,T = 0..3).
* GC-41% DNA (C3): u = mix64(seed, i) >> 32; A if u < T_A, C if u < T_C,
  G if u < T_G, else T, with T_A = 0x4B851EB8 (0.295), T_C = 0x80000000
  (0.5), T_G = 0xB47AE148 (0.705).
* N-runs (C3): an alternating renewal process, gap ~ Geom(mean 990,000),
  N run ~ Geom(mean 10,000), starting with a gap; draw j uses
  U_j = ((mix64(seed, j) >> 11) + 1) * 2^-53 in (0, 1] and
  L = 1 + floor(ln U / ln(1 - 1/mean)).  Expected N fraction 1 %.
* long reads (C4): length L_r = max(1, round(exp(mu + sigma*z_r))),
  mu = 8.96299, sigma = 0.70335 (lognormal mean 10 kbp, sd 8 kbp),
  z_r by Box-Muller from draws 2r, 2r+1; start_r = floor(U_r * (2^30 - L_r + 1));
  base t of read r = template[start_r + t], substituted when
  (mix64(seed_sub, g) >> 32) < 429,496,730 (10 %) by
  (b + 1 + (mix64(seed_sub, g) & 0xffffffff) % 3) & 3, g = global base index.
* C2 u32: element i = 32-bit half (i & 1) of mix64(seed, i >> 1) (little-endian
  view of a u64 stream).
* C2 f32: element i = TABLE[mix64(seed, i) >> 48], TABLE[j] = float32(Phi^-1((j + 0.5) / 65536)):
  a 65,536-level inverse-CDF N(0, 1) sample that host and device reproduce exactly.
"""
from __future__ import annotations

import math

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

# stream seeds (one per config stream)
SEED_C1 = 1811
SEED_C2_U32 = 1812
SEED_C2_F32 = 1813
SEED_C3_BASES = 1814
SEED_C3_NRUNS = 1815
SEED_C4_TEMPLATE = 1816
SEED_C4_LENGTHS = 1817
SEED_C4_STARTS = 1818
SEED_C4_SUBST = 1819

GC41_THRESHOLDS = (0x4B851EB8, 0x80000000, 0xB47AE148)
C4_MU = 8.96299
C4_SIGMA = 0.70335
C4_TEMPLATE_LEN = 1 << 30
C4_SUBST_T = 429_496_730
ACGT = np.frombuffer(b"ACGT", dtype=np.uint8)


def mix64(seed: int, idx) -> np.ndarray:
    """SplitMix64 output of counter `idx` (uint64 array) in stream `seed`."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (idx + np.uint64(1)) * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        return z ^ (z >> np.uint64(31))


def _arange(lo: int, n: int) -> np.ndarray:
    return np.arange(lo, lo + n, dtype=np.uint64)


# --------------------------------------------------------------------------
# DNA bases
# --------------------------------------------------------------------------
def uniform_codes(seed: int, lo: int, n: int) -> np.ndarray:
    """Codes 0..3 of bases [lo, lo+n) of an iid uniform A/C/G/T stream."""
    return (mix64(seed, _arange(lo, n)) >> np.uint64(62)).astype(np.uint8)


def gc_codes(seed: int, lo: int, n: int, thresholds=GC41_THRESHOLDS) -> np.ndarray:
    """Codes of bases [lo, lo+n) of an iid stream with the given cumulative thresholds."""
    u = (mix64(seed, _arange(lo, n)) >> np.uint64(32)).astype(np.uint32)
    ta, tc, tg = (np.uint32(t) for t in thresholds)
    return ((u >= ta).astype(np.uint8) + (u >= tc).astype(np.uint8) + (u >= tg).astype(np.uint8))


def codes_to_ascii(codes: np.ndarray) -> np.ndarray:
    return ACGT[codes]


def geometric_draws(seed: int, lo: int, n: int, mean: float) -> np.ndarray:
    """Draws lo..lo+n-1 of Geom(p = 1/mean) on {1, 2, ...} by inverse CDF."""
    r = mix64(seed, _arange(lo, n))
    u = ((r >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)
    p = 1.0 / mean
    return (1 + np.floor(np.log(u) / math.log1p(-p))).astype(np.int64)


def nrun_intervals(seed: int, n: int, n_frac: float = 0.01, mean_run: float = 10_000.0) -> np.ndarray:
    """Sorted disjoint N-run intervals [s, e) over [0, n), as an int64 array of shape (m, 2)."""
    mean_gap = mean_run * (1.0 - n_frac) / n_frac
    out = []
    pos = 0
    j = 0
    batch = 4096
    while pos < n:
        # draw 2j is the gap, draw 2j+1 the N-run of renewal cycle j
        r = mix64(seed, _arange(2 * j, 2 * batch))
        u = ((r >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)
        g = (1 + np.floor(np.log(u[0::2]) / math.log1p(-1.0 / mean_gap))).astype(np.int64)
        l = (1 + np.floor(np.log(u[1::2]) / math.log1p(-1.0 / mean_run))).astype(np.int64)
        for gi, li in zip(g.tolist(), l.tolist()):
            pos += gi
            if pos >= n:
                break
            e = min(n, pos + li)
            out.append((pos, e))
            pos = e
            if pos >= n:
                break
        j += batch
    return np.asarray(out, dtype=np.int64).reshape(-1, 2)


def invalid_mask_from_intervals(lo: int, n: int, iv: np.ndarray) -> np.ndarray:
    """Boolean mask of bases [lo, lo+n) that fall inside any interval of `iv`."""
    m = np.zeros(n, dtype=bool)
    if len(iv):
        sel = (iv[:, 1] > lo) & (iv[:, 0] < lo + n)
        for s, e in iv[sel].tolist():
            m[max(s, lo) - lo: min(e, lo + n) - lo] = True
    return m


def c1_ascii(n: int = 1_000_000, seed: int = SEED_C1, lo: int = 0) -> np.ndarray:
    """C1: iid uniform ACGT, bases [lo, lo+n)."""
    return codes_to_ascii(uniform_codes(seed, lo, n))


class C3:
    """C3: human-genome-shaped sequence of `n` bases (GC 41 %, 1 % N in runs)."""

    def __init__(self, n: int = 3_100_000_000, seed_bases: int = SEED_C3_BASES,
                 seed_nruns: int = SEED_C3_NRUNS, n_frac: float = 0.01, mean_run: float = 10_000.0):
        self.n = n
        self.seed_bases = seed_bases
        self.intervals = nrun_intervals(seed_nruns, n, n_frac, mean_run)

    def ascii(self, lo: int = 0, n: int | None = None) -> np.ndarray:
        if n is None:
            n = self.n - lo
        a = codes_to_ascii(gc_codes(self.seed_bases, lo, n))
        a[invalid_mask_from_intervals(lo, n, self.intervals)] = ord("N")
        return a


class C4:
    """C4: a long-read batch cut from a uniform 2^30-base template with 10 % substitutions."""

    def __init__(self, nreads: int = 1_000_000, tlen: int = C4_TEMPLATE_LEN, mu: float = C4_MU,
                 sigma: float = C4_SIGMA, seed_t: int = SEED_C4_TEMPLATE, seed_len: int = SEED_C4_LENGTHS,
                 seed_start: int = SEED_C4_STARTS, seed_sub: int = SEED_C4_SUBST):
        self.nreads, self.tlen = nreads, tlen
        self.seed_t, self.seed_sub = seed_t, seed_sub
        r = _arange(0, nreads)
        u1 = ((mix64(seed_len, 2 * r) >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)
        u2 = (mix64(seed_len, 2 * r + np.uint64(1)) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
        L = np.maximum(1, np.rint(np.exp(mu + sigma * z))).astype(np.int64)
        L = np.minimum(L, tlen)
        us = (mix64(seed_start, r) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        self.lengths = L
        self.starts = np.floor(us * (tlen - L + 1).astype(np.float64)).astype(np.int64)
        self.read_off = np.zeros(nreads + 1, dtype=np.int64)
        np.cumsum(L, out=self.read_off[1:])
        self.n = int(self.read_off[-1])

    def read_ascii(self, r: int) -> np.ndarray:
        return self.ascii_range(int(self.read_off[r]), int(self.read_off[r + 1]))

    def ascii_range(self, lo: int, hi: int) -> np.ndarray:
        """Bytes of the concatenated read batch, global positions [lo, hi)."""
        g = _arange(lo, hi - lo)
        rid = np.searchsorted(self.read_off, g.astype(np.int64), side="right") - 1
        t = g.astype(np.int64) - self.read_off[rid] + self.starts[rid]
        b = (mix64(self.seed_t, t.astype(np.uint64)) >> np.uint64(62)).astype(np.uint8)
        v = mix64(self.seed_sub, g)
        sub = (v >> np.uint64(32)) < np.uint64(C4_SUBST_T)
        alt = ((b.astype(np.uint64) + np.uint64(1) + (v & np.uint64(0xFFFFFFFF)) % np.uint64(3)) & np.uint64(3)).astype(np.uint8)
        b = np.where(sub, alt, b)
        return codes_to_ascii(b)


# --------------------------------------------------------------------------
# C2 element streams
# --------------------------------------------------------------------------
def c2_u32(n: int, seed: int = SEED_C2_U32, lo: int = 0) -> np.ndarray:
    """Elements [lo, lo+n) of the u32 stream (little-endian halves of mix64)."""
    i = _arange(lo, n)
    r = mix64(seed, i >> np.uint64(1))
    sh = (i & np.uint64(1)) * np.uint64(32)
    return ((r >> sh) & np.uint64(0xFFFFFFFF)).astype(np.uint32)


_NORMAL_TABLE = None


def normal_table() -> np.ndarray:
    """TABLE[j] = float32(Phi^-1((j + 0.5) / 65536)), j in [0, 65536)."""
    global _NORMAL_TABLE
    if _NORMAL_TABLE is None:
        from scipy.special import ndtri
        j = np.arange(65536, dtype=np.float64)
        _NORMAL_TABLE = ndtri((j + 0.5) / 65536.0).astype(np.float32)
    return _NORMAL_TABLE


def c2_f32(n: int, seed: int = SEED_C2_F32, lo: int = 0) -> np.ndarray:
    """Elements [lo, lo+n) of the f32 N(0,1)-shaped stream."""
    r = mix64(seed, _arange(lo, n))
    return normal_table()[(r >> np.uint64(48)).astype(np.int64)]
