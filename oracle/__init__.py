"""CPU oracle for the hot path of arxiv 1811.10074 -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this package.  The product package
`paper_1811_10074_b200` never imports it; the two share no code (only the input
generators in `synthgen/`).

The arithmetic lives in `oracle/oracle.c` (plain C, each function citing the
PAPER.md passage it evaluates); this module only loads it with ctypes and
marshals numpy arrays.  Build with `python -m oracle.build` (or
`__graft_entry__.build()`).

Pins (tests/test_oracle_*.py, all `-m "not gpu"`):
  * orc_slsum   closed form for ADD_U32 (prefix differences), numpy
                sliding_window_view min/max, the f64 sum within the float32
                rounding bound, function-evaluation semantics for AFFINE,
                SPEC.md worked examples, w = 1 identity, w = n full fold.
  * orc_hash    exhaustive bijectivity for b <= 20, inverse round trip,
                external test vectors, a shift/add
                restatement of the published Wang mix.
  * orc_mz      Fig. 2 caption facts on a constructed
                instance, SPEC.md examples, numpy argmin brute force, exhaustive
                4^L strings, density band (L85), invariants.
  * orc_mz_ties hand examples, a pure-Python brute force from the reading (R35), equality
                with orc_mz when no window repeats a key, containment of orc_mz's set.
  * orc_seedtable  sort-based construction (Python sorted), partition property.
  * orc_kmer_rc / canonical keys: hand-computed reverse complements, involution, the
                canonical code of a k-mer equals that of its reverse complement, and strand
                symmetry of canonical minimizers (S and revcomp(S) give mirrored positions).
  * orc_lookup  SPEC S:L327-330 examples, a Python dict of every stored seed, the partition
                property (looking up every stored seed reproduces the table).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")

MIN_U32, MAX_U32, ADD_U32, ADD_F32, AFFINE_U32X2, MIN_U64, CONCAT_U32X2 = range(7)
KEY_HASH, KEY_RAW, KEY_CANON, KEY_CANON_RAW = 0, 1, 2, 3
_DTYPE = {MIN_U32: np.uint32, MAX_U32: np.uint32, ADD_U32: np.uint32, ADD_F32: np.float32,
          AFFINE_U32X2: np.uint32, MIN_U64: np.uint64, CONCAT_U32X2: np.uint32}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            from . import build as _b
            _b.build()
        L = ctypes.CDLL(LIB_PATH)
        u64, i64, i32, u32, vp = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p
        L.orc_slsum.argtypes = [i32, u32, vp, vp, u64]
        L.orc_slsum.restype = i32
        L.orc_prefix.argtypes = [i32, vp, vp, u64]
        L.orc_prefix.restype = i32
        L.orc_encode.argtypes = [vp, u64, vp, vp]
        L.orc_pack.argtypes = [vp, u64, vp, vp]
        L.orc_kmer.argtypes = [vp, u64, i32]
        L.orc_kmer.restype = u64
        L.orc_kmer_rc.argtypes = [vp, u64, i32]
        L.orc_kmer_rc.restype = u64
        L.orc_hash.argtypes = [u64, i32]
        L.orc_hash.restype = u64
        L.orc_unhash.argtypes = [u64, i32]
        L.orc_unhash.restype = u64
        L.orc_hash_array.argtypes = [vp, vp, u64, i32]
        L.orc_mz.argtypes = [vp, u64, i32, i32, vp, u64, i32, u64, u64, u64, vp, vp, u64]
        L.orc_mz.restype = i64
        L.orc_mz_ties.argtypes = [vp, u64, i32, i32, vp, u64, i32, u64, vp, vp, u64]
        L.orc_mz_ties.restype = i64
        L.orc_fingerprint.argtypes = [u64, i32]
        L.orc_fingerprint.restype = u32
        L.orc_seedtable.argtypes = [vp, vp, u64, i32, i32, vp, vp, vp]
        L.orc_seedtable.restype = i32
        L.orc_lookup.argtypes = [vp, u64, i32, i32, vp, vp, vp, vp, vp, u64]
        L.orc_lookup.restype = i64
        L.orc_num_threads.restype = i32
        L.orc_set_num_threads.argtypes = [i32]
        _lib = L
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return lib().orc_num_threads()


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))


def as_bytes(seq) -> np.ndarray:
    if isinstance(seq, (bytes, bytearray)):
        return np.frombuffer(bytes(seq), dtype=np.uint8)
    if isinstance(seq, str):
        return np.frombuffer(seq.encode("ascii"), dtype=np.uint8)
    return np.ascontiguousarray(seq, dtype=np.uint8)


# ---------------------------------------------------------------- sliding sums
def slsum(op: int, w: int, x: np.ndarray) -> np.ndarray:
    """Eq. 2 by the naive O(wN) strict left fold.  AFFINE_U32X2 and CONCAT_U32X2 take x of
    shape (n, 2)."""
    x = np.ascontiguousarray(x, dtype=_DTYPE[op])
    n = x.shape[0]
    shape = (max(0, n - w + 1),) + x.shape[1:]
    y = np.zeros(shape, dtype=x.dtype)
    rc = lib().orc_slsum(op, w, _p(x), _p(y), n)
    if rc != 0:
        raise ValueError(f"orc_slsum: error {rc}")
    return y


def prefix(op: int, x: np.ndarray) -> np.ndarray:
    """Eq. 1 prefix sums (strict left fold)."""
    x = np.ascontiguousarray(x, dtype=_DTYPE[op])
    y = np.zeros_like(x)
    rc = lib().orc_prefix(op, _p(x), _p(y), x.shape[0])
    if rc != 0:
        raise ValueError(f"orc_prefix: error {rc}")
    return y


# ---------------------------------------------------------------- DNA
def encode(seq):
    s = as_bytes(seq)
    code = np.zeros(len(s), np.uint8)
    valid = np.zeros(len(s), np.uint8)
    lib().orc_encode(_p(s), len(s), _p(code), _p(valid))
    return code, valid.astype(bool)


def pack(seq):
    """MSB-first 2-bit words (32 bases per uint64) and the invalid bitmap (uint32 per 32 bases)."""
    s = as_bytes(seq)
    nw = (len(s) + 31) // 32
    words = np.zeros(nw, np.uint64)
    inval = np.zeros(nw, np.uint32)
    lib().orc_pack(_p(s), len(s), _p(words), _p(inval))
    return words, inval


def kmer(codes: np.ndarray, i: int, k: int) -> int:
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    return int(lib().orc_kmer(_p(codes), i, k))


def kmer_rc(codes: np.ndarray, i: int, k: int) -> int:
    """Code of the reverse complement of the k-mer at i (R32)."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    return int(lib().orc_kmer_rc(_p(codes), i, k))


def hash_(x: int, b: int) -> int:
    return int(lib().orc_hash(x, b))


def unhash(y: int, b: int) -> int:
    return int(lib().orc_unhash(y, b))


def hash_array(x: np.ndarray, b: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.uint64)
    y = np.zeros_like(x)
    lib().orc_hash_array(_p(x), _p(y), len(x), b)
    return y


def mz(seq, k: int, w: int, read_off=None, keymode: int = KEY_HASH, pos_base: int = 0,
       win_lo: int = 0, win_hi: int = 2 ** 64 - 1, cap: int | None = None):
    """Minimizers: returns (key uint64[M], pos uint64[M]) by ascending pos.

    `cap` (marshalling only): when given, the output arrays are allocated with that many
    entries and orc_mz runs once; if the count exceeds it, it runs again with the exact
    count.  Without it, a counting call precedes the filling call."""
    s = as_bytes(seq)
    ro = None if read_off is None else np.ascontiguousarray(read_off, dtype=np.uint64)
    nreads = 0 if ro is None else len(ro) - 1
    L = lib()
    if cap is not None:
        key = np.empty(max(1, cap), np.uint64)
        pos = np.empty(max(1, cap), np.uint64)
        cnt = L.orc_mz(_p(s), len(s), k, w, _p(ro), nreads, keymode, pos_base, win_lo, win_hi,
                       _p(key), _p(pos), cap)
        if cnt < 0:
            raise ValueError(f"orc_mz: error {cnt}")
        if cnt <= cap:
            return key[:cnt], pos[:cnt]
    cnt = L.orc_mz(_p(s), len(s), k, w, _p(ro), nreads, keymode, pos_base, win_lo, win_hi, None, None, 0)
    if cnt < 0:
        raise ValueError(f"orc_mz: error {cnt}")
    key = np.zeros(cnt, np.uint64)
    pos = np.zeros(cnt, np.uint64)
    if cnt:
        L.orc_mz(_p(s), len(s), k, w, _p(ro), nreads, keymode, pos_base, win_lo, win_hi, _p(key), _p(pos), cnt)
    return key, pos


def mz_ties(seq, k: int, w: int, read_off=None, keymode: int = KEY_HASH, pos_base: int = 0):
    """minimap2-compatible minimizers (R35: all tied minima, run-end windows,
    symmetric k-mers skipped): returns (key uint64[M], pos uint64[M]) by ascending pos."""
    s = as_bytes(seq)
    ro = None if read_off is None else np.ascontiguousarray(read_off, dtype=np.uint64)
    nreads = 0 if ro is None else len(ro) - 1
    L = lib()
    cnt = L.orc_mz_ties(_p(s), len(s), k, w, _p(ro), nreads, keymode, pos_base, None, None, 0)
    if cnt < 0:
        raise ValueError(f"orc_mz_ties: error {cnt}")
    key = np.zeros(cnt, np.uint64)
    pos = np.zeros(cnt, np.uint64)
    if cnt:
        L.orc_mz_ties(_p(s), len(s), k, w, _p(ro), nreads, keymode, pos_base, _p(key), _p(pos), cnt)
    return key, pos


def fingerprint(key: int, k: int) -> int:
    return int(lib().orc_fingerprint(key, k))


def lookup(q: np.ndarray, k: int, bits: int, offsets: np.ndarray, fp: np.ndarray, pos_tab: np.ndarray):
    """Seed lookup (Fig. 1, L63-65; NEXT f1): returns (hit_off[nq+1], hit_pos[total])."""
    q = np.ascontiguousarray(q, dtype=np.uint64)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    fp = np.ascontiguousarray(fp, dtype=np.uint32)
    pos_tab = np.ascontiguousarray(pos_tab, dtype=np.uint64)
    nq = len(q)
    hit_off = np.zeros(nq + 1, np.uint64)
    tot = lib().orc_lookup(_p(q), nq, k, bits, _p(offsets), _p(fp), _p(pos_tab), _p(hit_off), None, 0)
    if tot < 0:
        raise ValueError(f"orc_lookup: error {tot}")
    hit_pos = np.zeros(max(1, tot), np.uint64)
    lib().orc_lookup(_p(q), nq, k, bits, _p(offsets), _p(fp), _p(pos_tab), _p(hit_off), _p(hit_pos), tot)
    return hit_off, hit_pos[:tot]


def seedtable(key: np.ndarray, pos: np.ndarray, k: int, bits: int):
    """Seed pointer table (offsets[2^bits+1]) + position table (+ fingerprints), Fig. 1."""
    key = np.ascontiguousarray(key, dtype=np.uint64)
    pos = np.ascontiguousarray(pos, dtype=np.uint64)
    m = len(key)
    offsets = np.zeros((1 << bits) + 1, np.uint64)
    fp = np.zeros(m, np.uint32)
    pos_out = np.zeros(m, np.uint64)
    rc = lib().orc_seedtable(_p(key), _p(pos), m, k, bits, _p(offsets), _p(fp), _p(pos_out))
    if rc != 0:
        raise ValueError(f"orc_seedtable: error {rc}")
    return offsets, fp, pos_out
