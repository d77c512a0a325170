"""MSDT serialization of a seed table ("External Interfaces").

Little-endian layout:
  magic b"MSDT" | version u32 = 1 | mode u8 (0 = direct, 1 = hashed) | k u8 | w u8 | reserved u8 |
  entry count u64 | (direct mode) 4^k + 1 u64 pointer offsets | count x (seed u64, position u64)

The tables of this library are bucketed CSRs (include/mzslsum.h, R21):
  * direct mode is the Fig. 1 table: RAW keys with bucket_bits = 2k (k <= 12), so the
    pointer table has 4^k + 1 offsets and an entry's seed is its bucket;
  * hashed mode stores each entry's 32-bit fingerprint as its seed (the table keeps the top 32
    bits of the 2k-bit hash, not the hash itself), with no pointer table (SPEC's sorted-hash mode):
    entries are written sorted by (seed, position), so the seed column is non-decreasing.
Readers reject an unknown magic or version.  Host-side I/O only (numpy), not the hot path.
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"MSDT"
VERSION = 1
MODE_DIRECT, MODE_HASHED = 0, 1
_HDR = struct.Struct("<4sIBBBBQ")


def save(path: str, offsets, fp, pos, k: int, w: int, mode: int) -> None:
    """Write a table (offsets[2^bits+1], fingerprints fp[m], positions pos[m]) as MSDT."""
    offsets = np.ascontiguousarray(np.asarray(offsets), dtype=np.uint64)
    fp = np.ascontiguousarray(np.asarray(fp).view(np.uint32) if np.asarray(fp).dtype != np.uint32
                              else np.asarray(fp), dtype=np.uint32)
    pos = np.ascontiguousarray(np.asarray(pos), dtype=np.uint64)
    m = int(offsets[-1])
    if len(fp) < m or len(pos) < m:
        raise ValueError("fp/pos shorter than the table")
    if mode == MODE_DIRECT:
        if not 1 <= k <= 12 or len(offsets) != (1 << (2 * k)) + 1:
            raise ValueError("direct mode needs k <= 12 and 4^k + 1 offsets (bucket_bits = 2k, raw keys)")
        seeds = (fp[:m].astype(np.uint64) >> np.uint64(32 - 2 * k))
    elif mode == MODE_HASHED:
        # SPEC's hashed mode lists entries by (seed, position) so a reader can binary-search the
        # seed column.  The table is in (bucket, position) order and a bucket holds several
        # fingerprints, so sort stably by the fingerprint: positions stay ascending per seed.
        o = np.argsort(fp[:m], kind="stable")
        seeds = fp[:m][o].astype(np.uint64)
        pos = pos[:m][o]
    else:
        raise ValueError(f"unknown mode {mode}")
    with open(path, "wb") as f:
        f.write(_HDR.pack(MAGIC, VERSION, mode, k, w, 0, m))
        if mode == MODE_DIRECT:
            f.write(offsets.astype("<u8").tobytes())
        ent = np.empty((m, 2), dtype="<u8")
        ent[:, 0] = seeds
        ent[:, 1] = pos[:m]
        f.write(ent.tobytes())


def load(path: str):
    """Read an MSDT file: returns dict(mode, k, w, offsets or None, seeds, pos)."""
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < _HDR.size:
        raise ValueError("truncated MSDT header")
    magic, version, mode, k, w, _, m = _HDR.unpack_from(raw, 0)
    if magic != MAGIC:
        raise ValueError(f"bad magic {magic!r}")
    if version != VERSION:
        raise ValueError(f"unsupported MSDT version {version}")
    o = _HDR.size
    offsets = None
    if mode == MODE_DIRECT:
        n_off = (1 << (2 * k)) + 1
        offsets = np.frombuffer(raw, dtype="<u8", count=n_off, offset=o).astype(np.uint64)
        o += 8 * n_off
    elif mode != MODE_HASHED:
        raise ValueError(f"unknown mode {mode}")
    ent = np.frombuffer(raw, dtype="<u8", count=2 * m, offset=o).reshape(m, 2)
    return {"mode": mode, "k": k, "w": w, "offsets": offsets, "seeds": ent[:, 0].astype(np.uint64),
            "pos": ent[:, 1].astype(np.uint64)}
