"""ctypes binding of libmzslsum.so (include/mzslsum.h).  Argument marshalling only.

Every step of the hot path runs in the CUDA library; this module only turns torch
tensors into device pointers and the current CUDA stream into a cudaStream_t.  There is
no CPU fallback: if the shared library is missing, importing the module raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
# MZS_LIB: an alternative build of the same library (tools/prof_nsweep.py's instrumented one)
LIB_PATH = os.environ.get("MZS_LIB") or os.path.join(HERE, "libmzslsum.so")

# ---------------------------------------------------------------- constants (mzslsum.h)
SLSUM_OK, SLSUM_EINVAL, SLSUM_EUNSUPPORTED, SLSUM_ECAPACITY, SLSUM_ECUDA, SLSUM_ENOMEM = 0, -1, -2, -3, -4, -5
SLSUM_MIN_U32, SLSUM_MAX_U32, SLSUM_ADD_U32, SLSUM_ADD_F32, SLSUM_AFFINE_U32X2, SLSUM_MIN_U64, SLSUM_CONCAT_U32X2 = range(7)
SLSUM_PATH_GENERIC, SLSUM_PATH_COMMUTATIVE, SLSUM_PATH_AUTO, SLSUM_PATH_RECURRENT, SLSUM_PATH_SCALAR = range(5)
MZ_IN_ASCII, MZ_IN_PACKED2 = 0, 1
MZ_KEY_HASH, MZ_KEY_RAW, MZ_KEY_CANON, MZ_KEY_CANON_RAW = 0, 1, 2, 3
U64_MAX = 2 ** 64 - 1

OP_DTYPE = {SLSUM_MIN_U32: torch.uint32, SLSUM_MAX_U32: torch.uint32, SLSUM_ADD_U32: torch.uint32,
            SLSUM_ADD_F32: torch.float32, SLSUM_AFFINE_U32X2: torch.uint32, SLSUM_MIN_U64: torch.uint64,
            SLSUM_CONCAT_U32X2: torch.uint32}


class SlsumError(RuntimeError):
    def __init__(self, rc: int, what: str):
        self.rc = rc
        super().__init__(f"{what}: {strerror(rc)} ({rc})")


class MzIn(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("seq", ctypes.c_void_p), ("invalid", ctypes.c_void_p),
                ("n", ctypes.c_uint64), ("read_off", ctypes.c_void_p), ("nreads", ctypes.c_uint64),
                ("pos_base", ctypes.c_uint64), ("win_lo", ctypes.c_uint64), ("win_hi", ctypes.c_uint64)]


class MzOut(ctypes.Structure):
    _fields_ = [("hash", ctypes.c_void_p), ("pos", ctypes.c_void_p), ("capacity", ctypes.c_uint64),
                ("d_count", ctypes.c_void_p), ("items", ctypes.c_void_p), ("hist", ctypes.c_void_p),
                ("hist_bucket_bits", ctypes.c_int)]


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_1811_10074_b200/build.py` "
                      "(there is no CPU fallback)")

_L = ctypes.CDLL(LIB_PATH)
_u64, _i32, _u32, _vp, _sz = ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_size_t


def _sig(name, res, *args):
    f = getattr(_L, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_strerror = _sig("slsum_strerror", ctypes.c_char_p, _i32)
_version = _sig("slsum_version", _i32)
_slsum_run = _sig("slsum_run", _i32, _i32, _u32, _vp, _vp, _u64)
_slsum_run_ex = _sig("slsum_run_ex", _i32, _i32, _u32, _vp, _vp, _u64, _i32, _vp)
_mz_encode = _sig("mz_encode", _i32, _vp, _u64, _vp, _vp, _vp)
_mz_ws = _sig("mz_workspace_bytes", _sz, _u64, _i32, _i32, _i32)
_mz_extract_ex = _sig("mz_extract_ex", _i32, ctypes.POINTER(MzIn), _i32, _i32, _i32, ctypes.POINTER(MzOut), _vp, _sz, _vp)
_mz_extract_path = _sig("mz_extract_path", _i32, ctypes.POINTER(MzIn), _i32, _i32, _i32, ctypes.POINTER(MzOut), _vp,
                        _sz, _vp, _i32)
_mz_extract = _sig("mz_extract", _i32, _vp, _u64, _i32, _i32, ctypes.POINTER(MzOut))
_mz_ties_ws = _sig("mz_ties_workspace_bytes", _sz, _u64, _i32, _i32, _i32)
_mz_extract_ties = _sig("mz_extract_ties", _i32, ctypes.POINTER(MzIn), _i32, _i32, _i32, ctypes.POINTER(MzOut), _vp,
                        _sz, _vp)
_st_ws = _sig("seedtable_workspace_bytes", _sz, _u64, _i32)
_st_build = _sig("seedtable_build", _i32, _vp, _vp, _u64, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp)
_st_build_items = _sig("seedtable_build_items", _i32, _vp, _vp, _vp, _u64, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _sz,
                       _vp)
_st_build_items32 = _sig("seedtable_build_items32", _i32, _vp, _vp, _vp, _u64, _vp, _i32, _i32, _vp, _vp, _vp, _vp,
                         _sz, _vp)
_st_hist_words = _sig("seedtable_hist_words", _sz, _u64, _i32)
_st_build_items_ex = _sig("seedtable_build_items_ex", _i32, _vp, _vp, _vp, _u64, _vp, _i32, _i32, _vp, _vp, _vp, _vp,
                          _vp, _vp, _sz, _vp)
_st_count = _sig("seedtable_count", _i32, _vp, _u64, _vp, _i32, _i32, _vp, _vp)
_st_part_ws = _sig("seedtable_partition_workspace_bytes", _sz, _u64, _i32)
_st_part = _sig("seedtable_partition", _i32, _vp, _vp, _u64, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp)
_st_p2p_ws = _sig("seedtable_partition_p2p_workspace_bytes", _sz, _u64, _i32)
_st_p2p = _sig("seedtable_partition_p2p", _i32, _vp, _vp, _u64, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp)
_st_p2p_it = _sig("seedtable_partition_p2p_items", _i32, _vp, _vp, _u64, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp,
                  _sz, _vp)
_st_fin_ws = _sig("seedtable_finalize_workspace_bytes", _sz, _u64, _i32, _i32)
_st_lk_ws = _sig("seedtable_lookup_workspace_bytes", _sz, _u64)
_st_lk = _sig("seedtable_lookup", _i32, _vp, _u64, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _u64, _vp, _vp, _sz, _vp)
_st_fin = _sig("seedtable_finalize", _i32, _vp, _vp, _u64, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp)

EXPORTS = ["slsum_strerror", "slsum_version", "slsum_run", "slsum_run_ex", "mz_encode", "mz_workspace_bytes",
           "mz_extract_ex", "mz_extract", "seedtable_workspace_bytes", "seedtable_build", "seedtable_build_items", "seedtable_build_items32", "seedtable_count",
           "seedtable_partition_workspace_bytes", "seedtable_partition", "seedtable_finalize_workspace_bytes",
           "seedtable_finalize", "seedtable_lookup_workspace_bytes", "seedtable_lookup",
           "seedtable_partition_p2p_workspace_bytes", "seedtable_partition_p2p", "seedtable_partition_p2p_items",
           "mz_extract_path", "mz_ties_workspace_bytes", "mz_extract_ties"]


def strerror(rc: int) -> str:
    return _strerror(rc).decode()


def version() -> int:
    return _version()


def _check(rc: int, what: str) -> int:
    if rc != SLSUM_OK:
        raise SlsumError(rc, what)
    return rc


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("device tensor required (the library takes device pointers)")
    if not t.is_contiguous():
        raise ValueError("contiguous tensor required")
    return t.data_ptr()


def _need(t: torch.Tensor | None, name: str, dtype, numel: int, allow_none: bool = False) -> None:
    """Argument check before a raw device pointer crosses the ABI: the kernels trust sizes."""
    if t is None:
        if allow_none:
            return
        raise ValueError(f"{name} is required")
    if t.dtype != dtype:
        raise ValueError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if t.numel() < numel:
        raise ValueError(f"{name}: {t.numel()} elements, at least {numel} needed")


# element layout of each slsum op: (dtype, values per element)
OP_LAYOUT = {SLSUM_MIN_U32: (torch.uint32, 1), SLSUM_MAX_U32: (torch.uint32, 1), SLSUM_ADD_U32: (torch.uint32, 1),
             SLSUM_ADD_F32: (torch.float32, 1), SLSUM_AFFINE_U32X2: (torch.uint32, 2),
             SLSUM_MIN_U64: (torch.uint64, 1), SLSUM_CONCAT_U32X2: (torch.uint32, 2)}


def _stream(stream: torch.cuda.Stream | None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(1, int(nbytes)), dtype=torch.uint8, device=device)


# ---------------------------------------------------------------- sliding sums (Eq. 2)
def slsum_run(op: int, w: int, x: torch.Tensor, y: torch.Tensor | None = None, path: int = SLSUM_PATH_GENERIC,
              stream=None) -> torch.Tensor:
    """y_i = x_i (+) ... (+) x_{i+w-1} on the device.  AFFINE_U32X2 and CONCAT_U32X2 take x of
    shape (n, 2)."""
    if op not in OP_LAYOUT:
        raise ValueError(f"unknown op {op}")
    dt, per = OP_LAYOUT[op]
    if x.dtype != dt or tuple(x.shape[1:]) != ((per,) if per > 1 else ()):
        raise ValueError(f"op {op} takes x of dtype {dt} and shape (n{', %d' % per if per > 1 else ''}); "
                         f"got {x.dtype} {tuple(x.shape)}")
    n = x.shape[0]
    nout = max(0, n - w + 1)
    if y is None:
        y = torch.empty((nout,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    _need(y, "y", dt, nout * per)
    _check(_slsum_run_ex(op, w, _ptr(x), _ptr(y), n, path, _stream(stream)), "slsum_run_ex")
    return y


# ---------------------------------------------------------------- 2-bit packing
def mz_encode(seq: torch.Tensor, words: torch.Tensor | None = None, invalid: torch.Tensor | None = None,
              stream=None):
    n = seq.numel()
    nw = (n + 31) // 32
    if words is None:
        words = torch.empty(nw, dtype=torch.uint64, device=seq.device)
    if invalid is None:
        invalid = torch.empty(nw, dtype=torch.uint32, device=seq.device)
    _need(seq, "seq", torch.uint8, n)
    _need(words, "words", torch.uint64, nw)
    _need(invalid, "invalid", torch.uint32, nw)
    _check(_mz_encode(_ptr(seq), n, _ptr(words), _ptr(invalid), _stream(stream)), "mz_encode")
    return words, invalid


# ---------------------------------------------------------------- minimizers
def mz_workspace_bytes(n: int, k: int, w: int, kind: int = MZ_IN_ASCII) -> int:
    return int(_mz_ws(n, k, w, kind))


def mz_extract_ex(seq: torch.Tensor, k: int, w: int, *, n: int | None = None, kind: int = MZ_IN_ASCII,
                  invalid: torch.Tensor | None = None, read_off: torch.Tensor | None = None, pos_base: int = 0,
                  win_lo: int = 0, win_hi: int = U64_MAX, keymode: int = MZ_KEY_HASH,
                  capacity: int | None = None, out_hash: torch.Tensor | None = None,
                  out_pos: torch.Tensor | None = None, d_count: torch.Tensor | None = None,
                  ws: torch.Tensor | None = None, stream=None, path: int = 0,
                  out_items: torch.Tensor | None = None, out_hist: torch.Tensor | None = None,
                  hist_bits: int = 0):
    """Asynchronous minimizer extraction; returns (hash, pos, d_count) device tensors (count on device).
    out_items (uint64, capacity entries, optional) also receives the packed seed-table items
    (seedtable_build_items); out_hist (uint32, seedtable_hist_words(capacity, hist_bits)) the
    first radix pass's digit counts of a table of `hist_bits` buckets (seedtable_build_items_ex)."""
    if n is None:
        n = seq.numel() if kind == MZ_IN_ASCII else seq.numel() * 32
    span = k + w - 1
    nwin = max(0, n - span + 1)
    if capacity is None:
        capacity = out_hash.numel() if out_hash is not None else nwin
    dev = seq.device
    if out_hash is None:
        out_hash = torch.empty(max(1, capacity), dtype=torch.uint64, device=dev)
    if out_pos is None:
        out_pos = torch.empty(max(1, capacity), dtype=torch.uint64, device=dev)
    if d_count is None:
        d_count = torch.zeros(1, dtype=torch.uint64, device=dev)
    if ws is None:
        ws = _ws(mz_workspace_bytes(n, k, w, kind), dev)
    nreads = 0 if read_off is None else read_off.numel() - 1
    if kind == MZ_IN_ASCII:
        _need(seq, "seq", torch.uint8, n)
    else:
        _need(seq, "seq (packed words)", torch.uint64, (n + 31) // 32)
        _need(invalid, "invalid", torch.uint32, (n + 31) // 32, allow_none=True)
    for name, t in (("out_hash", out_hash), ("out_pos", out_pos), ("out_items", out_items)):
        _need(t, name, torch.uint64, capacity, allow_none=name == "out_items")
    _need(d_count, "d_count", torch.uint64, 1)
    _need(read_off, "read_off", torch.uint64, 2, allow_none=True)
    if out_hist is not None:
        _need(out_hist, "out_hist", torch.uint32, seedtable_hist_words(capacity, hist_bits))
    if ws.numel() < mz_workspace_bytes(n, k, w, kind):
        raise ValueError("ws smaller than mz_workspace_bytes")
    mi = MzIn(kind, _ptr(seq), _ptr(invalid), n, _ptr(read_off), nreads, pos_base, win_lo, win_hi)
    mo = MzOut(_ptr(out_hash), _ptr(out_pos), capacity, _ptr(d_count), _ptr(out_items), _ptr(out_hist), hist_bits)
    if path == 0:      # the declared entry point (automatic kernel choice)
        _check(_mz_extract_ex(ctypes.byref(mi), k, w, keymode, ctypes.byref(mo), _ptr(ws), ws.numel(),
                              _stream(stream)), "mz_extract_ex")
    else:              # test hook: force the generic kernel (include/mzslsum.h mz_extract_path)
        _check(_mz_extract_path(ctypes.byref(mi), k, w, keymode, ctypes.byref(mo), _ptr(ws), ws.numel(),
                                _stream(stream), path), "mz_extract_path")
    return out_hash, out_pos, d_count


def mz_extract(seq: torch.Tensor, k: int, w: int, **kw):
    """Synchronous convenience: returns (hash, pos) trimmed to the record count."""
    h, p, c = mz_extract_ex(seq, k, w, **kw)
    cnt = int(c.item())
    cap = kw.get("capacity", h.numel())
    if cnt > h.numel():
        raise SlsumError(SLSUM_ECAPACITY, f"mz_extract: {cnt} records > capacity {cap}")
    return h[:cnt], p[:cnt]


# ---------------------------------------------------------------- seed table (Fig. 1)
def mz_ties_workspace_bytes(n: int, k: int, w: int, kind: int = MZ_IN_ASCII) -> int:
    return int(_mz_ties_ws(n, k, w, kind))


def mz_extract_ties(seq: torch.Tensor, k: int, w: int, *, n: int | None = None, kind: int = MZ_IN_ASCII,
                    invalid: torch.Tensor | None = None, read_off: torch.Tensor | None = None, pos_base: int = 0,
                    keymode: int = MZ_KEY_HASH, capacity: int | None = None,
                    out_hash: torch.Tensor | None = None, out_pos: torch.Tensor | None = None,
                    d_count: torch.Tensor | None = None, out_items: torch.Tensor | None = None,
                    ws: torch.Tensor | None = None, stream=None):
    """minimap2-compatible minimizers (include/mzslsum.h mz_extract_ties; R35), asynchronous:
    returns (hash, pos, d_count) device tensors, count on the device."""
    if n is None:
        n = seq.numel() if kind == MZ_IN_ASCII else seq.numel() * 32
    nk = max(0, n - k + 1)
    if capacity is None:
        capacity = out_hash.numel() if out_hash is not None else nk
    dev = seq.device
    if out_hash is None:
        out_hash = torch.empty(max(1, capacity), dtype=torch.uint64, device=dev)
    if out_pos is None:
        out_pos = torch.empty(max(1, capacity), dtype=torch.uint64, device=dev)
    if d_count is None:
        d_count = torch.zeros(1, dtype=torch.uint64, device=dev)
    if ws is None:
        ws = _ws(mz_ties_workspace_bytes(n, k, w, kind), dev)
    nreads = 0 if read_off is None else read_off.numel() - 1
    if kind == MZ_IN_ASCII:
        _need(seq, "seq", torch.uint8, n)
    else:
        _need(seq, "seq (packed words)", torch.uint64, (n + 31) // 32)
        _need(invalid, "invalid", torch.uint32, (n + 31) // 32, allow_none=True)
    for name, t in (("out_hash", out_hash), ("out_pos", out_pos), ("out_items", out_items)):
        _need(t, name, torch.uint64, capacity, allow_none=name == "out_items")
    _need(d_count, "d_count", torch.uint64, 1)
    _need(read_off, "read_off", torch.uint64, 2, allow_none=True)
    if ws.numel() < mz_ties_workspace_bytes(n, k, w, kind):
        raise ValueError("ws smaller than mz_ties_workspace_bytes")
    mi = MzIn(kind, _ptr(seq), _ptr(invalid), n, _ptr(read_off), nreads, pos_base, 0, U64_MAX)
    mo = MzOut(_ptr(out_hash), _ptr(out_pos), capacity, _ptr(d_count), _ptr(out_items), None, 0)
    _check(_mz_extract_ties(ctypes.byref(mi), k, w, keymode, ctypes.byref(mo), _ptr(ws), ws.numel(),
                            _stream(stream)), "mz_extract_ties")
    return out_hash, out_pos, d_count


def seedtable_workspace_bytes(m: int, bits: int) -> int:
    return int(_st_ws(m, bits))


def _table_checks(hash_, pos, m, d_m, bits, offsets, pos_out, fp_out, ws):
    _need(hash_, "hash", torch.uint64, m)
    _need(pos, "pos", torch.uint64, m)
    _need(d_m, "d_m", torch.uint64, 1, allow_none=True)
    if 1 <= bits <= 30:                      # other values are the library's EINVAL to report
        _need(offsets, "offsets", torch.uint64, (1 << bits) + 1)
    _need(pos_out, "pos_out", torch.uint64, m, allow_none=pos_out is None)
    _need(fp_out, "fp_out", torch.uint32, m, allow_none=True)
    if 1 <= bits <= 30 and ws.numel() < seedtable_workspace_bytes(max(1, m), bits):
        raise ValueError("ws smaller than seedtable_workspace_bytes")


def seedtable_build(hash_: torch.Tensor, pos: torch.Tensor, k: int, bits: int, *, m: int | None = None,
                    d_m: torch.Tensor | None = None, with_fp: bool = True, offsets: torch.Tensor | None = None,
                    pos_out: torch.Tensor | None = None, fp_out: torch.Tensor | None = None,
                    ws: torch.Tensor | None = None, stream=None):
    """Returns (offsets[2^bits+1], pos_out[m], fp_out[m] or None)."""
    if m is None:
        m = hash_.numel()
    dev = hash_.device
    if offsets is None:
        offsets = torch.empty((1 << bits) + 1, dtype=torch.uint64, device=dev)
    if pos_out is None:
        pos_out = torch.empty(max(1, m), dtype=torch.uint64, device=dev)
    if fp_out is None and with_fp:
        fp_out = torch.empty(max(1, m), dtype=torch.uint32, device=dev)
    if ws is None:
        ws = _ws(seedtable_workspace_bytes(max(1, m), bits), dev)
    _table_checks(hash_, pos, m, d_m, bits, offsets, pos_out, fp_out, ws)
    _check(_st_build(_ptr(hash_), _ptr(pos), m, _ptr(d_m), k, bits, _ptr(offsets), _ptr(fp_out), _ptr(pos_out),
                     _ptr(ws), ws.numel(), _stream(stream)), "seedtable_build")
    return offsets, pos_out, fp_out


def seedtable_build_items(items: torch.Tensor, hash_: torch.Tensor, pos: torch.Tensor, k: int, bits: int, *,
                          m: int | None = None, d_m: torch.Tensor | None = None, with_fp: bool = True,
                          offsets: torch.Tensor | None = None, pos_out: torch.Tensor | None = None,
                          fp_out: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None):
    """seedtable_build from mz_extract_ex's packed items (out_items) beside hash/pos."""
    if m is None:
        m = hash_.numel()
    dev = hash_.device
    if offsets is None:
        offsets = torch.empty((1 << bits) + 1, dtype=torch.uint64, device=dev)
    if pos_out is None:
        pos_out = torch.empty(max(1, m), dtype=torch.uint64, device=dev)
    if fp_out is None and with_fp:
        fp_out = torch.empty(max(1, m), dtype=torch.uint32, device=dev)
    if ws is None:
        ws = _ws(seedtable_workspace_bytes(max(1, m), bits), dev)
    _table_checks(hash_, pos, m, d_m, bits, offsets, pos_out, fp_out, ws)
    _need(items, "items", torch.uint64, m)
    _check(_st_build_items(_ptr(items), _ptr(hash_), _ptr(pos), m, _ptr(d_m), k, bits, _ptr(offsets), _ptr(fp_out),
                           _ptr(pos_out), _ptr(ws), ws.numel(), _stream(stream)), "seedtable_build_items")
    return offsets, pos_out, fp_out


def seedtable_build_items32(items: torch.Tensor, hash_: torch.Tensor, pos: torch.Tensor, k: int, bits: int, *,
                            m: int | None = None, d_m: torch.Tensor | None = None, with_fp: bool = True,
                            offsets: torch.Tensor | None = None, pos_out: torch.Tensor | None = None,
                            fp_out: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None):
    """seedtable_build_items with a uint32 position table (positions mod 2^32; exact below 2^32)."""
    if m is None:
        m = hash_.numel()
    dev = hash_.device
    if offsets is None:
        offsets = torch.empty((1 << bits) + 1, dtype=torch.uint64, device=dev)
    if pos_out is None:
        pos_out = torch.empty(max(1, m), dtype=torch.uint32, device=dev)
    if fp_out is None and with_fp:
        fp_out = torch.empty(max(1, m), dtype=torch.uint32, device=dev)
    if ws is None:
        ws = _ws(seedtable_workspace_bytes(max(1, m), bits), dev)
    _table_checks(hash_, pos, m, d_m, bits, offsets, None, fp_out, ws)
    _need(items, "items", torch.uint64, m)
    _need(pos_out, "pos_out", torch.uint32, m)
    _check(_st_build_items32(_ptr(items), _ptr(hash_), _ptr(pos), m, _ptr(d_m), k, bits, _ptr(offsets), _ptr(fp_out),
                             _ptr(pos_out), _ptr(ws), ws.numel(), _stream(stream)), "seedtable_build_items32")
    return offsets, pos_out, fp_out


def seedtable_hist_words(capacity: int, bits: int) -> int:
    return int(_st_hist_words(capacity, bits))


def seedtable_build_items_ex(items: torch.Tensor, hash_: torch.Tensor, pos: torch.Tensor, k: int, bits: int, *,
                             m: int | None = None, d_m: torch.Tensor | None = None, hist: torch.Tensor | None = None,
                             pos32: bool = False, with_fp: bool = True, offsets: torch.Tensor | None = None,
                             pos_out: torch.Tensor | None = None, fp_out: torch.Tensor | None = None,
                             ws: torch.Tensor | None = None, stream=None):
    """seedtable_build_items(32) starting from mz_extract_ex's first-pass digit counts (out_hist,
    made with capacity == m and hist_bits == bits); hist=None counts here."""
    if m is None:
        m = hash_.numel()
    dev = hash_.device
    if offsets is None:
        offsets = torch.empty((1 << bits) + 1, dtype=torch.uint64, device=dev)
    if pos_out is None:
        pos_out = torch.empty(max(1, m), dtype=torch.uint32 if pos32 else torch.uint64, device=dev)
    if fp_out is None and with_fp:
        fp_out = torch.empty(max(1, m), dtype=torch.uint32, device=dev)
    if ws is None:
        ws = _ws(seedtable_workspace_bytes(max(1, m), bits), dev)
    _table_checks(hash_, pos, m, d_m, bits, offsets, None, fp_out, ws)
    _need(items, "items", torch.uint64, m)
    _need(pos_out, "pos_out", torch.uint32 if pos32 else torch.uint64, m)
    _need(hist, "hist", torch.uint32, seedtable_hist_words(m, bits), allow_none=True)
    p64, p32 = (None, pos_out) if pos32 else (pos_out, None)
    _check(_st_build_items_ex(_ptr(items), _ptr(hash_), _ptr(pos), m, _ptr(d_m), k, bits, _ptr(hist), _ptr(offsets),
                              _ptr(fp_out), _ptr(p64), _ptr(p32), _ptr(ws), ws.numel(), _stream(stream)),
           "seedtable_build_items_ex")
    return offsets, pos_out, fp_out


def seedtable_lookup_workspace_bytes(nq: int) -> int:
    return int(_st_lk_ws(nq))


def seedtable_lookup(qkey: torch.Tensor, k: int, bits: int, offsets: torch.Tensor, fp: torch.Tensor,
                     pos_tab: torch.Tensor, *, nq: int | None = None, d_nq: torch.Tensor | None = None,
                     hit_cap: int | None = None, hit_off: torch.Tensor | None = None,
                     hit_pos: torch.Tensor | None = None, d_total: torch.Tensor | None = None,
                     ws: torch.Tensor | None = None, stream=None):
    """Batch seed lookup (Fig. 1).  Returns (hit_off[nq+1], hit_pos, d_total).  With
    hit_cap=None the hits are counted first and hit_pos is sized from the total (one sync)."""
    if nq is None:
        nq = qkey.numel()
    dev = qkey.device
    if hit_off is None:
        hit_off = torch.empty(nq + 1, dtype=torch.uint64, device=dev)
    if d_total is None:
        d_total = torch.zeros(1, dtype=torch.uint64, device=dev)
    if ws is None:
        ws = _ws(seedtable_lookup_workspace_bytes(max(1, nq)), dev)
    _need(qkey, "qkey", torch.uint64, nq)
    _need(d_nq, "d_nq", torch.uint64, 1, allow_none=True)
    _need(hit_off, "hit_off", torch.uint64, nq + 1)
    _need(fp, "fp", torch.uint32, 0)
    _need(pos_tab, "pos_tab", torch.uint64, 0)
    if 1 <= bits <= 30:
        _need(offsets, "offsets", torch.uint64, (1 << bits) + 1)
    if hit_cap is None:
        _check(_st_lk(_ptr(qkey), nq, _ptr(d_nq), k, bits, _ptr(offsets), _ptr(fp), _ptr(pos_tab), _ptr(hit_off),
                      None, 0, _ptr(d_total), _ptr(ws), ws.numel(), _stream(stream)), "seedtable_lookup")
        hit_cap = int(d_total.view(torch.int64).item())
    if hit_pos is None:
        hit_pos = torch.empty(max(1, hit_cap), dtype=torch.uint64, device=dev)
    _need(hit_pos, "hit_pos", torch.uint64, hit_cap)
    _check(_st_lk(_ptr(qkey), nq, _ptr(d_nq), k, bits, _ptr(offsets), _ptr(fp), _ptr(pos_tab), _ptr(hit_off),
                  _ptr(hit_pos), hit_cap, _ptr(d_total), _ptr(ws), ws.numel(), _stream(stream)), "seedtable_lookup")
    return hit_off, hit_pos, d_total


def seedtable_count(hash_: torch.Tensor, k: int, bits: int, *, m: int | None = None, d_m=None, counts=None,
                    stream=None) -> torch.Tensor:
    if m is None:
        m = hash_.numel()
    if counts is None:
        counts = torch.empty(1 << bits, dtype=torch.uint32, device=hash_.device)
    _check(_st_count(_ptr(hash_), m, _ptr(d_m), k, bits, _ptr(counts), _stream(stream)), "seedtable_count")
    return counts


def seedtable_partition(hash_: torch.Tensor, pos: torch.Tensor, k: int, bits: int, nranks: int, *,
                        m: int | None = None, d_m=None, ws=None, stream=None):
    """Returns (send_fp[m], send_pos[m], send_counts[nranks]) grouped by owner rank."""
    if m is None:
        m = hash_.numel()
    dev = hash_.device
    send_fp = torch.empty(max(1, m), dtype=torch.uint32, device=dev)
    send_pos = torch.empty(max(1, m), dtype=torch.uint64, device=dev)
    send_counts = torch.empty(nranks, dtype=torch.uint64, device=dev)
    if ws is None:
        ws = _ws(_st_part_ws(max(1, m), nranks), dev)
    _check(_st_part(_ptr(hash_), _ptr(pos), m, _ptr(d_m), k, bits, nranks, _ptr(send_fp), _ptr(send_pos),
                    _ptr(send_counts), _ptr(ws), ws.numel(), _stream(stream)), "seedtable_partition")
    return send_fp, send_pos, send_counts


def seedtable_partition_p2p(hash_: torch.Tensor, pos: torch.Tensor, k: int, bits: int, peer_fp: list[int],
                            peer_pos: list[int], peer_base: list[int], *, m: int | None = None, d_m=None, ws=None,
                            stream=None, items: torch.Tensor | None = None) -> int:
    """Partition fused with the all-to-all: entries go straight into the owners' receive
    buffers (device pointers, e.g. peer-mapped symmetric memory).  Returns the status code:
    SLSUM_OK, or SLSUM_EUNSUPPORTED when the narrow precondition fails (use the NCCL path).
    With `items` (mz_extract_ex's out_items) the pass reads the packed items instead of hash."""
    if m is None:
        m = hash_.numel()
    nranks = len(peer_fp)
    _need(hash_, "hash", torch.uint64, m)
    _need(pos, "pos", torch.uint64, m)
    _need(items, "items", torch.uint64, m, allow_none=True)
    _need(d_m, "d_m", torch.uint64, 1, allow_none=True)
    if ws is None:
        ws = _ws(_st_p2p_ws(max(1, m), nranks), hash_.device)
    arr = ctypes.c_uint64 * nranks
    if items is not None:
        rc = _st_p2p_it(_ptr(items), _ptr(pos), m, _ptr(d_m), k, bits, nranks, arr(*peer_fp), arr(*peer_pos),
                        arr(*peer_base), _ptr(ws), ws.numel(), _stream(stream))
    else:
        rc = _st_p2p(_ptr(hash_), _ptr(pos), m, _ptr(d_m), k, bits, nranks, arr(*peer_fp), arr(*peer_pos),
                     arr(*peer_base), _ptr(ws), ws.numel(), _stream(stream))
    if rc not in (SLSUM_OK, SLSUM_EUNSUPPORTED):
        _check(rc, "seedtable_partition_p2p")
    return rc


def seedtable_finalize(recv_fp: torch.Tensor, recv_pos: torch.Tensor, m_recv: int, global_counts, bits: int,
                       rank: int, nranks: int, *, with_fp: bool = True, ws=None, stream=None):
    """Returns (offsets_local[2^bits/nranks + 1], pos_out[m_recv], fp_out or None)."""
    dev = recv_pos.device
    nbl = (1 << bits) // nranks
    offsets = torch.empty(nbl + 1, dtype=torch.uint64, device=dev)
    pos_out = torch.empty(max(1, m_recv), dtype=torch.uint64, device=dev)
    fp_out = torch.empty(max(1, m_recv), dtype=torch.uint32, device=dev) if with_fp else None
    if ws is None:
        ws = _ws(_st_fin_ws(max(1, m_recv), bits, nranks), dev)
    _check(_st_fin(_ptr(recv_fp), _ptr(recv_pos), m_recv, _ptr(global_counts), bits, rank, nranks, _ptr(offsets),
                   _ptr(pos_out), _ptr(fp_out), _ptr(ws), ws.numel(), _stream(stream)), "seedtable_finalize")
    return offsets, pos_out, fp_out
