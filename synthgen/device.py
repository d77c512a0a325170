"""Device twin of synthgen/host.py: the same counter-based streams written straight into
device memory (for the 3.1 Gbp / 10 Gbp inputs).  ctypes over libsynthgen.so."""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import host as H

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libsynthgen.so")
        if not os.path.exists(path):
            from .build import build
            build()
        L = ctypes.CDLL(path)
        u64, u32, vp, i32 = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_int
        L.sg_uniform_ascii.argtypes = [vp, u64, u64, u64, vp]
        L.sg_gc_ascii.argtypes = [vp, u64, u64, u64, u32, u32, u32, vp, u64, vp]
        L.sg_reads_ascii.argtypes = [vp, vp, vp, u64, u64, u64, u32, vp]
        L.sg_u32.argtypes = [vp, u64, u64, u64, vp]
        L.sg_f32_table.argtypes = [vp, u64, u64, u64, vp, vp]
        for f in (L.sg_uniform_ascii, L.sg_gc_ascii, L.sg_reads_ascii, L.sg_u32, L.sg_f32_table):
            f.restype = i32
        _LIB = L
    return _LIB


def _s():
    return torch.cuda.current_stream().cuda_stream


def _ok(rc):
    if rc != 0:
        raise RuntimeError(f"synthgen CUDA error {rc}")


def c1_ascii(n: int = 1_000_000, seed: int = H.SEED_C1, lo: int = 0, device="cuda") -> torch.Tensor:
    out = torch.empty(n, dtype=torch.uint8, device=device)
    _ok(lib().sg_uniform_ascii(out.data_ptr(), lo, n, seed, _s()))
    return out


def c3_ascii(c3: "H.C3", lo: int = 0, n: int | None = None, device="cuda", out=None) -> torch.Tensor:
    if n is None:
        n = c3.n - lo
    if out is None:
        out = torch.empty(n, dtype=torch.uint8, device=device)
    iv = torch.from_numpy(np.ascontiguousarray(c3.intervals, dtype=np.int64)).to(device)
    ta, tc, tg = H.GC41_THRESHOLDS
    _ok(lib().sg_gc_ascii(out.data_ptr(), lo, n, c3.seed_bases, ta, tc, tg, iv.data_ptr(), len(c3.intervals), _s()))
    torch.cuda.current_stream().synchronize()
    return out


def c4_ascii(c4: "H.C4", device="cuda", out=None) -> torch.Tensor:
    if out is None:
        out = torch.empty(c4.n, dtype=torch.uint8, device=device)
    ro = torch.from_numpy(c4.read_off).to(device)
    st = torch.from_numpy(c4.starts).to(device)
    _ok(lib().sg_reads_ascii(out.data_ptr(), ro.data_ptr(), st.data_ptr(), c4.nreads, c4.seed_t, c4.seed_sub,
                             H.C4_SUBST_T, _s()))
    torch.cuda.current_stream().synchronize()
    return out


def c4_ascii_reads(c4: "H.C4", r0: int, r1: int, device="cuda") -> torch.Tensor:
    """Bases of reads [r0, r1) of the C4 batch (global positions [read_off[r0], read_off[r1]))."""
    a, b = int(c4.read_off[r0]), int(c4.read_off[r1])
    out = torch.empty(max(1, b - a), dtype=torch.uint8, device=device)
    if r1 > r0:
        ro = torch.from_numpy(c4.read_off[r0:r1 + 1]).to(device)
        st = torch.from_numpy(c4.starts[r0:r1]).to(device)
        # the kernel writes base t of read r at out[read_off[r] + t]: shift the base pointer by -a
        _ok(lib().sg_reads_ascii(out.data_ptr() - a, ro.data_ptr(), st.data_ptr(), r1 - r0, c4.seed_t, c4.seed_sub,
                                 H.C4_SUBST_T, _s()))
        torch.cuda.current_stream().synchronize()
    return out[: b - a]


def c2_u32(n: int, seed: int = H.SEED_C2_U32, lo: int = 0, device="cuda") -> torch.Tensor:
    out = torch.empty(n, dtype=torch.uint32, device=device)
    _ok(lib().sg_u32(out.data_ptr(), lo, n, seed, _s()))
    return out


def c2_f32(n: int, seed: int = H.SEED_C2_F32, lo: int = 0, device="cuda") -> torch.Tensor:
    out = torch.empty(n, dtype=torch.float32, device=device)
    table = torch.from_numpy(H.normal_table()).to(device)
    _ok(lib().sg_f32_table(out.data_ptr(), lo, n, seed, table.data_ptr(), _s()))
    torch.cuda.current_stream().synchronize()
    return out
