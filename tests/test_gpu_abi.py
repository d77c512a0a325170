"""The BASELINE-shape synchronous entry points, called through ctypes exactly as
include/mzslsum.h declares them (not through the Python binding):
  slsum_run(op, w, x, y, n)           Eq. 2, GENERIC path, default stream
  mz_extract(seq, n, k, w, out)       minimizers (L85, Fig. 2), ASCII in, hashed keys
and mz_extract_ex / mz_extract_path with a hand-built mz_in_t / mz_out_t.  Each is compared
with the oracle; mz_extract's SLSUM_ECAPACITY contract (the count is still reported, the first
`capacity` records are valid) is checked too."""
import ctypes

import numpy as np
import pytest
import torch

import oracle as O
from synthgen import host as G

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1811_10074_b200")
L = P._lib

u64, i32, u32, vp = ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p


def _lib():
    lib = ctypes.CDLL(L.LIB_PATH)
    lib.slsum_run.argtypes = [i32, u32, vp, vp, u64]
    lib.slsum_run.restype = i32
    lib.mz_extract.argtypes = [vp, u64, i32, i32, ctypes.POINTER(L.MzOut)]
    lib.mz_extract.restype = i32
    lib.mz_extract_ex.argtypes = [ctypes.POINTER(L.MzIn), i32, i32, i32, ctypes.POINTER(L.MzOut), vp,
                                  ctypes.c_size_t, vp]
    lib.mz_extract_ex.restype = i32
    lib.mz_extract_path.argtypes = [ctypes.POINTER(L.MzIn), i32, i32, i32, ctypes.POINTER(L.MzOut), vp,
                                    ctypes.c_size_t, vp, i32]
    lib.mz_extract_path.restype = i32
    lib.mz_workspace_bytes.argtypes = [u64, i32, i32, i32]
    lib.mz_workspace_bytes.restype = ctypes.c_size_t
    return lib


@pytest.mark.parametrize("op,w", [(0, 10), (1, 7), (2, 64), (3, 16), (5, 33)])
def test_slsum_run_declared_signature(op, w):
    lib = _lib()
    rng = np.random.default_rng(op * 100 + w)
    n = 300_001
    if op == 3:
        x = rng.standard_normal(n).astype(np.float32)
    elif op == 5:
        x = rng.integers(0, 2 ** 63, size=n, dtype=np.uint64)
    else:
        x = rng.integers(0, 2 ** 32, size=n, dtype=np.uint64).astype(np.uint32)
    xt = torch.from_numpy(x).cuda()
    yt = torch.empty(n - w + 1, dtype=xt.dtype, device="cuda")
    torch.cuda.synchronize()
    assert lib.slsum_run(op, w, xt.data_ptr(), yt.data_ptr(), n) == 0    # synchronous: no sync needed
    want = O.slsum(op, w, x)
    got = yt.cpu().numpy()
    if op == 3:
        assert np.all(np.abs(got.astype(np.float64) - want) <= 1e-5 * np.abs(want) + 1e-6 * w)
    else:
        assert np.array_equal(got, want)
    assert lib.slsum_run(op, 0, xt.data_ptr(), yt.data_ptr(), n) == L.SLSUM_EINVAL
    assert lib.slsum_run(op, n + 1, xt.data_ptr(), yt.data_ptr(), n) == 0   # n < w: zero outputs


def test_mz_extract_declared_signature_and_capacity():
    lib = _lib()
    c3 = G.C3(n=600_000, mean_run=2_000.0, n_frac=0.02)
    seq = c3.ascii()
    n, k, w = len(seq), 19, 10
    want_k, want_p = O.mz(seq, k, w)
    m = len(want_p)
    st = torch.from_numpy(seq).cuda()
    cap = m + 100
    h = torch.empty(cap, dtype=torch.uint64, device="cuda")
    p = torch.empty(cap, dtype=torch.uint64, device="cuda")
    d = torch.zeros(1, dtype=torch.uint64, device="cuda")
    out = L.MzOut(h.data_ptr(), p.data_ptr(), cap, d.data_ptr(), None)
    torch.cuda.synchronize()
    assert lib.mz_extract(st.data_ptr(), n, k, w, ctypes.byref(out)) == 0
    assert int(d.item()) == m
    assert np.array_equal(p[:m].cpu().numpy(), want_p) and np.array_equal(h[:m].cpu().numpy(), want_k)
    # capacity too small: SLSUM_ECAPACITY, the full count in d_count, the first `capacity` records valid
    small = m // 3
    h.fill_(0)
    out = L.MzOut(h.data_ptr(), p.data_ptr(), small, d.data_ptr(), None)
    assert lib.mz_extract(st.data_ptr(), n, k, w, ctypes.byref(out)) == L.SLSUM_ECAPACITY
    assert int(d.item()) == m
    assert np.array_equal(p[:small].cpu().numpy(), want_p[:small])
    assert np.array_equal(h[:small].cpu().numpy(), want_k[:small])
    assert not bool(h[small:].view(torch.int64).any())                 # nothing written past capacity
    # degenerate: shorter than k + w - 1 -> 0 records, OK
    out = L.MzOut(h.data_ptr(), p.data_ptr(), cap, d.data_ptr(), None)
    assert lib.mz_extract(st.data_ptr(), k + w - 2, k, w, ctypes.byref(out)) == 0 and int(d.item()) == 0
    assert lib.mz_extract(st.data_ptr(), n, 0, w, ctypes.byref(out)) == L.SLSUM_EINVAL


@pytest.mark.parametrize("path", [0, 1])
def test_mz_extract_ex_and_path_declared_structs(path):
    """mz_extract_ex (path 0, the automatic kernel) and mz_extract_path (1: the generic kernel)
    with hand-built structs, packed input with the invalid bitmap, reads and a window range."""
    lib = _lib()
    rng = np.random.default_rng(7 + path)
    n, k, w = 400_000, 15, 10
    seq = np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, size=n)].copy()
    seq[rng.random(n) < 0.002] = ord("N")
    ro = np.unique(np.concatenate([[0, n], rng.integers(1, n, size=30)])).astype(np.uint64)
    a = 50_000
    want_k, want_p = O.mz(seq, k, w, read_off=ro, pos_base=1000, win_lo=a, win_hi=n)
    words, inval = O.pack(seq)
    wt, it = torch.from_numpy(words).cuda(), torch.from_numpy(inval).cuda()
    rt = torch.from_numpy(ro).cuda()
    cap = len(want_p) + 64
    h = torch.empty(cap, dtype=torch.uint64, device="cuda")
    p = torch.empty(cap, dtype=torch.uint64, device="cuda")
    d = torch.zeros(1, dtype=torch.uint64, device="cuda")
    ws = torch.empty(lib.mz_workspace_bytes(n, k, w, L.MZ_IN_PACKED2), dtype=torch.uint8, device="cuda")
    mi = L.MzIn(L.MZ_IN_PACKED2, wt.data_ptr(), it.data_ptr(), n, rt.data_ptr(), len(ro) - 1, 1000, a, 2 ** 64 - 1)
    mo = L.MzOut(h.data_ptr(), p.data_ptr(), cap, d.data_ptr(), None)
    s = torch.cuda.current_stream().cuda_stream
    if path == 0:
        rc = lib.mz_extract_ex(ctypes.byref(mi), k, w, L.MZ_KEY_HASH, ctypes.byref(mo), ws.data_ptr(), ws.numel(), s)
    else:
        rc = lib.mz_extract_path(ctypes.byref(mi), k, w, L.MZ_KEY_HASH, ctypes.byref(mo), ws.data_ptr(),
                                 ws.numel(), s, path)
    assert rc == 0
    torch.cuda.synchronize()
    m = int(d.item())
    assert m == len(want_p)
    assert np.array_equal(p[:m].cpu().numpy(), want_p) and np.array_equal(h[:m].cpu().numpy(), want_k)
