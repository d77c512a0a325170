"""CPU-only: the C-ABI library loads and exports every function include/mzslsum.h declares
(no compute calls without a GPU).  Also the header builds as plain C."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "mzslsum.h")
LIB = os.path.join(ROOT, "paper_1811_10074_b200", "libmzslsum.so")


def declared():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:int|size_t|char\s*\*|const char\s*\*)\s*\*?\s*(\w+)\s*\(",
                                 txt, flags=re.M)))


def _ensure_built():
    if not os.path.exists(LIB):
        subprocess.check_call(["python", os.path.join(ROOT, "paper_1811_10074_b200", "build.py")])


def test_every_declared_symbol_is_exported():
    _ensure_built()
    names = declared()
    assert len(names) >= 14, names
    lib = ctypes.CDLL(LIB)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_strerror_and_version_without_gpu():
    _ensure_built()
    lib = ctypes.CDLL(LIB)
    lib.slsum_strerror.restype = ctypes.c_char_p
    assert lib.slsum_strerror(-2) == b"unsupported operator/path/size combination"
    assert lib.slsum_version() > 0


def test_header_is_plain_c(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "mzslsum.h"\nint main(void){ mz_in_t a; mz_out_t b; (void)a; (void)b; return 0; }\n')
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           "-c", str(src), "-o", str(tmp_path / "t.o")])


def test_argument_errors_are_rejected_before_any_launch():
    """EINVAL paths return before touching the device (safe without a GPU)."""
    _ensure_built()
    lib = ctypes.CDLL(LIB)
    lib.slsum_run_ex.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
    assert lib.slsum_run_ex(0, 0, None, None, 10, 0, None) == -1      # w = 0
    assert lib.slsum_run_ex(99, 3, None, None, 10, 0, None) == -1     # bad op
    assert lib.slsum_run_ex(0, 3, None, None, 2, 0, None) == 0        # n < w: zero outputs


def test_binding_rejects_mis_sized_buffers_before_the_abi():
    """The Python binding checks dtypes and sizes before a raw device pointer crosses the ABI
    (the kernels trust them).  The checks run before any device use, so CPU tensors serve."""
    import pytest
    import torch
    P = __import__("paper_1811_10074_b200")
    L = P._lib
    x32 = torch.zeros(100, dtype=torch.uint32)
    with pytest.raises(ValueError, match="dtype|elements|shape"):                     # MIN_U64 on a uint32 tensor
        L.slsum_run(L.SLSUM_MIN_U64, 4, x32)
    with pytest.raises(ValueError, match="dtype|elements|shape"):                     # a pair op on a 1-D tensor
        L.slsum_run(L.SLSUM_AFFINE_U32X2, 4, x32)
    with pytest.raises(ValueError, match="dtype|elements|shape"):                     # y too short
        L.slsum_run(L.SLSUM_MIN_U32, 4, x32, y=torch.zeros(10, dtype=torch.uint32))
    seq = torch.zeros(1000, dtype=torch.uint8)
    with pytest.raises(ValueError, match="dtype|elements|shape"):                     # capacity beyond out_hash
        L.mz_extract_ex(seq, 15, 10, capacity=500, out_hash=torch.zeros(10, dtype=torch.uint64))
    with pytest.raises(ValueError, match="dtype|elements|shape"):                     # items shorter than capacity
        L.mz_extract_ex(seq, 15, 10, capacity=500, out_items=torch.zeros(10, dtype=torch.uint64))
    h = torch.zeros(100, dtype=torch.uint64)
    with pytest.raises(ValueError, match="dtype|elements|shape"):                     # pos shorter than m
        L.seedtable_build(h, torch.zeros(50, dtype=torch.uint64), 19, 24)
    with pytest.raises(ValueError, match="dtype|elements|shape"):                     # items shorter than m
        L.seedtable_build_items(torch.zeros(5, dtype=torch.uint64), h, h, 19, 24)
    with pytest.raises(ValueError, match="dtype|elements|shape"):                     # offsets too short for 2^bits + 1
        L.seedtable_build(h, h, 19, 10, offsets=torch.zeros(1024, dtype=torch.uint64))
