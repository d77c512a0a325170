#!/usr/bin/env python
"""Per-phase cycle profile of the narrow seed-table downsweep (design aid).

    python tools/prof_nsweep.py build     # here: libmzslsum_prof.so with -DMZS_PROF
    python tools/prof_nsweep.py run       # on the GPU box: C3 minimizers -> seed table, phase split
"""
import ctypes
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tools", "libmzslsum_prof.so")


def build():
    srcs = sorted(glob.glob(os.path.join(ROOT, "paper_1811_10074_b200", "csrc", "*.cu")))
    cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
           "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", "--expt-relaxed-constexpr", "-DMZS_PROF",
           "-I", os.path.join(ROOT, "include"), "-shared", "-o", OUT, *srcs, "-lcudart"]
    subprocess.check_call(cmd)
    print(OUT)


def run():
    os.environ["MZS_LIB"] = OUT
    sys.path.insert(0, ROOT)
    import torch
    import paper_1811_10074_b200 as P
    from synthgen import device as SD
    from synthgen import host as H
    lib = ctypes.CDLL(OUT)
    buf = (ctypes.c_ulonglong * 8)()
    k, w, bits = 19, 10, 24
    c3 = H.C3()
    n = c3.n
    seq = SD.c3_ascii(c3, lo=0, n=n, device=torch.device("cuda"))
    words = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device="cuda")
    inval = torch.empty((n + 31) // 32 + 1, dtype=torch.uint32, device="cuda")
    cap = int(0.25 * n)
    oh = torch.empty(cap, dtype=torch.uint64, device="cuda")
    op = torch.empty(cap, dtype=torch.uint64, device="cuda")
    dc = torch.zeros(1, dtype=torch.uint64, device="cuda")
    P.mz_encode(seq, words, inval)
    P.mz_extract_ex(words, k, w, n=n, kind=P.MZ_IN_PACKED2, invalid=inval, capacity=cap, out_hash=oh, out_pos=op,
                    d_count=dc)
    torch.cuda.synchronize()
    m = int(dc.view(torch.int64).item())
    ws = torch.empty(P.seedtable_workspace_bytes(m, bits), dtype=torch.uint8, device="cuda")
    P.seedtable_build(oh[:m], op[:m], k, bits, ws=ws)
    torch.cuda.synchronize()
    lib.seedtable_prof_read(buf, 1)
    P.seedtable_build(oh[:m], op[:m], k, bits, ws=ws)
    torch.cuda.synchronize()
    lib.seedtable_prof_read(buf, 1)
    names = ["tma wait", "rank", "scan", "stage", "write"]
    tot = sum(buf[i] for i in range(5))
    print(f"m = {m}; thread-0 cycles per phase, summed over CTAs and the 3 passes:")
    for i, nm in enumerate(names):
        print(f"  {nm:9s} {buf[i] / 1e9:8.3f} Gclk  {buf[i] / tot * 100:5.1f}%")


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
