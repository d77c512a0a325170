"""Time the C3 minimizer kernel alone (bench.py's launch: PACKED2 input + invalid bitmap, device
count, packed items) with CUDA events; print median/best ms and a checksum of the records so
that library variants (MZS_LIB=...) can be compared.  Usage: python tools/mz_c3.py [reps] [k]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_10074_b200 as P
from synthgen import device as SD
from synthgen import host as H

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
k = int(sys.argv[2]) if len(sys.argv) > 2 else 19
w = 10
c3 = H.C3()
n = c3.n
seq = SD.c3_ascii(c3)
nw = (n + 31) // 32
words = torch.empty(nw + 1, dtype=torch.uint64, device="cuda")
inval = torch.empty(nw + 1, dtype=torch.uint32, device="cuda")
P.mz_encode(seq, words, inval)
del seq
cap = int(0.25 * (n - k - w + 2)) + 1024
h = torch.empty(cap, dtype=torch.uint64, device="cuda")
p = torch.empty(cap, dtype=torch.uint64, device="cuda")
items = torch.empty(cap, dtype=torch.uint64, device="cuda")
c = torch.zeros(1, dtype=torch.uint64, device="cuda")
ws = torch.empty(P.mz_workspace_bytes(n, k, w, P.MZ_IN_PACKED2), dtype=torch.uint8, device="cuda")


def run():
    P.mz_extract_ex(words, k, w, n=n, kind=P.MZ_IN_PACKED2, invalid=inval, capacity=cap, out_hash=h, out_pos=p,
                    d_count=c, ws=ws, out_items=items)


for _ in range(3):
    run()
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
m = int(c.item())
mix = (h[:m].view(torch.int64) * 0x9E3779B97F4A7C15 + p[:m].view(torch.int64) * 31 + items[:m].view(torch.int64)).sum().item()
print(f"{os.path.basename(os.environ.get('MZS_LIB', 'libmzslsum.so'))} k={k} m={m} mz ms: median "
      f"{sorted(ts)[len(ts) // 2]:.3f} best {min(ts):.3f} checksum {mix & 0xFFFFFFFFFFFFFFFF:016x}", flush=True)
