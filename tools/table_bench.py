"""Time the seed table of the C3 bench step alone (seedtable_build_items on the C3 minimizer
items, as bench.py builds it), with CUDA events, and print a checksum of the table so that two
configurations (e.g. MZS_LB=0 / 1) can be compared.  Usage: python tools/table_bench.py [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_10074_b200 as P
from synthgen import device as SD
from synthgen import host as H

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
k, w, bits = 19, 10, 24
c3 = H.C3()
n = c3.n
seq = SD.c3_ascii(c3)
nw = (n + 31) // 32
words = torch.empty(nw + 1, dtype=torch.uint64, device="cuda")
inval = torch.empty(nw + 1, dtype=torch.uint32, device="cuda")
P.mz_encode(seq, words, inval)
del seq
cap = int(0.25 * (n - k - w + 2)) + 1024
items = torch.empty(cap, dtype=torch.uint64, device="cuda")
fused = os.environ.get("MZS_FUSED_HIST", "1") != "0"   # the first pass's counts from the minimizer kernel
hist = torch.empty(P.seedtable_hist_words(cap, bits), dtype=torch.uint32, device="cuda") if fused else None
h, p, c = P.mz_extract_ex(words, k, w, n=n, kind=P.MZ_IN_PACKED2, invalid=inval, capacity=cap, out_items=items,
                          out_hist=hist, hist_bits=bits)
ws = torch.empty(P.seedtable_workspace_bytes(cap, bits), dtype=torch.uint8, device="cuda")
off = torch.empty((1 << bits) + 1, dtype=torch.uint64, device="cuda")
pos32 = os.environ.get("MZS_TB_POS32", "0") == "1"   # bench.py's table: 32-bit positions
po = torch.empty(cap, dtype=torch.uint32 if pos32 else torch.uint64, device="cuda")
fp = torch.empty(cap, dtype=torch.uint32, device="cuda")


def run():
    P.seedtable_build_items_ex(items, h, p, k, bits, m=cap, d_m=c, hist=hist, offsets=off, pos_out=po, fp_out=fp,
                               ws=ws, pos32=pos32)


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
pv = po[:m].view(torch.int32).to(torch.int64) if pos32 else po[:m].view(torch.int64)
mix = (pv * 0x9E3779B97F4A7C15 + fp[:m].view(torch.int32).to(torch.int64)).sum().item()
print(f"fused_hist={int(fused)} pos32={int(pos32)} ncfg={os.environ.get('MZS_NCFG', '-')}/{os.environ.get('MZS_NCFG_LAST', '-')} m={m} table ms: median {sorted(ts)[len(ts) // 2]:.3f} best {min(ts):.3f} "
      f"checksum {mix & 0xFFFFFFFFFFFFFFFF:016x} off_last {int(off[-1].item())}", flush=True)
