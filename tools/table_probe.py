"""Probe: build a seed table of m random 38-bit keys on the GPU, check its invariants at
full size (offsets monotone, offsets[-1] = m, bucket(fp) inside [offsets[b], offsets[b+1]),
positions ascending inside buckets), and time the call."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1811_10074_b200 as P

m = int(sys.argv[1]) if len(sys.argv) > 1 else 557_847_913
k, bits = 19, 24
g = torch.Generator(device="cuda").manual_seed(1)
h = torch.randint(0, 1 << 38, (m,), device="cuda", dtype=torch.int64, generator=g).view(torch.uint64)
pos = (torch.arange(m, device="cuda", dtype=torch.int64) * 5).view(torch.uint64)
ws = torch.empty(P.seedtable_workspace_bytes(m, bits), dtype=torch.uint8, device="cuda")
off = torch.empty((1 << bits) + 1, dtype=torch.uint64, device="cuda")
po = torch.empty(m, dtype=torch.uint64, device="cuda")
fp = torch.empty(m, dtype=torch.uint32, device="cuda")
for it in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    P.seedtable_build(h, pos, k, bits, offsets=off, pos_out=po, fp_out=fp, ws=ws)
    torch.cuda.synchronize()
    print("build ms", (time.perf_counter() - t) * 1e3, flush=True)
o = off.view(torch.int64)
assert int(o[0]) == 0 and int(o[-1]) == m, (int(o[0]), int(o[-1]))
assert bool((o[1:] >= o[:-1]).all())
b = (fp.view(torch.int32).to(torch.int64) & 0xFFFFFFFF) >> 8
assert bool((b[1:] >= b[:-1]).all()), "fingerprints not sorted by bucket"
idx = torch.arange(m, device="cuda")
assert bool((o[b] <= idx).all()) and bool((idx < o[b + 1]).all())
p = po.view(torch.int64)
same = b[1:] == b[:-1]
assert bool((p[1:][same] > p[:-1][same]).all()), "positions not ascending in bucket"
print("table invariants OK", flush=True)
