"""Seed table of the C4 minimizers (1.88e9 entries, positions spanning 1e10 > 2^32, so the
wide radix path): build time and a sampled check of the pointer table."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1811_10074_b200 as P  # noqa: E402
from synthgen import device as SD  # noqa: E402
from synthgen import host as H  # noqa: E402

c4 = H.C4()
n = c4.n
seq = SD.c4_ascii(c4)
ro = torch.from_numpy(c4.read_off.astype(np.int64)).cuda().view(torch.uint64)
words, inval = P.mz_encode(seq)
del seq
cap = int(0.2 * n)
h, p, c = P.mz_extract_ex(words, 15, 10, n=n, kind=P.MZ_IN_PACKED2, invalid=inval, read_off=ro, capacity=cap)
torch.cuda.synchronize()
m = int(c.view(torch.int64).item())
del words, inval
print("records", m)
bits = 24
ws = torch.empty(P.seedtable_workspace_bytes(m, bits), dtype=torch.uint8, device="cuda")
off = torch.empty((1 << bits) + 1, dtype=torch.uint64, device="cuda")
po = torch.empty(m, dtype=torch.uint64, device="cuda")
fo = torch.empty(m, dtype=torch.uint32, device="cuda")
hh, pp = h[:m], p[:m]
for rep in range(4):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    P.seedtable_build(hh, pp, 15, bits, offsets=off, pos_out=po, fp_out=fo, ws=ws)
    b.record()
    torch.cuda.synchronize()
    print(f"build {a.elapsed_time(b):.2f} ms  ({m / a.elapsed_time(b) / 1e6:.2f} G entries/s)")
o = off.view(torch.int64)
assert int(o[0]) == 0 and int(o[-1]) == m and bool((o[1:] >= o[:-1]).all())
# sampled buckets: entries in bucket order, positions ascending within each
rng = np.random.default_rng(0)
for bk in rng.integers(0, 1 << bits, size=200):
    lo_, hi_ = int(o[bk]), int(o[bk + 1])
    if hi_ > lo_:
        f = fo[lo_:hi_].view(torch.int32).cpu().numpy().view(np.uint32)
        assert np.all((f >> 8) == bk)
        ps = po[lo_:hi_].view(torch.int64).cpu().numpy()
        assert np.all(np.diff(ps) > 0)
print("sampled checks ok")
