"""Time mz_extract_ex on the C4 input with and without the read offsets (how much the read
starts cost), and on C1-style uniform bases at C4 size."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1811_10074_b200 as P  # noqa: E402
from synthgen import device as SD  # noqa: E402
from synthgen import host as H  # noqa: E402


def timeit(f, reps=5):
    f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


c4 = H.C4()
n = c4.n
seq = SD.c4_ascii(c4)
ro = torch.from_numpy(c4.read_off.astype(np.int64)).cuda().view(torch.uint64)
nw = (n + 31) // 32
words = torch.empty(nw + 1, dtype=torch.uint64, device="cuda")
inval = torch.empty(nw + 1, dtype=torch.uint32, device="cuda")
P.mz_encode(seq, words, inval)
cap = int(0.21 * n) + 1024
oh = torch.empty(cap, dtype=torch.uint64, device="cuda")
op = torch.empty(cap, dtype=torch.uint64, device="cuda")
dc = torch.zeros(1, dtype=torch.uint64, device="cuda")
ws = torch.empty(P.mz_workspace_bytes(n, 15, 10, P.MZ_IN_PACKED2), dtype=torch.uint8, device="cuda")
for name, kw in (("reads", dict(read_off=ro)), ("no_reads", {})):
    ms = timeit(lambda: P.mz_extract_ex(words, 15, 10, n=n, kind=P.MZ_IN_PACKED2, invalid=inval, capacity=cap,
                                        out_hash=oh, out_pos=op, d_count=dc, ws=ws, **kw))
    print(name, f"{ms:.2f} ms", f"{n / ms / 1e6:.1f} Gbases/s", int(dc.view(torch.int64).item()))
