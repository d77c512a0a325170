"""Quick GPU check of seedtable_build on a few shapes (debug aid; prints progress)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import oracle as O
import paper_1811_10074_b200 as P

def run(m, span, k=19, bits=24, seed=0):
    rng = np.random.default_rng(seed)
    key = rng.integers(0, 1 << (2 * k), size=m, dtype=np.uint64)
    pos = np.sort(rng.choice(span, size=m, replace=False)).astype(np.uint64)
    t = time.time()
    off, po, fp = P.seedtable_build(torch.from_numpy(key).cuda(), torch.from_numpy(pos).cuda(), k, bits)
    torch.cuda.synchronize()
    wo, wf, wp = O.seedtable(key, pos, k, bits)
    ok = np.array_equal(off.cpu().numpy(), wo) and np.array_equal(po[:m].cpu().numpy(), wp) and np.array_equal(fp[:m].cpu().numpy(), wf)
    print(f"m={m} span={span} ok={ok} {time.time()-t:.2f}s", flush=True)

for m, span in [(1, 10), (7, 100), (4097, 10**6), (4097, 10**11), (300001, 10**7), (300001, 10**11)]:
    run(m, span)
