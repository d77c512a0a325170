"""Small launches of every kernel family for compute-sanitizer (racecheck / synccheck /
memcheck): the fast and the generic minimizer kernels (clean, N-runs, reads), the narrow
(packed items) and wide (positions spanning >= 2^32) seed-table passes, the fused p2p
partition, lookup, and the slsum generic / lane-tiled / CTA / doubling / recurrent / scalar
kernels.  Each result is checked against the oracle so a silent corruption also fails.
Run:  compute-sanitizer --tool racecheck python tools/sanitize_cases.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
import paper_1811_10074_b200 as P
from synthgen import host as H


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check(name, ok):
    print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        raise SystemExit(1)


rng = np.random.default_rng(5)
# ---- minimizers: fast kernel (k=19 and 15, w=10), generic kernel (w=37), N-runs and reads
c3 = H.C3(n=120_000, mean_run=500.0, n_frac=0.05)
seq = c3.ascii()
for k, w, path in ((19, 10, 0), (15, 10, 0), (19, 10, 1), (21, 37, 0)):
    h, p = P.mz_extract(dev(seq), k, w, path=path)
    wk, wp = O.mz(seq, k, w)
    check(f"mz k={k} w={w} path={path}", np.array_equal(p.cpu().numpy(), wp) and np.array_equal(h.cpu().numpy(), wk))
ro = np.unique(np.concatenate([[0, len(seq)], rng.integers(1, len(seq), size=40)])).astype(np.uint64)
for path in (0, 1):
    h, p = P.mz_extract(dev(seq), 15, 10, read_off=dev(ro), path=path)
    wk, wp = O.mz(seq, 15, 10, read_off=ro)
    check(f"mz reads path={path}", np.array_equal(p.cpu().numpy(), wp))
# ---- seed table: narrow (items and hash/pos) and wide (span >= 2^32)
key, pos = O.mz(seq, 19, 10)
wo, wf, wpt = O.seedtable(key, pos, 19, 24)
off, po, fp = P.seedtable_build(dev(key), dev(pos), 19, 24)
check("seedtable narrow", np.array_equal(off.cpu().numpy(), wo) and np.array_equal(po.cpu().numpy(), wpt))
fpk = np.array([O.fingerprint(int(x), 19) for x in key], np.uint64)
it = dev((fpk << np.uint64(32)) | (pos & np.uint64(0xFFFFFFFF)))
off, po, fp = P.seedtable_build_items(it, dev(key), dev(pos), 19, 24)
check("seedtable items", np.array_equal(off.cpu().numpy(), wo) and np.array_equal(po.cpu().numpy(), wpt))
wide = pos * np.uint64(1 << 20)
wo2, wf2, wp2 = O.seedtable(key, wide, 19, 24)
off, po, fp = P.seedtable_build(dev(key), dev(wide), 19, 24)
check("seedtable wide", np.array_equal(off.cpu().numpy(), wo2) and np.array_equal(po.cpu().numpy(), wp2))
# ---- multi-GPU phases (one process): partition and finalize for 2 owners, fused p2p into local buffers
fp2, pp2, cnt = P.seedtable_partition(dev(key), dev(pos), 19, 24, 2)
check("partition", int(cnt.cpu().numpy().sum()) == len(key))
m = len(key)
bufs_fp = [torch.empty(m, dtype=torch.uint32, device="cuda") for _ in range(2)]
bufs_pos = [torch.empty(m, dtype=torch.uint64, device="cuda") for _ in range(2)]
rc = P.seedtable_partition_p2p(dev(key), dev(pos), 19, 24, [b.data_ptr() for b in bufs_fp],
                               [b.data_ptr() for b in bufs_pos], [0, 0])
check("partition p2p", rc == 0)
# ---- lookup
ho, hp, tot = P.seedtable_lookup(dev(key[:3000]), 19, 24, dev(wo), dev(wf), dev(wpt))
lo, lp = O.lookup(key[:3000], 19, 24, wo, wf, wpt)
check("lookup", np.array_equal(ho.cpu().numpy(), lo) and np.array_equal(hp[: len(lp)].cpu().numpy(), lp))
# ---- sliding sums: every kernel family
x = rng.integers(0, 2 ** 32, size=200_003, dtype=np.uint64).astype(np.uint32)
xt = dev(x)
for w in (4, 10, 16, 33, 64, 100, 256, 1024):
    for path in (P.SLSUM_PATH_GENERIC, P.SLSUM_PATH_COMMUTATIVE):
        y = P.slsum_run(P.SLSUM_MIN_U32, w, xt, path=path)
        check(f"slsum min w={w} path={path}", np.array_equal(y.cpu().numpy(), O.slsum(O.MIN_U32, w, x)))
for w in (10, 300):
    y = P.slsum_run(P.SLSUM_ADD_U32, w, xt, path=P.SLSUM_PATH_RECURRENT)
    check(f"slsum recurrent w={w}", np.array_equal(y.cpu().numpy(), O.slsum(O.ADD_U32, w, x)))
    y = P.slsum_run(P.SLSUM_ADD_U32, w, xt[:20_000], path=P.SLSUM_PATH_SCALAR)
    check(f"slsum scalar w={w}", np.array_equal(y.cpu().numpy(), O.slsum(O.ADD_U32, w, x[:20_000])))
xa = rng.integers(0, 2 ** 32, size=(50_001, 2), dtype=np.uint64).astype(np.uint32)
y = P.slsum_run(P.SLSUM_AFFINE_U32X2, 24, dev(xa))
check("slsum affine w=24", np.array_equal(y.cpu().numpy(), O.slsum(O.AFFINE_U32X2, 24, xa)))
torch.cuda.synchronize()
print("all cases ok", flush=True)
