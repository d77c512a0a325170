"""Run ONE C2 sliding-sum configuration a fixed number of times (for ncu captures whose kernel
must be unambiguous): `python tools/slsum_one.py --op min --w 16 --path generic --reps 4`
launches exactly `reps` slsum kernels (C2 input, 2^28 elements), so `ncu -k regex:slsum
-s <reps-1> -c 1` captures the last, warm launch of the named configuration."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1811_10074_b200 as P  # noqa: E402
from synthgen import device as D  # noqa: E402

OPS = {"min": P.SLSUM_MIN_U32, "add": P.SLSUM_ADD_U32, "addf": P.SLSUM_ADD_F32}
PATHS = {"generic": P.SLSUM_PATH_GENERIC, "commutative": P.SLSUM_PATH_COMMUTATIVE,
         "recurrent": P.SLSUM_PATH_RECURRENT, "scalar": P.SLSUM_PATH_SCALAR}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--op", choices=list(OPS), default="min")
    ap.add_argument("--w", type=int, default=16)
    ap.add_argument("--path", choices=list(PATHS), default="generic")
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--n", type=int, default=1 << 28)
    a = ap.parse_args()
    x = D.c2_f32(a.n) if a.op == "addf" else D.c2_u32(a.n)
    y = torch.empty(a.n - a.w + 1, dtype=x.dtype, device="cuda")
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    P.slsum_run(OPS[a.op], a.w, x, y=y, path=PATHS[a.path])
    t0.record()
    for _ in range(a.reps - 1):
        P.slsum_run(OPS[a.op], a.w, x, y=y, path=PATHS[a.path])
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / max(1, a.reps - 1)
    print(f"ok {a.op} w={a.w} {a.path} x{a.reps}: {ms:.3f} ms/run, {a.n / ms / 1e6:.1f} Gelem/s, "
          f"{8 * a.n / ms / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
