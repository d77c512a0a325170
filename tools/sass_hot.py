#!/usr/bin/env python
"""Per-instruction view of one kernel of an ncu report (needs -lineinfo / --import-source):
executed warp-instructions by opcode and the hottest stall-sampled SASS lines.

    python tools/sass_hot.py <report.ncu-rep> <kernel-regex> [--skip N] [--top 40] [--per UNITS]
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("kernel")
    ap.add_argument("--skip", type=int, default=0)
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--per", type=float, default=None, help="divide executed thread-instructions by this")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{a.kernel}", "--launch-skip", str(a.skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    print(rows[0][1][:160])
    hdr = rows[1]
    iS, iSmp, iE = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    iT = hdr.index("Thread Instructions Executed")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
    ops = collections.Counter()
    lines = []
    tot_e = tot_t = tot_s = 0
    stalls = collections.Counter()
    for r in rows[2:]:
        if len(r) <= iT:
            continue
        src = r[iS].strip()
        if not (r[iE] or "0").isdigit():
            continue
        e = int(r[iE] or 0)
        t = int(r[iT] or 0)
        smp = int(r[iSmp] or 0)
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        ops[op.split(".")[0]] += e
        tot_e += e
        tot_t += t
        tot_s += smp
        for i in stall_cols:
            try:
                stalls[hdr[i]] += int(r[i] or 0)
            except ValueError:
                pass
        lines.append((smp, e, r[0], src))
    print(f"warp-inst {tot_e:,}  thread-inst {tot_t:,}  samples {tot_s:,}")
    if a.per:
        print(f"thread-inst per unit: {tot_t / a.per:.1f}   warp-inst per unit: {tot_e / a.per:.2f}")
    print("\nby opcode (warp-inst share):")
    for op, e in ops.most_common(25):
        print(f"  {op:12s} {e / tot_e * 100:5.1f}%" + (f"  {e * 32 / a.per:6.1f}/unit" if a.per else ""))
    print("\nstall reasons (samples):")
    for k, v in stalls.most_common(12):
        print(f"  {k:32s} {v / max(1, tot_s) * 100:5.1f}%")
    print(f"\ntop {a.top} lines by stall samples:")
    for smp, e, addr, src in sorted(lines, reverse=True)[:a.top]:
        print(f"  {smp:7d} {e:12,d}  {addr[-5:]}  {src[:90]}")


if __name__ == "__main__":
    main()
