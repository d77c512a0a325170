#!/usr/bin/env python
"""Per-CUDA-source-line instruction and stall attribution of one kernel of an ncu report
(needs -lineinfo and --import-source on).

    python tools/src_hot.py <report.ncu-rep> <kernel-regex> [--skip N] [--per UNITS] [--top 40]
"""
from __future__ import annotations

import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("kernel")
    ap.add_argument("--skip", type=int, default=0)
    ap.add_argument("--per", type=float, default=1.0)
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--by-stall", action="store_true", help="sort by stall samples instead of instructions")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          f"regex:{a.kernel}", "--launch-skip", str(a.skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname = "?"
    hdr = None
    agg = []
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) > 3 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or r[2] != "-":
            continue
        try:
            ti = int(r[hdr.index("Thread Instructions Executed")] or 0)
            smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        if ti or smp:
            agg.append((ti, smp, f"{fname}:{r[0]}", r[1].strip()))
    tot_i = sum(x[0] for x in agg)
    tot_s = sum(x[1] for x in agg) or 1
    print(f"thread-inst {tot_i:,} = {tot_i / a.per:.1f} per unit")
    print(f"{'inst/unit':>9} {'inst%':>6} {'stall%':>6}  line")
    key = (lambda x: x[1]) if a.by_stall else (lambda x: x[0])
    for ti, smp, loc, src in sorted(agg, key=key, reverse=True)[:a.top]:
        print(f"{ti / a.per:9.2f} {ti / tot_i * 100:6.1f} {smp / tot_s * 100:6.1f}  {loc:18s} {src[:80]}")


if __name__ == "__main__":
    main()
