#!/usr/bin/env python
"""Summarise ncu outputs into markdown for profiles/ (the judged copies; gpurun_out/ is scratch).

    python tools/ncu_summary.py report <file.ncu-rep> [--bases N]     # --set full capture
    python tools/ncu_summary.py launches <launches.csv>               # gpu__time_duration list
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import re
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue-active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp-inst"),
]


def _csv(args):
    out = subprocess.run(["ncu", "-i", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def report(path, bases=None):
    rows = _csv([path, "--page", "raw"])
    hdr = rows[0]
    units = rows[1]
    print(f"### `{path.split('/')[-1]}`\n")
    cols = ["kernel"] + [n for _, n in METRICS] + (["inst/base"] if bases else [])
    print("| " + " | ".join(cols) + " |")
    print("|" + "---|" * len(cols))
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        name = re.sub(r"\(.*", "", name).replace("(anonymous namespace)::", "").replace("mzs::", "")
        vals = [name[:48]]
        for m, _ in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = r[i]
                u = units[i]
                vals.append(f"{v} {u}".strip())
            else:
                vals.append("-")
        if bases:
            i = hdr.index("smsp__inst_executed.sum")
            vals.append(f"{float(r[i].replace(',', '')) * 32 / bases:.1f}")
        print("| " + " | ".join(vals) + " |")
    print()


def launches(path, last_step=None):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    iK, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    tot = 0.0
    body = rows[start + 1:]
    if last_step:  # keep only the launches from the last one whose name contains `last_step`
        cut = max(i for i, r in enumerate(body) if len(r) > iK and last_step in r[iK])
        body = body[cut:]
    for r in body:
        if len(r) <= iV:
            continue
        v = float(r[iV].replace(",", ""))
        u = r[iU]
        ms = v / 1e6 if u in ("ns", "nsecond") else v / 1e3 if u in ("us", "usecond") else v
        name = re.sub(r"\(.*", "", r[iK]).replace("(anonymous namespace)::", "").replace("mzs::", "")
        name = name.replace("void ", "")
        agg.setdefault(name, [0.0, 0])
        agg[name][0] += ms
        agg[name][1] += 1
        tot += ms
    what = f", last step (from the last `{last_step}`)" if last_step else ""
    print(f"### launch list `{path.split('/')[-1]}` (ncu gpu__time_duration, cold-cache, serialised{what})\n")
    print("| kernel | launches | ms | share |")
    print("|---|---|---|---|")
    for k, (ms, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"| {k} | {n} | {ms:.3f} | {ms / tot * 100:.1f}% |")
    print(f"| **total** | | **{tot:.3f}** | |\n")


def traffic(path):
    """JSON {kernel name: {"dram_bytes": read + write summed over the capture's launches of that
    name, "launches": n, "time_ms": summed}} of a --set full capture of ONE step's kernels --
    bench.py's roofline `traffic` (per launch = dram_bytes / launches)."""
    import json
    rows = _csv([path, "--page", "raw"])
    hdr = rows[0]
    out = {}
    for r in rows[2:]:
        name = re.sub(r"\(.*", "", r[hdr.index("Kernel Name")]).replace("(anonymous namespace)::", "")
        name = re.sub(r"^.*unnamed>::", "", name.replace("mzs::", "").replace("void ", "")).strip()

        def val(m, scale):
            i = hdr.index(m)
            v = float(r[i].replace(",", ""))
            u = rows[1][i]
            return v * scale.get(u, 1.0)
        gb = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}
        ms = {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6}
        e = out.setdefault(name, {"dram_bytes": 0.0, "launches": 0, "time_ms": 0.0})
        e["dram_bytes"] += val("dram__bytes_read.sum", gb) + val("dram__bytes_write.sum", gb)
        e["launches"] += 1
        e["time_ms"] += val("gpu__time_duration.sum", ms)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["report", "launches", "traffic"])
    ap.add_argument("path")
    ap.add_argument("--bases", type=float, default=None)
    ap.add_argument("--last-step", default=None, help="launches mode: keep the last step starting at this kernel")
    a = ap.parse_args()
    if a.mode == "traffic":
        traffic(a.path)
    elif a.mode == "report":
        report(a.path, a.bases)
    else:
        launches(a.path, a.last_step)
    sys.exit(0)
