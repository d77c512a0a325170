"""Per-opcode SASS summary of one kernel's ncu source page (instructions, shared-memory L1
wavefronts, global L1 tag requests, L2 sectors, stall samples), per `unit` items:
    ncu -i rep --page source --csv --print-source sass --kernel-name-base demangled -k regex:K --launch-count 1 > s.csv
    python tools/sass_l1.py s.csv <units> [per]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2])
per = float(sys.argv[3]) if len(sys.argv) > 3 else 32.0
hdr = None
data = []
for r in rows:
    if len(r) > 3 and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = collections.Counter()
for d in data:
    t = d["Source"].strip().split()
    op = t[1] if t[0].startswith("@") else t[0]
    op = ".".join(op.split(".")[:2]) if op.startswith(("ATOMS", "LDS", "STS", "STG", "LDG")) else op.split(".")[0]
    for key, col in (("wf", "L1 Wavefronts Shared"), ("ideal", "L1 Wavefronts Shared Ideal"),
                     ("inst", "Instructions Executed"), ("samp", "Warp Stall Sampling (All Samples)"),
                     ("tag", "L1 Tag Requests Global"), ("l2s", "L2 Theoretical Sectors Global")):
        tot[(op, key)] += f(d.get(col, "0"))
ops = sorted(set(k[0] for k in tot), key=lambda o: -tot[(o, "samp")])
S = sum(tot[(o, "samp")] for o in ops) or 1
W = sum(tot[(o, "wf")] for o in ops)
I = sum(tot[(o, "inst")] for o in ops)
print(f"per {per:g} units: {'op':12s} {'inst':>7s} {'smem wf':>8s} {'ideal':>7s} {'g tags':>7s} {'L2 sec':>7s} {'samp%':>6s}")
for o in ops[:30]:
    g = lambda k: tot[(o, k)] / units * per
    print(f"{'':16s}{o:12s} {g('inst'):7.2f} {g('wf'):8.2f} {g('ideal'):7.2f} {g('tag'):7.2f} {g('l2s'):7.2f} {100 * tot[(o, 'samp')] / S:6.1f}")
print(f"total: warp inst {I / units * per:.2f}, smem wavefronts {W / units * per:.2f} per {per:g} units")
