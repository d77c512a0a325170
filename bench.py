#!/usr/bin/env python
"""Benchmark of the hot path of arxiv 1811.10074 on B200 (contract: README of the task / DESIGN.md).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3|c1|c2|c4]

One STEP = one pass of the whole hot path over one synthetic genome (default: BASELINE.json
configs[2], "C3": 3.1 Gbp human-genome-shaped, GC 41 %, 1 % N in runs, k=19, w=10):
  a1 2-bit packing (mz_encode)  ->  a2-a7 fused k-mer/hash/window-min/compaction (mz_extract_ex)
  ->  a8 seed table with 2^24 buckets (seedtable_build; at N>1: count -> NCCL all_reduce ->
  partition -> NCCL all_to_all -> finalize, a9).
`value` = input bases of the whole job / device step time (max over ranks), in Gbases/s.
`e2e` = the same through the public API with HOST buffers: pinned ASCII in (H2D), seed table
(pointer table + position table) out (D2H), both inside the timed region.
Rank 0 prints ONE JSON line.  `--impl reference` times the CPU oracle (the tier's
reference arm) on a bounded sample of the same workload.

Secondary configs (not the driver's default line; their JSON lines are kept under profiles/):
  --config c2   BASELINE configs[1]: generic sliding sums slsum_run_ex on 2^28 elements,
                {MIN_U32, ADD_U32, ADD_F32} x w in {4,16,64,256,1024} x {GENERIC, COMMUTATIVE};
                Gelem/s and the HBM roofline per run (8 B algorithmic traffic per element).
  --config c4   BASELINE configs[3]: 1M long reads (9.98e9 bases), k=15 w=10, segmented
                minimizer extraction (encode + mz_extract_ex with read offsets), Gbases/s.
  --config lookup  SURVEY NEXT f1: seed lookup of the minimizers of the first 100k C4 reads
                against the seed table (2^28 buckets) of their 2^30-base template, k=15 w=10;
                Gqueries/s of seedtable_lookup (count + scan + emit).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

K_MER, W_WIN, BITS = 19, 10, 24
# algorithmic bytes per unit
SEEDTABLE_BYTES_PER_REC = 8 + 12 + 12   # histogram reads 8 B, the scatter reads 12 B and writes 12 B
# algorithmic 32-bit integer operations per base of the fused minimizer kernel
# (k=19, w=10): roll 3 + H_38 28 + key 2 + three 64-bit minima 12 + change/emit 3
MZ_INT_OPS_PER_BASE = {19: 48, 15: 30}
SURVEY_OPS_PER_BASE = {19: 65, 15: 35}
# N>1 seed-table exchange: "p2p" = partition fused with the all-to-all over symmetric memory
# (dist.exchange_seedtable_p2p, the product); "nccl" = partition + NCCL all_to_all_single
EXCHANGE = os.environ.get("MZS_EXCHANGE", "p2p")
# MZS_FUSED_HIST=0: the table counts its first pass itself instead of taking the minimizer
# kernel's fused histogram (mz_out.hist; A/B switch)
FUSED_HIST = os.environ.get("MZS_FUSED_HIST", "1") != "0"
SM_COUNT, INT32_LANES_PER_SM_CLK = 148, 128   # 4 SMSPs x 32 lanes issue (B200_PROFILING / B300_MICROARCH)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=["c3", "c1", "c2", "c4", "lookup", "ties"])
    ap.add_argument("--graph-reps", type=int, default=1000, help="c1: CUDA-graph replays timed (0: off)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--canonical", action="store_true",
                    help="c3/c4: canonical (strand-symmetric) minimizers, MZ_KEY_CANON (NEXT f4)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pos64", action="store_true", help="c3: skip the u64-position-table step timed beside the line")
    ap.add_argument("--cpu-sample-bases", type=int, default=32_000_000)
    return ap.parse_args()


def load_traffic(name):
    """DRAM bytes per launch of the step's kernels from the latest committed ncu --set full
    capture (profiles/r02 or r01 traffic_c3.json, written by tools/ncu_summary.py traffic);
    None if absent."""
    for rd in ("r02", "r01"):
        p = os.path.join(ROOT, "profiles", rd, name)
        if os.path.exists(p):
            break
    else:
        return None
    try:
        return json.load(open(p))
    except Exception:
        return None


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured", float(d.get("sm_max_mhz", 1965.0))
    return 6650.0, "fallback", 1965.0


def load_int_peak():
    """The INT32 issue roof measured by tools/microbench_int.cu (profiles/r01/int_peak.json):
    a 1:1 ALU/FMA-pipe mix, reported beside the derived peak (which stays the denominator)."""
    p = os.path.join(ROOT, "profiles", "r01", "int_peak.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return {"tops": d.get("mixed_imm_tops"), "alu_pipe_only_tops": d.get("lop3_tops"),
            "source": "profiles/r01/int_peak.json (tools/microbench_int.cu)"}


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ the reference arm (CPU oracle)
def cpu_oracle_run(sample_bases: int):
    """The oracle as it stands, on a bounded sample of the C3 workload (bases [0, sample))."""
    import oracle as O
    from synthgen import host as H
    c3 = H.C3()
    seq = c3.ascii(0, sample_bases)
    t0 = time.perf_counter()
    key, pos = O.mz(seq, K_MER, W_WIN)
    O.seedtable(key, pos, K_MER, BITS)
    dt = time.perf_counter() - t0
    return sample_bases / dt / 1e9, dt, O.num_threads(), len(key)


def cpu_model() -> str:
    """The host CPU's model name (record it beside the oracle's core count)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_main(args, rank, world):
    if rank != 0:
        return 0
    import oracle as O
    sample = args.cpu_sample_bases // 4    # per step: a bounded sample so K+W steps stay within minutes
    for _ in range(args.warmup):
        cpu_oracle_run(min(sample, 2_000_000))
    vals = []
    for _ in range(max(1, args.steps)):
        v, dt, cores, m = cpu_oracle_run(sample)
        vals.append(v)
    v = statistics.median(vals)
    line = {
        "impl": "reference", "metric": "minimizer extraction + seed table, Gbases/s (whole job)",
        "value": v, "unit": "Gbases/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sample / (v * 1e9) * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": "C3 sample", "k": K_MER, "w": W_WIN, "bucket_bits": BITS, "bases": sample},
        "cpu_baseline": {"value": v, "unit": "Gbases/s", "cores": O.num_threads(), "cpu_model": cpu_model(), "kind": "oracle",
                         "sample": f"first {sample} bases of C3 (mz + seedtable oracle)"},
        "e2e": {"value": v, "unit": "Gbases/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ secondary configs
def _nccl_log_env():
    """NCCL's communicator init lines (rank, nranks, transport) in the run's stderr, so the
    number of ranks a communicator really spans can be checked from the log."""
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")


def _timed(fn, steps, warmup, stream, world=1):
    """Device time per call (CUDA events on the launching stream, synchronize on both sides);
    at N>1 a barrier before and after, and the maximum over ranks."""
    import torch
    import torch.distributed as dist
    for _ in range(max(3, warmup)):
        fn()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
        torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def bench_c2(args, rank=0, world=1):
    """C2: slsum_run_ex on 2^28 elements (inputs 1 GiB >> L2, no flush needed).  At N>1 every
    rank owns a contiguous range of the outputs and reads its inputs with a w-1 halo
    (dist.plan_slsum; no collective on the data path); each run's time is the max over ranks."""
    import torch
    import paper_1811_10074_b200 as P
    from paper_1811_10074_b200 import dist as D
    from synthgen import device as SD
    hbm_peak, peak_kind, _ = load_peaks()
    n = 1 << 28
    stream = torch.cuda.current_stream()
    names = [("MIN_U32", P.SLSUM_MIN_U32), ("ADD_U32", P.SLSUM_ADD_U32), ("ADD_F32", P.SLSUM_ADD_F32)]
    runs, tot_ms = [], 0.0
    with Clocks(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        for w in (4, 16, 64, 256, 1024):
            oa, ob, lo, hi = D.plan_slsum(n, w, world)[rank]
            xu = SD.c2_u32(hi - lo, lo=lo)
            xf = SD.c2_f32(hi - lo, lo=lo)
            yu = torch.empty(max(1, ob - oa), dtype=torch.uint32, device="cuda")
            yf = torch.empty(max(1, ob - oa), dtype=torch.float32, device="cuda")
            for name, op in names:
                x, y = (xf, yf) if op == P.SLSUM_ADD_F32 else (xu, yu)
                paths = [("generic", P.SLSUM_PATH_GENERIC), ("commutative", P.SLSUM_PATH_COMMUTATIVE),
                         ("scalar_alg1", P.SLSUM_PATH_SCALAR)]
                if op == P.SLSUM_ADD_U32:   # the invertible op also has the recurrent path (NEXT f2)
                    paths.append(("recurrent", P.SLSUM_PATH_RECURRENT))
                for pname, path in paths:
                    ms = _timed(lambda: P.slsum_run(op, w, x, y[: ob - oa], path=path), args.steps, args.warmup,
                                stream, world)
                    tot_ms += ms
                    gbs = 8.0 * n / world / (ms * 1e-3) / 1e9          # per GPU
                    runs.append({"op": name, "w": w, "path": pname, "ms": ms, "gelem_s": n / (ms * 1e-3) / 1e9,
                                 "hbm_gbs": gbs, "hbm_frac": gbs / hbm_peak})
            del xu, xf, yu, yf
    clk_sum = clk.summary()
    if rank != 0:
        return 0
    best = max(runs, key=lambda r: r["hbm_frac"])
    gen = [r for r in runs if r["path"] == "generic"]
    # the headline aggregates the O(1)/O(log w) paths; Alg. 1 is O(w) per output by design
    fast = [r for r in runs if r["path"] != "scalar_alg1"]
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        # the oracle's strict O(wN) left fold on the same 15 (op, w) runs, first 2^23 elements each
        import oracle as O
        ns = 1 << 23
        xs_u, xs_f = SD.c2_u32(ns).cpu().numpy(), SD.c2_f32(ns).cpu().numpy()
        t0 = time.perf_counter()
        for oop, xs in ((O.MIN_U32, xs_u), (O.ADD_U32, xs_u), (O.ADD_F32, xs_f)):
            for w in (4, 16, 64, 256, 1024):
                O.slsum(oop, w, xs)
        dt = time.perf_counter() - t0
        cpu = {"value": 15 * ns / dt / 1e9, "unit": "Gelem/s", "cores": O.num_threads(), "cpu_model": cpu_model(), "kind": "oracle",
               "sample": f"the 15 (op, w) runs on the first {ns} C2 elements each ({dt:.1f} s)"}
    line = {
        "metric": "generic sliding window sums (Eq. 2), Gelem/s",
        "value": len(fast) * n / (sum(r["ms"] for r in fast) * 1e-3) / 1e9,
        "unit": "Gelem/s", "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
        "ms_per_step": tot_ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32/f32",
        "data": "synthetic",
        "config": {"workload": "C2: 2^28 elements x {MIN_U32, ADD_U32, ADD_F32} x w {4..1024} x {generic, commutative,"
                               " scalar (Alg. 1)} (+ recurrent for ADD_U32)",
                   "step": f"all {len(runs)} runs", "l2": "inputs 1 GiB >> L2; no flush needed",
                   "parallelism": f"output ranges over {world} GPUs, w-1 input halo, no collective"},
        "roofline": {"bound": "hbm", "kernel": f"slsum {best['path']} {best['op']} w={best['w']} (best)",
                     "achieved": best["hbm_gbs"], "peak": hbm_peak, "unit": "GB/s", "frac": best["hbm_frac"],
                     "traffic": None, "peak_kind": peak_kind},
        "roofline_generic_min_frac": min(r["hbm_frac"] for r in gen),
        "runs": runs, "cpu_baseline": cpu, "clocks": clk_sum, "gpu_launches": len(runs) * args.steps,
    }
    print(json.dumps(line), flush=True)
    return 0


def bench_c4(args, rank=0, world=1):
    """C4: 1M lognormal reads, k=15 w=10; encode + segmented minimizer extraction.  At N>1 every
    rank takes a contiguous range of reads balanced by bases (dist.plan_reads; windows never
    cross a read, so no halo and no collective); the time is the max over ranks."""
    import torch
    import paper_1811_10074_b200 as P
    from paper_1811_10074_b200 import dist as D
    from synthgen import device as SD
    from synthgen import host as H
    hbm_peak, peak_kind, sm_max = load_peaks()
    k, w = 15, 10
    c4 = H.C4()
    n_total = c4.n
    r0, r1 = D.plan_reads(c4.read_off, world)[rank]
    base = int(c4.read_off[r0])
    n = int(c4.read_off[r1]) - base
    seq = SD.c4_ascii(c4) if world == 1 else SD.c4_ascii_reads(c4, r0, r1)
    ro = torch.from_numpy((c4.read_off[r0:r1 + 1] - base).astype(np.uint64).view(np.int64)).cuda().view(torch.uint64)
    nw = (n + 31) // 32
    words = torch.empty(nw + 1, dtype=torch.uint64, device="cuda")
    inval = torch.empty(nw + 1, dtype=torch.uint32, device="cuda")
    cap = int(0.21 * n) + 1024
    out_h = torch.empty(cap, dtype=torch.uint64, device="cuda")
    out_p = torch.empty(cap, dtype=torch.uint64, device="cuda")
    d_count = torch.zeros(1, dtype=torch.uint64, device="cuda")
    ws = torch.empty(P.mz_workspace_bytes(n, k, w, P.MZ_IN_PACKED2), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    keymode = P.MZ_KEY_CANON if args.canonical else P.MZ_KEY_HASH
    ev = []

    def step(record=False):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if record else None
        if record:
            e[0].record(stream)
        P.mz_encode(seq, words, inval)
        if record:
            e[1].record(stream)
        P.mz_extract_ex(words, k, w, n=n, kind=P.MZ_IN_PACKED2, invalid=inval, read_off=ro, capacity=cap,
                        out_hash=out_h, out_pos=out_p, d_count=d_count, ws=ws, keymode=keymode, pos_base=base)
        if record:
            e[2].record(stream)
            ev.append(e)

    with Clocks(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        ms = _timed(lambda: step(True), args.steps, args.warmup, stream, world)
    m = int(d_count.view(torch.int64).item())
    if m > cap:
        raise RuntimeError(f"capacity {cap} < {m} records")
    ev = ev[-args.steps:]
    enc_ms = statistics.mean(a.elapsed_time(b) for a, b, _ in ev)
    mz_ms = statistics.mean(b.elapsed_time(c) for _, b, c in ev)
    clk_sum = clk.summary()
    sm_mhz = clk_sum.get("sm_mhz") or sm_max
    int_peak = SM_COUNT * INT32_LANES_PER_SM_CLK * sm_mhz * 1e6 / 1e12
    ops = MZ_INT_OPS_PER_BASE[15] * n
    ach = ops / (mz_ms * 1e-3) / 1e12
    if rank != 0:
        return 0
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        import oracle as O
        r1 = 2000
        hi = int(c4.read_off[r1])
        s = c4.ascii_range(0, hi)
        t0 = time.perf_counter()
        O.mz(s, k, w, read_off=c4.read_off[: r1 + 1].astype(np.uint64))
        dt = time.perf_counter() - t0
        cpu = {"value": hi / dt / 1e9, "unit": "Gbases/s", "cores": O.num_threads(), "cpu_model": cpu_model(), "kind": "oracle",
               "sample": f"first {r1} reads ({hi} bases) of C4 ({dt:.1f} s)"}
    line = {
        "metric": "minimizer extraction over a long-read batch, Gbases/s", "value": n_total / (ms * 1e-3) / 1e9,
        "unit": "Gbases/s", "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": "C4: 1M reads, lognormal(mean 10 kbp, sd 8 kbp), 10% substitutions"
                               + (" (canonical minimizers)" if args.canonical else ""), "k": k, "w": w,
                   "bases": n_total, "reads": c4.nreads, "records_rank0": m, "density": m / n,
                   "parallelism": f"reads balanced by bases over {world} GPUs, no halo, no collective",
                   "l2": f"inputs ({n / 1e9:.1f} GB) >> L2; no flush needed"},
        "roofline": {"bound": "alu", "kernel": "mz_fast_kernel<10,0,15> (a2-a7 fused, read-segmented)",
                     "achieved": ach, "peak": int_peak, "unit": "Tops/s", "frac": ach / int_peak, "traffic": None,
                     "peak_kind": f"derived: {SM_COUNT} SMs x {INT32_LANES_PER_SM_CLK} int32 lanes/clk x {sm_mhz:.0f} MHz",
                     "ops_per_base": MZ_INT_OPS_PER_BASE[15], "ms": mz_ms,
                     "frac_survey_ops": SURVEY_OPS_PER_BASE[15] * n / (mz_ms * 1e-3) / 1e12 / int_peak,
                     "survey_ops_per_base": SURVEY_OPS_PER_BASE[15]},
        "hbm_step": {"encode_ms": enc_ms, "extract_ms": mz_ms,
                     "encode_frac": n * 1.375 / (enc_ms * 1e-3) / 1e9 / hbm_peak,
                     "extract_frac": (n * 0.375 + m * 16) / (mz_ms * 1e-3) / 1e9 / hbm_peak, "peak": hbm_peak,
                     "peak_kind": peak_kind},
        "cpu_baseline": cpu, "clocks": clk_sum, "gpu_launches": 2 * args.steps,
    }
    print(json.dumps(line), flush=True)
    return 0


TIES_N = 400_000_000
# bytes per base the ties composition moves at w <= 32 (K10): encode 1 + 0.28, keys
# 0.28 + 8, the min sum 8 + 8, mark (K and m read, bitmap written) 16 + 0.125; per record the
# write kernel reads K (8) and writes hash + pos (16)
TIES_BYTES_PER_BASE = 1.28 + 8.28 + 16 + 16.125
TIES_BYTES_PER_RECORD = 8 + 16


def bench_ties(args):
    """f4: minimap2-compatible minimizers (mz_extract_ties: all tied minima, run-end windows) on a
    400 Mbp C3-shaped prefix (GC 41 %, 1 % N in runs), k=19, w=10, ASCII input resident in HBM."""
    import torch
    import paper_1811_10074_b200 as P
    from synthgen import device as SD
    from synthgen import host as H
    hbm_peak, peak_kind, sm_max = load_peaks()
    k, w, n = K_MER, W_WIN, TIES_N
    c3 = H.C3()
    seq = SD.c3_ascii(c3, lo=0, n=n, device="cuda")
    cap = int(0.25 * n) + 1024
    out_h = torch.empty(cap, dtype=torch.uint64, device="cuda")
    out_p = torch.empty(cap, dtype=torch.uint64, device="cuda")
    d_count = torch.zeros(1, dtype=torch.uint64, device="cuda")
    ws = torch.empty(P.mz_ties_workspace_bytes(n, k, w, P.MZ_IN_ASCII), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        P.mz_extract_ties(seq, k, w, capacity=cap, out_hash=out_h, out_pos=out_p, d_count=d_count, ws=ws)

    with Clocks(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        ms = _timed(step, args.steps, args.warmup, stream)
    m = int(d_count.view(torch.int64).item())
    if m > cap:
        raise RuntimeError(f"capacity {cap} < {m} records")
    byts = TIES_BYTES_PER_BASE * n + TIES_BYTES_PER_RECORD * m
    ach = byts / (ms * 1e-3) / 1e9
    # DRAM bytes of one step's six kernels from the committed ncu --set full capture, if any
    tr = load_traffic("traffic_ties.json")
    traffic = sum(v["dram_bytes"] / max(1, v.get("launches", 1)) for v in tr.values()) if tr else None
    cpu = None
    if not args.no_cpu_baseline:
        import oracle as O
        ns = min(n, args.cpu_sample_bases)
        s = seq[:ns].cpu().numpy()
        t0 = time.perf_counter()
        O.mz_ties(s, k, w)
        dt = time.perf_counter() - t0
        cpu = {"value": ns / dt / 1e9, "unit": "Gbases/s", "cores": O.num_threads(), "cpu_model": cpu_model(),
               "kind": "oracle", "sample": f"orc_mz_ties on the first {ns} bases of the prefix ({dt:.1f} s)"}
    line = {
        "metric": "minimap2-compatible minimizer extraction, Gbases/s", "value": n / (ms * 1e-3) / 1e9,
        "unit": "Gbases/s", "n_gpus": 1, "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": "f4: mz_extract_ties on a 400 Mbp C3-shaped prefix (GC 41 %, 1 % N in runs)",
                   "k": k, "w": w, "bases": n, "records": m, "density": m / n,
                   "l2": f"inputs and intermediates ({n * 33 / 1e9:.0f} GB) >> L2; no flush needed"},
        "roofline": {"bound": "hbm", "kernel": "the whole composition (encode, keys, slsum MIN_U64, mark with the "
                                               "shared-memory max, scan, write)",
                     "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak, "traffic": traffic,
                     "traffic_note": "DRAM bytes of one step's kernels, ncu --set full "
                                     f"(profiles/r0x/traffic_ties.json); algorithmic {byts:.4g} B",
                     "bytes_per_base": TIES_BYTES_PER_BASE, "peak_kind": peak_kind},
        "cpu_baseline": cpu, "clocks": clk.summary(),
        "gpu_launches": 6 * args.steps,
    }
    print(json.dumps(line), flush=True)
    return 0


def bench_lookup(args):
    """NEXT f1: batch seed lookup (Fig. 1 lookups) of read minimizers against a template table."""
    import torch
    import paper_1811_10074_b200 as P
    from synthgen import device as SD
    from synthgen import host as H
    hbm_peak, peak_kind, _ = load_peaks()
    # 2^28 buckets (offsets 2 GiB): minimizer hashes are skewed low, so with 2^24 buckets a query
    # scans ~120 fingerprints of its (size-biased) bucket; at 2^28 about 8 (R30)
    k, w, bits = 15, 10, int(os.environ.get("MZS_LOOKUP_BITS", "28"))  # 24: the C5 table geometry
    nq_reads = 100_000
    c4 = H.C4()
    tn = c4.tlen
    # template table (untimed): encode + minimizers + seed table, all through the library
    tmpl = SD.c1_ascii(tn, seed=c4.seed_t)
    tw, ti = P.mz_encode(tmpl)
    th, tp, tc = P.mz_extract_ex(tw, k, w, n=tn, kind=P.MZ_IN_PACKED2, invalid=ti, capacity=int(0.25 * tn))
    torch.cuda.synchronize()
    mt = int(tc.view(torch.int64).item())
    off, pos_tab, fp = P.seedtable_build(th[:mt], tp[:mt], k, bits)
    del tmpl, tw, ti, th, tp
    # queries (untimed): minimizers of the first 100k reads
    seq = SD.c4_ascii(c4)
    nb = int(c4.read_off[nq_reads])
    ro = torch.from_numpy(c4.read_off[: nq_reads + 1].astype(np.int64)).cuda().view(torch.uint64)
    qh, qp, qc = P.mz_extract_ex(seq[:nb], k, w, read_off=ro, capacity=int(0.25 * nb))
    torch.cuda.synchronize()
    nq = int(qc.view(torch.int64).item())
    del seq
    q = qh[:nq]
    hit_off = torch.empty(nq + 1, dtype=torch.uint64, device="cuda")
    d_total = torch.zeros(1, dtype=torch.uint64, device="cuda")
    ws = torch.empty(P.seedtable_lookup_workspace_bytes(nq), dtype=torch.uint8, device="cuda")
    P.seedtable_lookup(q, k, bits, off, fp, pos_tab, hit_off=hit_off, d_total=d_total, hit_cap=0, ws=ws)
    torch.cuda.synchronize()
    hits = int(d_total.view(torch.int64).item())
    hit_pos = torch.empty(max(1, hits), dtype=torch.uint64, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        P.seedtable_lookup(q, k, bits, off, fp, pos_tab, hit_off=hit_off, hit_pos=hit_pos, hit_cap=hits,
                           d_total=d_total, ws=ws)

    with Clocks(0) as clk:
        ms = _timed(step, args.steps, args.warmup, stream)
    clk_sum = clk.summary()
    mean_slice = mt / (1 << bits)
    # algorithmic bytes per query (R30): key 8, two offsets 16, its CSR offset written + read 16,
    # the fingerprints of ITS bucket 4 per entry (the hits are the entries of that slice whose
    # fingerprint matches, so one scan of the slice is the method's own work), and per hit its
    # position read + written 16.  Minimizer hashes are skewed low, so the buckets queries fall
    # in are longer than the mean bucket: the slice lengths are summed over the actual queries.
    kk = 2 * k
    qf = (q.view(torch.int64) >> (kk - 32)) if kk >= 32 else ((q.view(torch.int64) << (32 - kk)) & 0xFFFFFFFF)
    qb = (qf & 0xFFFFFFFF) >> (32 - bits)
    offl = off.view(torch.int64)
    qlen = int((offl[qb + 1] - offl[qb]).sum().item())
    del qf, qb
    alg = nq * (8 + 16 + 16) + 4 * qlen + hits * 16
    # the earlier accounting (2 passes over a bucket of the MEAN length), kept for comparison
    alg_mean = nq * (2 * (8 + 16 + 4 * mean_slice) + 16) + hits * 16
    cpu = None
    if not args.no_cpu_baseline:
        import oracle as O
        ts = 1 << 25                                   # a 32 Mbp template prefix for the oracle table
        tk, tpp = O.mz(H.c1_ascii(ts, seed=c4.seed_t), k, w)
        to, tf, tpt = O.seedtable(tk, tpp, k, bits)
        qs = q[: 40_000_000].cpu().numpy()
        t0 = time.perf_counter()
        O.lookup(qs, k, bits, to, tf, tpt)
        dt = time.perf_counter() - t0
        cpu = {"value": len(qs) / dt / 1e9, "unit": "Gqueries/s", "cores": O.num_threads(), "cpu_model": cpu_model(), "kind": "oracle",
               "sample": f"{len(qs)} of the queries against the oracle's table of a {ts}-base template prefix "
                         f"({dt:.1f} s)"}
    line = {
        "metric": "seed lookup (Fig. 1) of read minimizers against a template seed table, Gqueries/s",
        "value": nq / (ms * 1e-3) / 1e9, "unit": "Gqueries/s", "n_gpus": 1, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"minimizers of the first {nq_reads} C4 reads vs the 2^30-base C4 template table",
                   "k": k, "w": w, "bucket_bits": bits, "queries": nq, "table_entries": mt, "hits": hits,
                   "hits_per_query": hits / max(1, nq), "l2": "table (>1.6 GB) >> L2; no flush needed"},
        "roofline": {"bound": "hbm", "kernel": "lookup_kernel count + emit, scan (one step)",
                     "achieved": alg / (ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                     "frac": alg / (ms * 1e-3) / 1e9 / hbm_peak, "traffic": None, "peak_kind": peak_kind,
                     "algorithmic_bytes": alg, "query_bucket_mean_len": qlen / max(1, nq),
                     "frac_mean_bucket_model": alg_mean / (ms * 1e-3) / 1e9 / hbm_peak},
        "cpu_baseline": cpu, "clocks": clk_sum, "gpu_launches": 5 * args.steps,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_main(args, rank, world)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if args.config == "lookup":
        if world > 1 and rank != 0:
            return 0          # the lookup line is a single-GPU measurement
        return bench_lookup(args)
    if args.config == "ties":
        if world > 1 and rank != 0:
            return 0          # the f4 variant's line is a single-GPU measurement
        return bench_ties(args)
    if args.config in ("c2", "c4"):
        if world > 1:
            _nccl_log_env()
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        try:
            return {"c2": bench_c2, "c4": bench_c4}[args.config](args, rank, world)
        finally:
            if world > 1:
                dist.destroy_process_group()
    dev = torch.device("cuda", local)
    if world > 1:
        _nccl_log_env()
        dist.init_process_group("nccl", device_id=dev)
    import paper_1811_10074_b200 as P
    from paper_1811_10074_b200 import dist as D
    from synthgen import device as SD
    from synthgen import host as H

    hbm_peak, peak_kind, sm_max = load_peaks()
    k, w, bits = K_MER, W_WIN, BITS
    if args.config == "c3":
        c3 = H.C3()
        n_total = c3.n
    else:
        c3 = None
        n_total = 1_000_000
        k, w, bits = 15, 10, 24
    shards = D.plan_shards(n_total, k, w, world)
    sh = shards[rank]
    n = sh.base_hi - sh.base_lo
    # device input (generated on the device; outside the timed region)
    if c3 is not None:
        seq = SD.c3_ascii(c3, lo=sh.base_lo, n=n, device=dev)
    else:
        seq = SD.c1_ascii(n, lo=sh.base_lo, device=dev)
    nwin_local = max(0, sh.win_hi - sh.win_lo)
    cap = max(1024, int(0.25 * nwin_local) + 1024)     # density ~0.18; checked below
    stream = torch.cuda.current_stream()
    nw = (n + 31) // 32

    class Bufs:
        """One full set of device buffers of the step (the e2e pipeline uses two)."""

        def __init__(self):
            self.words = torch.empty(nw + 1, dtype=torch.uint64, device=dev)
            self.inval = torch.empty(nw + 1, dtype=torch.uint32, device=dev)
            self.out_h = torch.empty(cap, dtype=torch.uint64, device=dev)
            self.out_p = torch.empty(cap, dtype=torch.uint64, device=dev)
            # packed seed-table items written by the minimizer kernel beside (hash, pos): the
            # table's first radix pass (N=1) or the fused owner partition (N>1) reads 8 B per
            # record instead of 16
            self.out_i = torch.empty(cap, dtype=torch.uint64, device=dev)
            self.d_count = torch.zeros(1, dtype=torch.uint64, device=dev)
            self.mz_ws = torch.empty(P.mz_workspace_bytes(n, k, w, P.MZ_IN_PACKED2), dtype=torch.uint8, device=dev)
            if world == 1:
                self.st_ws = torch.empty(P.seedtable_workspace_bytes(cap, bits), dtype=torch.uint8, device=dev)
                self.offsets = torch.empty((1 << bits) + 1, dtype=torch.uint64, device=dev)
                self.pos_out = torch.empty(cap, dtype=torch.uint64, device=dev)
                self.fp_out = torch.empty(cap, dtype=torch.uint32, device=dev)
                self.pos32_out = None   # (e2e) the 32-bit position table, allocated on first use
                # the table's first radix pass digit counts, accumulated by the minimizer kernel
                # while it writes the records (mz_out.hist): the first pass skips its upsweep
                self.hist = (torch.empty(P.seedtable_hist_words(cap, bits), dtype=torch.uint32, device=dev)
                             if FUSED_HIST else None)

    B0 = Bufs()
    d_count = B0.d_count
    ev = {name: [] for name in ("encode", "extract", "table")}

    def step(seq_dev, record=False, bf=B0, pos32=False):
        st = torch.cuda.current_stream()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if record else None
        if record:
            e[0].record(st)
        P.mz_encode(seq_dev, bf.words, bf.inval)
        if record:
            e[1].record(st)
        P.mz_extract_ex(bf.words, k, w, n=n, kind=P.MZ_IN_PACKED2, invalid=bf.inval, pos_base=sh.base_lo,
                        win_lo=sh.win_lo, win_hi=sh.win_hi, capacity=cap, out_hash=bf.out_h, out_pos=bf.out_p,
                        d_count=bf.d_count, ws=bf.mz_ws, out_items=bf.out_i,
                        out_hist=bf.hist if world == 1 else None, hist_bits=bits,
                        keymode=P.MZ_KEY_CANON if args.canonical else P.MZ_KEY_HASH)
        if record:
            e[2].record(st)
        if world == 1 and pos32:
            # seedtable_build_items32: positions mod 2^32, exact here (C3 < 2^32 bases)
            if bf.pos32_out is None:
                bf.pos32_out = torch.empty(cap, dtype=torch.uint32, device=dev)
            P.seedtable_build_items_ex(bf.out_i, bf.out_h, bf.out_p, k, bits, m=cap, d_m=bf.d_count, hist=bf.hist,
                                       pos32=True, offsets=bf.offsets, pos_out=bf.pos32_out, fp_out=bf.fp_out,
                                       ws=bf.st_ws)
            res = (bf.offsets, bf.pos32_out)
        elif world == 1:
            P.seedtable_build_items_ex(bf.out_i, bf.out_h, bf.out_p, k, bits, m=cap, d_m=bf.d_count, hist=bf.hist,
                                       offsets=bf.offsets, pos_out=bf.pos_out, fp_out=bf.fp_out, ws=bf.st_ws)
            res = (bf.offsets, bf.pos_out)
        else:
            # the record count stays on the device (capacity-sized arrays + d_count) up to the
            # exchange's own host read of the gathered owner counts
            xchg = D.exchange_seedtable_p2p if EXCHANGE == "p2p" else D.exchange_seedtable
            res = xchg(bf.out_h, bf.out_p, cap, k, bits, D.CudaPhases(d_m=bf.d_count, items=bf.out_i))
        if record:
            e[3].record(st)
            ev["encode"].append((e[0], e[1]))
            ev["extract"].append((e[1], e[2]))
            ev["table"].append((e[2], e[3]))
        return res

    # encode + mz + seed table: path-select kernel, 3 narrow passes x (upsweep, chunk scan, digit
    # scan, downsweep), 3 wide passes (enqueued, gated off at entry), 4 pointer-table kernels
    table_launches = 1 + 12 + 12 + 4 - (1 if FUSED_HIST else 0) + (1 if (world == 1 and c3 is not None and n_total < (1 << 32)) else 0)  # + the gated wide-path u32 narrowing
    # N>1: count, partition (NCCL: ctl + 4 narrow + 4 wide; p2p: ctl + 3 scan kernels + the fused
    # nsweep writing into the peers), finalize (ctl + 2 passes x 12 + 4)
    part = 5 if EXCHANGE == "p2p" else 1 + 4 + 4
    launches_per_step = 1 + 1 + (table_launches if world == 1 else 1 + part + (1 + 12 + 12 + 4))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # positions below 2^32 (C3 at one GPU): the table stores them as u32, exactly (R34,
    # seedtable_build_items32) -- the table the e2e line reads back; the u64 table is timed beside it
    tab32 = world == 1 and c3 is not None and n_total < (1 << 32)
    for _ in range(max(3, args.warmup)):
        step(seq, pos32=tab32)
    torch.cuda.synchronize()
    m_local = int(d_count.view(torch.int64).item())
    if m_local > cap:
        raise RuntimeError(f"capacity {cap} < {m_local} records")

    # ---------------- timed: device-resident inputs (inputs >> L2, no flush needed)
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        t0.record(stream)
        for _ in range(args.steps):
            step(seq, record=True, pos32=tab32)
        t1.record(stream)
        barrier()
    ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_step = ms / args.steps
    gbases = n_total / (ms_step * 1e-3) / 1e9

    phase_ms = {kk: statistics.mean(a.elapsed_time(b) for a, b in v) for kk, v in ev.items()}
    pos64_line = None
    if tab32 and not args.no_pos64:
        # the same step with the u64 position table (seedtable_build_items_ex, pos_out)
        for _ in range(max(3, args.warmup)):
            step(seq)
        barrier()
        a64, b64 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a64.record(stream)
        for _ in range(args.steps):
            step(seq)
        b64.record(stream)
        barrier()
        ms64 = a64.elapsed_time(b64) / args.steps
        pos64_line = {"value": n_total / (ms64 * 1e-3) / 1e9, "unit": "Gbases/s", "ms_per_step": ms64,
                      "steps": args.steps, "table_positions": "u64 (seedtable_build_items_ex, pos_out)"}
    # per-step device times (encode start -> table end of each timed step): median and best
    per_step = [a.elapsed_time(d) for (a, _), (_, d) in zip(ev["encode"], ev["table"])]
    step_stats = {"median_ms": statistics.median(per_step), "best_ms": min(per_step), "steps": len(per_step)}

    # ---------------- C1 (1 Mbp, ~launch-bound): the step captured once in a CUDA graph and
    # replayed.  The inputs fit in L2, so every replay first overwrites a 256 MiB
    # buffer (L2 flush); a graph of the flush alone is timed the same way and subtracted.
    graph = None
    if c3 is None and world == 1 and args.graph_reps > 0:
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            flush.fill_(1)
            step(seq)
        torch.cuda.synchronize()
        g_step, g_flush = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_step):
            flush.fill_(1)
            step(seq)
        with torch.cuda.graph(g_flush):
            flush.fill_(1)

        def replay_ms(g):
            g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(args.graph_reps):
                g.replay()
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b) / args.graph_reps

        with Clocks(local) as gclk:
            t_step, t_flush = replay_ms(g_step), replay_ms(g_flush)
        g_ms = max(1e-6, t_step - t_flush)
        graph = {"value": n_total / (g_ms * 1e-3) / 1e9, "unit": "Gbases/s", "ms_per_step": g_ms,
                 "replays": args.graph_reps, "ms_flush_plus_step": t_step, "ms_flush": t_flush,
                 "l2": "256 MiB overwrite before every replay, its own graph's time subtracted",
                 "clocks": gclk.summary()}
        m_check = int(d_count.view(torch.int64).item())
        if m_check != int(B0.d_count.view(torch.int64).item()) or m_check > cap:
            raise RuntimeError("graph replay changed the record count")

    # ---------------- e2e: host buffers through the public API.  Every step copies its ASCII
    # input from pinned host memory (H2D) and reads its seed table back (D2H: pointer table +
    # the m positions).  Steps are pipelined over two buffer sets and three streams, so the
    # D2H of step i overlaps the H2D and compute of step i+1 (PCIe is full duplex).
    e2e = None
    if not args.no_e2e and world == 1:
        nset = max(2, int(os.environ.get("MZS_E2E_SETS", "2")))
        extra = [Bufs() for _ in range(nset - 1)]
        sets = (B0, *extra)
        host_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        host_in.copy_(seq)
        host_off = [torch.empty((1 << bits) + 1, dtype=torch.uint64, pin_memory=True) for _ in range(nset)]
        host_pos = [torch.empty(cap, dtype=torch.uint64, pin_memory=True) for _ in range(nset)]
        host_cnt = torch.zeros(nset, dtype=torch.int64, pin_memory=True)
        seqd = [torch.empty_like(seq) for _ in range(nset)]
        del seq
        s_h2d, s_cmp, s_d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()

        def e2e_run(pos32: bool):
            ev_h2d = [torch.cuda.Event() for _ in range(nset)]
            ev_cmp = [torch.cuda.Event() for _ in range(nset)]
            ev_d2h = [torch.cuda.Event() for _ in range(nset)]
            started = [False] * nset
            esz = 4 if pos32 else 8
            # pinned host position tables (u32 ones viewed out of the u64 buffers)
            hpos = [hp.view(torch.uint32)[:cap] if pos32 else hp for hp in host_pos]

            def enqueue(b):
                with torch.cuda.stream(s_h2d):
                    if started[b]:
                        s_h2d.wait_event(ev_cmp[b])      # set b's input was consumed by its last compute
                    seqd[b].copy_(host_in, non_blocking=True)
                    ev_h2d[b].record(s_h2d)
                with torch.cuda.stream(s_cmp):
                    s_cmp.wait_event(ev_h2d[b])
                    if started[b]:
                        s_cmp.wait_event(ev_d2h[b])      # set b's table was read back
                    step(seqd[b], bf=sets[b], pos32=pos32)
                    host_cnt[b:b + 1].copy_(sets[b].d_count.view(torch.int64), non_blocking=True)
                    ev_cmp[b].record(s_cmp)
                started[b] = True

            def readback(b):
                ev_cmp[b].synchronize()                  # the record count decides how much to read back
                m = int(host_cnt[b].item())
                with torch.cuda.stream(s_d2h):
                    s_d2h.wait_event(ev_cmp[b])
                    host_off[b].copy_(sets[b].offsets, non_blocking=True)
                    src = sets[b].pos32_out if pos32 else sets[b].pos_out
                    hpos[b][:m].copy_(src[:m], non_blocking=True)
                    ev_d2h[b].record(s_d2h)
                return 8 * ((1 << bits) + 1) + esz * m

            ke = max(3, args.steps)                      # the K timed steps (fill and drain amortised over K)
            enqueue(0)                                   # warm-up step (untimed)
            readback(0)
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            bev = torch.cuda.Event(enable_timing=True)
            a.record(s_h2d)
            d2h = 0
            for i in range(ke):
                enqueue(i % nset)
                if i > 0:
                    d2h = readback((i - 1) % nset)
            d2h = readback((ke - 1) % nset)
            bev.record(s_d2h)
            torch.cuda.synchronize()
            e2e_ms = a.elapsed_time(bev) / ke
            return {"value": n_total / (e2e_ms * 1e-3) / 1e9, "unit": "Gbases/s", "h2d_bytes_per_step": n,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "steps": ke,
                    "table_positions": "u32 (seedtable_build_items32; exact: C3 has < 2^32 bases)" if pos32
                    else "u64 (seedtable_build_items)",
                    "pipeline": f"{nset} buffer sets, streams H2D | compute | D2H; step i's D2H overlaps step i+1"}

        use32 = c3 is not None and n_total < (1 << 32)
        e2e = e2e_run(pos32=use32)
        if use32:
            e2e["pos64"] = e2e_run(pos32=False)    # the same pipeline with the u64 position table
        del host_in, host_off, host_pos, seqd, extra
    elif not args.no_e2e and world > 1:
        # N GPUs: every rank copies its shard's ASCII in (H2D), runs the step (extraction, then
        # the seed-table exchange, fused p2p or NCCL) and reads its slice of the table back (D2H); the
        # time is the max over ranks (no cross-step pipelining here)
        host_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        host_in.copy_(seq)
        seq2 = torch.empty_like(seq)
        torch.cuda.synchronize()

        hbuf = {}   # pinned read-back buffers, allocated in the untimed first call and reused

        def e2e_step_mg():
            seq2.copy_(host_in, non_blocking=True)
            off, pl, fl, base = step(seq2)
            for key, t in (("off", off), ("pos", pl)):
                if key not in hbuf or hbuf[key].numel() < t.numel() or hbuf[key].dtype != t.dtype:
                    hbuf[key] = torch.empty(max(1, t.numel() + t.numel() // 8), dtype=t.dtype, pin_memory=True)
            hbuf["off"][:off.numel()].copy_(off, non_blocking=True)
            hbuf["pos"][:pl.numel()].copy_(pl, non_blocking=True)
            torch.cuda.synchronize()
            return 8 * (off.numel() + pl.numel())

        e2e_step_mg()
        barrier()
        a = torch.cuda.Event(enable_timing=True)
        bev = torch.cuda.Event(enable_timing=True)
        ke = max(1, args.steps)
        a.record(stream)
        d2h = 0
        for _ in range(ke):
            d2h = e2e_step_mg()
        bev.record(stream)
        barrier()
        tt = torch.tensor([a.elapsed_time(bev) / ke], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
        e2e = {"value": n_total / (e2e_ms * 1e-3) / 1e9, "unit": "Gbases/s", "h2d_bytes_per_step": n,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "steps": ke,
               "note": "per-rank bytes (rank 0); time = max over ranks"}
        del host_in, seq2

    # ---------------- rooflines (algorithmic work / event time of the launches)
    m_rec = m_local
    per_phase_bytes = {
        "encode": n * (1 + 0.25 + 0.125),
        # records: hash + pos (16 B), plus the 8-byte packed item at N=1 (seedtable_build_items)
        "extract": n * (0.25 + 0.125) + m_rec * (24 if world == 1 else 16),
        # the last pass writes u32 positions with the 32-bit table (4 B less per entry)
        "table": m_rec * (SEEDTABLE_BYTES_PER_REC - (4 if tab32 else 0)) + 8 * ((1 << bits) + 1),
    }
    clk = clk_sum = clk.summary()
    sm_mhz = clk.get("sm_mhz") or sm_max
    int_peak = SM_COUNT * INT32_LANES_PER_SM_CLK * sm_mhz * 1e6 / 1e12          # T int32 ops/s
    ops = MZ_INT_OPS_PER_BASE.get(k, 48) * n
    ach = ops / (phase_ms["extract"] * 1e-3) / 1e12
    tr = load_traffic("traffic_c3.json") if k == 19 else None
    # per launch: the capture holds one step's kernels (tools/evidence.sh); mz runs once per step
    mzk = [v for kk, v in (tr or {}).items() if kk.startswith("mz_fast_kernel<10, 1, 19")]
    mz_traffic = mzk[0]["dram_bytes"] / max(1, mzk[0].get("launches", 1)) if mzk else None
    tab_traffic = sum(v["dram_bytes"] for kk, v in tr.items() if kk.startswith(("nsweep", "upsweep"))) if tr else None
    roof = {"bound": "alu", "kernel": "mz_fast_kernel (a2-a7 fused, one launch per step)",
            "achieved": ach, "peak": int_peak, "unit": "Tops/s", "frac": ach / int_peak, "traffic": mz_traffic,
            "traffic_note": "DRAM bytes per launch, ncu --set full (profiles/r0x/traffic_c3.json); algorithmic "
                            f"{per_phase_bytes['extract']:.3e} B",
            "peak_kind": f"derived: {SM_COUNT} SMs x {INT32_LANES_PER_SM_CLK} int32 lanes/clk x {sm_mhz:.0f} MHz",
            "peak_measured": load_int_peak(),
            "ops_per_base": MZ_INT_OPS_PER_BASE.get(k, 48), "ms": phase_ms["extract"],
            # the same fraction with SURVEY 8(d)'s estimate of the algorithmic work (65 ops/base at
            # k=19, 35 at k=15) instead of DESIGN.md's count
            "frac_survey_ops": SURVEY_OPS_PER_BASE.get(k, 65) * n / (phase_ms["extract"] * 1e-3) / 1e12 / int_peak,
            "survey_ops_per_base": SURVEY_OPS_PER_BASE.get(k, 65)}
    tab_ach = per_phase_bytes["table"] / (phase_ms["table"] * 1e-3) / 1e9
    roof_table = {"bound": "hbm", "kernel": "seed table (3 packed-item LSD radix passes + pointer table), "
                            "from the minimizer kernel's packed items",
                  "achieved": tab_ach, "peak": hbm_peak, "unit": "GB/s", "frac": tab_ach / hbm_peak,
                  "traffic": tab_traffic,
                  "traffic_note": "DRAM bytes of the radix passes' upsweeps + downsweeps (ncu; the first "
                                  "pass's counts come from the minimizer kernel, so 2 upsweeps); the "
                                  f"SURVEY's algorithmic model is {SEEDTABLE_BYTES_PER_REC - (4 if tab32 else 0)} "
                                  f"B/entry, the 3-pass LSD on 8-byte items moves {64 if tab32 else 68} B/entry",
                  "peak_kind": peak_kind, "frac_vs_nominal_8tbs": tab_ach / 8000.0, "ms": phase_ms["table"]}
    step_bytes = sum(per_phase_bytes.values())
    step_hbm = {"achieved": step_bytes / (ms_step * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                "frac": step_bytes / (ms_step * 1e-3) / 1e9 / hbm_peak, "peak_kind": peak_kind,
                "frac_vs_nominal_8tbs": step_bytes / (ms_step * 1e-3) / 1e9 / 8000.0,
                "phase_ms": phase_ms,
                "phase_frac": {kk: per_phase_bytes[kk] / (phase_ms[kk] * 1e-3) / 1e9 / hbm_peak for kk in phase_ms}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and c3 is not None:
        v, dt, cores, mm = cpu_oracle_run(args.cpu_sample_bases)
        cpu = {"value": v, "unit": "Gbases/s", "cores": cores, "cpu_model": cpu_model(), "kind": "oracle",
               "sample": f"first {args.cpu_sample_bases} bases of C3, k={k} w={w}: oracle mz + seedtable ({dt:.1f} s)"}
    elif rank == 0 and world == 1 and not args.no_cpu_baseline:
        # C1 in full: the oracle on all host cores and on one thread (SURVEY 8(d) "a 1-thread run on C1")
        import oracle as O
        s1 = H.c1_ascii(n_total)
        res = {}
        for nt in (O.num_threads(), 1):
            prev = O.num_threads()
            O.set_num_threads(nt)
            t0 = time.perf_counter()
            kk_, pp_ = O.mz(s1, k, w)
            O.seedtable(kk_, pp_, k, bits)
            res[nt] = time.perf_counter() - t0
            O.set_num_threads(prev)
        ncores = max(res)
        cpu = {"value": n_total / res[ncores] / 1e9, "unit": "Gbases/s", "cores": ncores, "cpu_model": cpu_model(),
               "kind": "oracle", "sample": f"C1 in full ({n_total} bases): oracle mz + seedtable ({res[ncores]:.2f} s)",
               "single_thread": {"value": n_total / res[1] / 1e9, "unit": "Gbases/s", "cores": 1,
                                 "seconds": res[1]}}

    if rank == 0:
        line = {
            "metric": "minimizer extraction + seed table, Gbases/s (whole job)",
            "value": gbases, "unit": "Gbases/s", "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": ms_step, "step_ms": step_stats,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u64", "data": "synthetic",
            "config": {"workload": ("C3: 3.1 Gbp GC41% 1% N-runs" if c3 is not None else "C1: 1 Mbp uniform")
                       + (" (canonical minimizers)" if args.canonical else ""),
                       "k": k, "w": w, "bucket_bits": bits, "bases": n_total, "records": m_rec if world == 1 else None,
                       "density": m_rec / max(1, nwin_local) if world == 1 else None,
                       "l2": ("inputs (3.1 GB) >> L2 (126 MB); no flush needed" if c3 is not None else
                              "eager loop on L2-resident inputs (1 MB); cuda_graph has the L2-flushed time"),
                       "parallelism": f"shards{world}",
                       "exchange": EXCHANGE if world > 1 else None,
                       "table_positions": ("u32 (seedtable_build_items_ex, pos32; exact: C3 has < 2^32 bases)"
                                           if tab32 else "u64")},
            "roofline": roof,
            "roofline_table": roof_table,
            "hbm_step": step_hbm,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "table_pos64": pos64_line,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk_sum,
        }
        if graph is not None:
            line["cuda_graph"] = graph
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
