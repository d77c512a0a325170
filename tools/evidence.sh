#!/bin/bash
# Collect the round's GPU evidence on a B200 box (run under gpurun from the repo root):
#   the ncu launch list of one C3 step, one `ncu --set full` capture of the step's kernels
#   (summarised: per-kernel table, DRAM traffic, per-source-line instructions of the minimizer
#   kernel), and one capture per named C2 kernel.  Outputs land in gpurun_out/ev/ (the big
#   .ncu-rep files are summarised there and dropped).  Bench lines are collected separately.
set -u
O=gpurun_out/ev
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
# launch list of one timed C3 step (cold-cache, serialised: compare shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-pos64 > $O/launches_c3.log 2>&1
# full sections of the step's kernels: encode, mz, 3 x (upsweep, nsweep) of the narrow path
# (the 3 x 2 gated wide-path launches also match and are captured as no-ops); the 3 warm-up
# steps are skipped (13 matching launches per step since the first pass takes its counts from the
# minimizer kernel)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"mz_fast|^nsweep|encode_kernel|upsweep" \
  -s 39 -c 13 -o $O/full_c3 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-pos64 > $O/full_c3.log 2>&1
for cfg in "min 256 generic" "min 1024 generic" "min 1024 commutative" "min 256 commutative"; do
  set -- $cfg
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"slsum" -s 3 -c 1 \
    -o $O/full_c2_$3_$1_w$2 python tools/slsum_one.py --op $1 --w $2 --path $3 --reps 4 > $O/full_c2_$3_$1_w$2.log 2>&1
done
python tools/ncu_summary.py launches $O/launches_c3.csv --last-step encode_kernel > $O/summary_launches.md
python tools/ncu_summary.py report $O/full_c3.ncu-rep --bases 3.1e9 > $O/summary_full_c3.md 2>&1
for r in $O/full_c2_*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  python tools/ncu_summary.py report $r --bases 268435456 > $O/summary_$b.md 2>&1
done
python tools/ncu_summary.py traffic $O/full_c3.ncu-rep > $O/traffic_c3.json
python tools/src_hot.py $O/full_c3.ncu-rep mz_fast --per 3.1e9 --top 60 > $O/srchot_mz.txt 2>&1
rm -f $O/*.ncu-rep
echo done
