#!/bin/bash
# Collect the round's GPU evidence on a B200 box (run under gpurun from the repo root):
#   tests, the bench lines (C3 default, C2, C4, reference arm), the ncu launch list of one C3
#   step and one `ncu --set full` capture of the top kernels.  Outputs land in gpurun_out/ev/.
set -u
O=gpurun_out/ev
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c2 --steps 10 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --config c4 --steps 5 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python bench.py --config c1 --steps 3000 > $O/bench_c1.json 2> $O/bench_c1.err
# launch list of one timed C3 step (cold-cache, serialised: compare shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/launches_c3.log 2>&1
# full sections of the top kernels of the C3 step (after 3 warm-up steps) and of slsum (C2)
# one step matches 14 kernels (encode, mz, 3 packed passes x (upsweep, nsweep), and the wide
# path's 3 x 2 enqueued-but-gated ones); skip the 3 warm-up steps, capture the timed one
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mz_fast|^nsweep|encode_kernel|upsweep" \
  -s 42 -c 14 -o $O/full_c3 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/full_c3.log 2>&1
# one named C2 configuration per capture (tools/slsum_one.py launches exactly 4 slsum kernels;
# the 4th, warm one is captured)
for cfg in "min 16 generic" "min 1024 generic" "min 4 commutative" "min 1024 commutative" "add 64 recurrent"; do
  set -- $cfg
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"slsum" -s 3 -c 1 \
    -o $O/full_c2_$3_$1_w$2 python tools/slsum_one.py --op $1 --w $2 --path $3 --reps 4 > $O/full_c2_$3_$1_w$2.log 2>&1
done
timeout 600 python bench.py --config lookup --steps 5 > $O/bench_lookup.json 2> $O/bench_lookup.err
# summaries are made here (gpurun copies back at most 64 MiB): launch list, --set full table,
# per-kernel DRAM traffic; the large reports are then dropped
python tools/ncu_summary.py launches $O/launches_c3.csv --last-step encode_kernel > $O/summary_launches.md
python tools/ncu_summary.py report $O/full_c3.ncu-rep --bases 3.1e9 > $O/summary_full_c3.md 2>&1
for r in $O/full_c2_*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  python tools/ncu_summary.py report $r --bases 268435456 > $O/summary_$b.md 2>&1
done
python tools/ncu_summary.py traffic $O/full_c3.ncu-rep > $O/traffic_c3.json
python tools/src_hot.py $O/full_c3.ncu-rep mz_fast --per 3.1e9 --top 40 > $O/srchot_mz.txt 2>&1
rm -f $O/*.ncu-rep
echo done
