#!/bin/bash
# One gpurun call: ncu launch list + one `ncu --set full` capture of one step of
# `bench.py --config ties` (after the plain run has exited 0), summarised into
# gpurun_out/ties/ (traffic_ties.json feeds the bench line's roofline.traffic), then the
# bench line itself, never under ncu.
O=gpurun_out/ties; mkdir -p $O
B="python bench.py --config ties --steps 1 --warmup 3 --no-cpu-baseline"
$B > $O/plain.json 2> $O/plain.err || { echo "plain run failed"; tail $O/plain.err; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_ties.csv \
  $B > $O/ncu_launch.log 2>&1
# the last step's six kernels: skip the 3 warm-up steps (18 launches of these names)
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"ties_|slsum_generic_warp|encode_kernel" -s 18 -c 6 -o $O/full_ties -f \
  $B > $O/ncu_full.log 2>&1
python tools/ncu_summary.py launches $O/launches_ties.csv --last-step encode_kernel > $O/ncu_launches_ties.md
python tools/ncu_summary.py report $O/full_ties.ncu-rep --bases 4e8 > $O/ncu_summary_full_ties.md 2>&1
python tools/ncu_summary.py traffic $O/full_ties.ncu-rep > $O/traffic_ties.json && cp $O/traffic_ties.json profiles/r02/traffic_ties.json
rm -f $O/*.ncu-rep
python bench.py --config ties > $O/bench_ties.json 2> $O/bench_ties.err
cat $O/traffic_ties.json; cat $O/bench_ties.json; tail -n 3 $O/bench_ties.err
