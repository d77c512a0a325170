#!/bin/bash
# Round-end GPU evidence (run under gpurun from the repo root): GPU test suite, smoke(), every
# bench line (C3 default, C1, C2, C4, lookup at 2^24 and 2^28 buckets, the reference arm), then
# the ncu launch list + full capture of the C3 step (tools/evidence.sh).  Outputs: gpurun_out/fin/.
set -u
O=gpurun_out/fin
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --durations=15 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/bench_c3_n1.json 2> $O/bench_c3.err
timeout 300 python bench.py --config c1 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --config c2 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config c4 > $O/bench_c4.json 2> $O/bench_c4.err
MZS_LOOKUP_BITS=24 timeout 600 python bench.py --config lookup > $O/bench_lookup24.json 2> $O/bench_lookup24.err
timeout 600 python bench.py --config lookup --no-cpu-baseline > $O/bench_lookup28.json 2> $O/bench_lookup28.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
bash tools/evidence.sh > $O/evidence.log 2>&1
cp -r gpurun_out/ev $O/ev 2>/dev/null
echo done
