#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over tools/sanitize_cases.py (every kernel
# family on small inputs, each result checked against the oracle).  Run under gpurun from the
# repo root; summaries land in gpurun_out/san/.
set -u
O=gpurun_out/san
mkdir -p $O
for tool in racecheck synccheck memcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_cases.py > $O/$tool.txt 2>&1
  echo "exit=$?" >> $O/$tool.txt
done
grep -h -E "ERROR SUMMARY|RACECHECK SUMMARY|exit=|all cases ok" $O/*.txt
