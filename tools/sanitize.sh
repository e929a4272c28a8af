#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel variant (tools/sanitize_cases.py)
# and the paired-TMEM-allocation reproducer (tools/racecheck_tmem_pair.cu, loaded as a library).
OUT=${1:-gpurun_out/sanitizer}
mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > $OUT/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/sanitize_$tool.log
done
for variant in 0 7; do
  timeout 300 compute-sanitizer --tool racecheck tools/bin/racecheck_tmem_pair 2 $variant >> $OUT/racecheck_repro.log 2>&1
  echo "pair variant=$variant rc=$?" >> $OUT/racecheck_repro.log
done
