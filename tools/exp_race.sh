#!/bin/bash
OUT=gpurun_out/${1:-race}
mkdir -p $OUT
for b in racecheck_tmem_pair racecheck_tmem_pair_shared; do
  echo "== $b (no sanitizer)" >> $OUT/race.log; timeout 60 tools/bin/$b >> $OUT/race.log 2>&1; echo "rc=$?" >> $OUT/race.log
  for tool in memcheck racecheck; do
    echo "== $b $tool" >> $OUT/race.log
    timeout 120 compute-sanitizer --tool $tool tools/bin/$b >> $OUT/race.log 2>&1; echo "rc=$?" >> $OUT/race.log
  done
done
