#!/bin/bash
# A/B: epilogue barrier waits with / without the suspend-time hint, x Gumbel pruning on / off
OUT=gpurun_out/${1:-r02f}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_prune.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > $OUT/pytest_sel.log 2>&1
echo rc=$? >> $OUT/pytest_sel.log
for c in llama3_8b qwen25_7b gemma3_27b; do
  timeout 900 python tools/sweep_opts.py $c 32,128,256 '{"spin_wait": [1, 0], "prune": [0, 1]}' >> $OUT/wait.log 2>&1
done
timeout 120 compute-sanitizer --tool racecheck tools/bin/racecheck_tmem_pair > $OUT/racecheck_repro.log 2>&1
echo "sanitizer rc=$?" >> $OUT/racecheck_repro.log
