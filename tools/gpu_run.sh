#!/bin/bash
# Usage (on the GPU box, via gpurun): tools/gpu_run.sh OUTDIR -- runs the GPU test suite, smoke and
# the default bench, logging under OUTDIR (gpurun_out/...).
set -u
OUT=${1:-gpurun_out/run}
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > "$OUT/smi.txt" 2>&1
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q ${PYTEST_ARGS:--x} --durations=30 -p no:cacheprovider > "$OUT/pytest_gpu.log" 2>&1
echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
echo "smoke rc=$?" >> "$OUT/smoke.log"
if [ -z "${NO_BENCH:-}" ]; then
  t0=$(date +%s)
  timeout ${BENCH_TIMEOUT:-900} python bench.py ${BENCH_ARGS:-} > "$OUT/bench.log" 2>&1
  echo "bench rc=$? wall_s=$(( $(date +%s) - t0 ))" >> "$OUT/bench.log"
fi
