#!/bin/bash
# ncu evidence (on the GPU box via gpurun): launch list of the headline bench command and one
# `--set full` capture per (config, B) of the stage-1 kernels.  Usage: tools/gpu_prof.sh OUTDIR [specs...]
set -u
OUT=${1:-gpurun_out/prof}; shift || true
SPECS=${@:-llama3_8b:1,32,256 qwen25_7b:1,32,256 gemma3_27b:1,32,256 llama3_70b:1,32,256 llama3_70b_n2:32 llama3_70b_n4:32 llama3_70b_n8:1,32,256}
mkdir -p "$OUT"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$OUT/launches_b32.csv" \
  python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu > "$OUT/launches_bench.log" 2>&1
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -f -o "$OUT/full" \
  python tools/ncu_capture.py $SPECS > "$OUT/full_capture.log" 2>&1
echo "ncu rc=$?" >> "$OUT/full_capture.log"
ncu -i "$OUT/full.ncu-rep" --page raw --csv > "$OUT/full_raw.csv" 2>/dev/null
ncu -i "$OUT/full.ncu-rep" --page details --csv > "$OUT/full_details.csv" 2>/dev/null
