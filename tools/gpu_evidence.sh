#!/bin/bash
# Full evidence run on the GPU box (via gpurun): GPU tests + smoke + default bench (tools/gpu_run.sh),
# then the ncu launch list and --set full captures (tools/gpu_prof.sh).  Usage: tools/gpu_evidence.sh OUTDIR
OUT=${1:-gpurun_out/evidence}
bash tools/gpu_run.sh "$OUT"
bash tools/gpu_prof.sh "$OUT/prof"
