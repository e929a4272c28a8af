# usage: bash tools/gpu_prof.sh TAG "bench args"   -> gpurun_out/prof_TAG.{ncu-rep,raw.csv,source.csv}
TAG=$1; shift
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_tc -s 5 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu "$@" > gpurun_out/ncu_$TAG.log 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_$TAG.raw.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page details --csv > gpurun_out/prof_$TAG.details.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_$TAG.source.csv 2>/dev/null
ls -la gpurun_out/prof_$TAG*
