# usage: bash tools/gpu_prof_opts.sh TAG B '{"pair":1}'   (kernel regex fused_tc)
TAG=$1; B=$2; OPTS=$3
mkdir -p gpurun_out
FS_OPTS="$OPTS" timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_tc -s 5 -c 1 -o gpurun_out/prof_$TAG python tools/exp_prof.py $B > gpurun_out/ncu_$TAG.log 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_$TAG.raw.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page details --csv > gpurun_out/prof_$TAG.details.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_$TAG.source.csv 2>/dev/null
rm -f gpurun_out/prof_$TAG.ncu-rep
