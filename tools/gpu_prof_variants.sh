mkdir -p gpurun_out
for v in logz grouped qwen; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_tc -s 2 -c 1 -o gpurun_out/prof_$v python tools/prof_variant.py $v 256 > /dev/null 2>&1
ncu -i gpurun_out/prof_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_$v.source.csv 2>/dev/null
ncu -i gpurun_out/prof_$v.ncu-rep --page details --csv > gpurun_out/prof_$v.details.csv 2>/dev/null
rm -f gpurun_out/prof_$v.ncu-rep
done
