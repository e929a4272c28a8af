mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_tc -s 2 -c 1 -o gpurun_out/prof_prq python tools/prof_prq.py 256 > /dev/null 2>&1
ncu -i gpurun_out/prof_prq.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_prq.source.csv 2>/dev/null
ncu -i gpurun_out/prof_prq.ncu-rep --page details --csv > gpurun_out/prof_prq.details.csv 2>/dev/null
rm -f gpurun_out/prof_prq.ncu-rep
