mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_groups -s 2 -c 1 -o gpurun_out/prof_red python tools/exp_prof.py 32 gemma3_27b > /dev/null 2>&1
ncu -i gpurun_out/prof_red.ncu-rep --page details --csv > gpurun_out/prof_red.details.csv 2>/dev/null
ncu -i gpurun_out/prof_red.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_red.source.csv 2>/dev/null
rm -f gpurun_out/prof_red.ncu-rep
