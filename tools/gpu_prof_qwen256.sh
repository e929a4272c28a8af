mkdir -p gpurun_out
python -c "import paper_2603_15854_b200" || exit 1
for cfg in "qwen25_7b 0" "qwen25_7b 1"; do set -- $cfg
FS_OPTS="{\"dbg_no_mma\": $2}" timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_tc2 -s 3 -c 1 -o gpurun_out/prof_q256 python tools/exp_prof.py 256 $1 > /dev/null 2>&1
ncu -i gpurun_out/prof_q256.ncu-rep --page details --csv > gpurun_out/prof_q256_m$2.details.csv 2>/dev/null
ncu -i gpurun_out/prof_q256.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_q256_m$2.source.csv 2>/dev/null
rm -f gpurun_out/prof_q256.ncu-rep
done
