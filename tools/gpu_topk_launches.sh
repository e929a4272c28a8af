mkdir -p gpurun_out
python -c "import paper_2603_15854_b200" || exit 1
for cfg in "1 1 50" "32 1 50" "1 2 50" "32 2 50"; do
  set -- $cfg
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/exp_topk_one.py $1 $2 $3 2>/dev/null | grep -v "^==" | awk -F'","' '{print $5" "$NF}' | tail -4 | sed "s/^/B=$1 mode=$2: /"
done
timeout 600 ncu --set full --clock-control none --import-source on --sampling-interval 0 -k regex:topk_final -s 2 -c 1 -o gpurun_out/prof_topkf python tools/exp_topk_one.py 1 1 50 > /dev/null 2>&1
ncu -i gpurun_out/prof_topkf.ncu-rep --page details --csv > gpurun_out/prof_topkf.details.csv 2>/dev/null
ncu -i gpurun_out/prof_topkf.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_topkf.source.csv 2>/dev/null
rm -f gpurun_out/prof_topkf.ncu-rep
