mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 400 python bench.py --no-cpu > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python tools/summarize_bench.py gpurun_out/bench_quick.json
for B in 32 256; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_tc -s 5 -c 1 -o gpurun_out/prof_b$B python bench.py --B $B --steps 10 --warmup 3 --no-sweep --no-cpu > /dev/null 2>&1
ncu -i gpurun_out/prof_b$B.ncu-rep --page raw --csv > gpurun_out/prof_b$B.raw.csv 2>/dev/null
ncu -i gpurun_out/prof_b$B.ncu-rep --page details --csv > gpurun_out/prof_b$B.details.csv 2>/dev/null
ncu -i gpurun_out/prof_b$B.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_b$B.source.csv 2>/dev/null
rm -f gpurun_out/prof_b$B.ncu-rep
done
ls -la gpurun_out
