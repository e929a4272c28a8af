# Evidence run on one B200: GPU tests, smoke, full bench (all configs), reference arm, ncu launch list,
# ncu --set full of the fused kernel at B = 1, 32, 256 (llama3_8b), compute-sanitizer.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/gpu_info.csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/bench.err
python tools/summarize_bench.py gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_b32.csv python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu > /dev/null 2>&1; echo "ncu launches rc=$?"
for B in 32 1 256; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_tc -s 5 -c 1 -o gpurun_out/prof_b$B python bench.py --B $B --steps 10 --warmup 3 --no-sweep --no-cpu > /dev/null 2>&1
ncu -i gpurun_out/prof_b$B.ncu-rep --page raw --csv > gpurun_out/prof_b$B.raw.csv 2>/dev/null
ncu -i gpurun_out/prof_b$B.ncu-rep --page details --csv > gpurun_out/prof_b$B.details.csv 2>/dev/null
ncu -i gpurun_out/prof_b$B.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_b$B.source.csv 2>/dev/null
rm -f gpurun_out/prof_b$B.ncu-rep
done
bash tools/gpu_sanitize.sh
ls gpurun_out | head -40
