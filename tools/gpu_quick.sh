# quick GPU iteration: parity tests + bench summary + kernel launch list (B=32)
mkdir -p gpurun_out
timeout 700 python -m pytest tests/test_gpu_rng.py tests/test_gpu_parity.py tests/test_gpu_grouped_tp.py -x -q -p no:cacheprovider --timeout 200 2>&1 | tail -3
timeout 400 python bench.py --no-cpu "$@" > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python tools/summarize_bench.py gpurun_out/bench_quick.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fused|reduce" -s 10 -c 8 --csv python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu 2>/dev/null | grep -E "gpu__time" | awk -F'","' '{print $5, $(NF)}' | cut -c1-120
