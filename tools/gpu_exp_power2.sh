mkdir -p gpurun_out
(nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 100 > gpurun_out/stream_clk3.txt &)
ONLY_BEST=1 ITERS=20000 ./tools/bin/tma_stream_bench r > gpurun_out/stream_long.txt 2>&1
