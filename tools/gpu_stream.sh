mkdir -p gpurun_out
(nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 200 > gpurun_out/stream_clk.txt &) 
./tools/bin/tma_stream_bench > gpurun_out/stream_const.txt 2>&1
./tools/bin/tma_stream_bench r > gpurun_out/stream_rand.txt 2>&1
