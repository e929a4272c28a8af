# Power / clock per configuration (nvidia-smi sampled over the last 60% of a 3 s loop).
mkdir -p gpurun_out
export KNOB_SECS=3
python tools/exp_knobs.py '{"epi_sleep":[0,100,1000,4000]}' 1,32 > gpurun_out/exp5.txt 2>&1
python tools/exp_knobs.py '{"dbg_no_mma":[1],"dbg_no_epi":[1]}' 1,32 >> gpurun_out/exp5.txt 2>&1
(nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 100 > gpurun_out/stream_clk2.txt &)
./tools/bin/tma_stream_bench > gpurun_out/stream_const2.txt 2>&1
