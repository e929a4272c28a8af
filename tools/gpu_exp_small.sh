# Small-B load path: fused kernel vs bare TMA ring (tools/bin/tma_stream_bench, 150 us best).
mkdir -p gpurun_out
python tools/exp_knobs.py '{"dbg_no_mma":[0,1],"dbg_no_epi":[0,1],"unit_rows":[16,128]}' 1,32 > gpurun_out/exp4.txt 2>&1
python tools/exp_knobs.py '{"kbps":[2,3,4],"stages":[0,2,3,4]}' 1,32 >> gpurun_out/exp4.txt 2>&1
python tools/exp_knobs.py '{"max_ctas":[148,146,144,140,132,120]}' 1,32 >> gpurun_out/exp4.txt 2>&1
