# Load-path / MMA / epilogue isolation at large B (debug knobs dbg_no_mma = 1 no MMA, 2 no TMA), with clocks.
mkdir -p gpurun_out
python tools/exp_knobs.py '{"dbg_no_mma":[0,1,2],"dbg_no_epi":[0,1]}' 32,128,256 > gpurun_out/exp3.txt 2>&1
