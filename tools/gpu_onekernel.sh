mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_onekernel.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_onek.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_onek.log
python tools/exp_knobs.py '{"fuse_reduce":[0,1],"pdl_w":[0,1]}' 1,32,128,256 > gpurun_out/exp7.txt 2>&1
python tools/exp_intercept.py 1,32 > gpurun_out/exp7b.txt 2>&1
