timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_requests.py tests/test_gpu_topk_fused.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
for i in 1 2; do
  TAG=old FS_LIB_PATH=$PWD/tools/bin/libflashsample_old.so python tools/exp_ab.py
  TAG=new python tools/exp_ab.py
done
