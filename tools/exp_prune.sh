#!/bin/bash
# A/B of the exact Gumbel pruning (option prune) + the GPU tests it touches
OUT=gpurun_out/${1:-r02e}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_prune.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_requests.py tests/test_gpu_onekernel.py -q -x -p no:cacheprovider > $OUT/pytest_sel.log 2>&1
echo rc=$? >> $OUT/pytest_sel.log
for c in llama3_8b qwen25_7b llama3_70b; do
  timeout 600 python tools/sweep_opts.py $c 1,32,128,256 '{"prune": [0, 1]}' >> $OUT/prune.log 2>&1
done
V=16032 D=8192 SHARD=1 PDL=0 timeout 300 python tools/cta_timeline.py 1,32 > $OUT/timeline_n8.log 2>&1
V=16032 D=8192 SHARD=0 PDL=0 timeout 300 python tools/cta_timeline.py 1,32 >> $OUT/timeline_n8.log 2>&1
