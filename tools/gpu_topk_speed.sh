mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_topk_fused.py -q -x -p no:cacheprovider > gpurun_out/pytest_topk.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_topk.log
python tools/exp_topk_speed.py > gpurun_out/exp14.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/topk_launches.csv python tools/exp_topk_speed.py 128 > /dev/null 2>&1
