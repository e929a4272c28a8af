mkdir -p gpurun_out
python -c "import paper_2603_15854_b200" || exit 1
timeout 900 python -m pytest tests/test_gpu_topk_fused.py tests/test_gpu_topk.py -x -q > gpurun_out/pytest_topk.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_topk.log
timeout 600 python tools/exp_topk_fused.py 2>&1 | tail -12
