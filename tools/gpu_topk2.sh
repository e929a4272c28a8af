mkdir -p gpurun_out
python -c "import paper_2603_15854_b200" || exit 1
timeout 900 python -m pytest tests/test_gpu_topk_fused.py tests/test_gpu_topk.py -x -q 2>&1 | tail -3
timeout 600 python tools/exp_topk_stage.py 50 2>&1 | tail -8
timeout 600 python tools/exp_topk_stage.py 200 2>&1 | tail -8
