# pytest -m gpu + racecheck only (after a kernel change)
mkdir -p gpurun_out
python -c "import paper_2603_15854_b200" || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_racecheck.log 2>&1
echo "racecheck rc=$?"; tail -4 gpurun_out/sanitize_racecheck.log
