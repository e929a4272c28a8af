set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_b32.csv python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu > /dev/null 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_tc -s 5 -c 1 -o gpurun_out/prof_b32 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu > gpurun_out/ncu_full_b32.log 2>&1; echo ncu2 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_tc -s 5 -c 1 -o gpurun_out/prof_b256 python bench.py --B 256 --steps 10 --warmup 3 --no-sweep --no-cpu > gpurun_out/ncu_full_b256.log 2>&1; echo ncu3 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_tc -s 5 -c 1 -o gpurun_out/prof_b1 python bench.py --B 1 --steps 10 --warmup 3 --no-sweep --no-cpu > gpurun_out/ncu_full_b1.log 2>&1; echo ncu4 rc=$?
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
