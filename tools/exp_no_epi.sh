mkdir -p gpurun_out/exp1
cd $GRAFT_REPO_ROOT
timeout 120 compute-sanitizer --tool racecheck tools/bin/racecheck_tmem_pair > gpurun_out/exp1/racecheck_repro.log 2>&1
tools/bin/racecheck_tmem_pair >> gpurun_out/exp1/racecheck_repro.log 2>&1
for c in llama3_8b qwen25_7b gemma3_27b; do
  timeout 600 python tools/sweep_opts.py $c 128,256 '{"dbg_no_epi": [0, 1]}' >> gpurun_out/exp1/no_epi.log 2>&1
done
