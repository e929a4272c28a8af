#!/bin/bash
# Round-2 A/B experiments on the GPU box (via gpurun), logs under gpurun_out/<out>/ (summarised in
# DESIGN.md §11 and copied to profiles/r02/).  Usage: tools/ab.sh <experiment> [out]
#   no_epi   epilogue off (dbg_no_epi) at B = 128 / 256                    (§11 entry 18)
#   wait     epilogue barrier waits: spin vs suspend hint                 (entry 19)
#   energy   NVML energy split: full / no epilogue / no MMA / no loads    (entry 22)
#   stage2   grouped stage-2 kernels (warp / lanes / block per row): ncu durations + step A/B
#   race     racecheck of the paired-TMEM-allocation reproducer            (§1 sanitizers)
EXP=${1:?experiment}
OUT=gpurun_out/${2:-$EXP}
mkdir -p $OUT
case $EXP in
  no_epi)
    for c in llama3_8b qwen25_7b gemma3_27b; do
      timeout 600 python tools/sweep_opts.py $c 128,256 '{"dbg_no_epi": [0, 1]}' >> $OUT/no_epi.log 2>&1; done ;;
  wait)
    for c in llama3_8b qwen25_7b gemma3_27b; do
      timeout 900 python tools/sweep_opts.py $c 32,128,256 '{"spin_wait": [1, 0]}' >> $OUT/wait.log 2>&1; done ;;
  energy)
    timeout 600 python tools/energy_split.py llama3_8b 32,128,256 > $OUT/energy.log 2>&1
    timeout 400 python tools/energy_split.py gemma3_27b 256 >> $OUT/energy.log 2>&1 ;;
  stage2)
    cat > /tmp/stage2_calls.py <<'PY'
import sys, os, torch
sys.path.insert(0, os.getcwd())
import bench, synth, paper_2603_15854_b200 as fs
dev = torch.device("cuda", 0)
for B in (1, 32, 128, 256):
    wl = bench.make_device_workload("gemma3_27b", B, dev)
    out = torch.empty(B, dtype=torch.int32, device=dev)
    fn = bench.fused_step_fn(fs, wl, [0], out)
    for kern in (1, 2, 3):
        fs.set_option("grp_kernel", kern)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        print("B", B, "grp_kernel", kern, flush=True)
    del wl
    torch.cuda.empty_cache()
PY
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:reduce_groups --csv \
      --log-file $OUT/stage2_ncu.csv python /tmp/stage2_calls.py > $OUT/stage2_calls.log 2>&1
    timeout 900 python tools/sweep_opts.py gemma3_27b 1,32,128,256 '{"grp_kernel": [1, 2, 3]}' > $OUT/stage2_ab.log 2>&1 ;;
  race)
    for variant in 0 1 2 3 4 5 6 7 9 13 15; do
      timeout 300 compute-sanitizer --tool racecheck tools/bin/racecheck_tmem_pair 2 $variant >> $OUT/racecheck_repro.log 2>&1
      echo "pair variant=$variant rc=$?" >> $OUT/racecheck_repro.log
    done ;;
  *) echo "unknown experiment $EXP"; exit 2 ;;
esac
