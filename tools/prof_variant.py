"""One variant of the fused step for an ncu capture: python tools/prof_variant.py {logz|grouped|qwen|prq} B"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_15854_b200 as fs
dev = torch.device("cuda", 0)
kind, B = sys.argv[1], int(sys.argv[2])
name = {"qwen": "qwen25_7b", "grouped": "gemma3_27b"}.get(kind, "llama3_8b")
wl = bench.make_device_workload(name, B, dev)
seeds = torch.arange(B, device=dev, dtype=torch.int64) * 7919 + 17
for s in range(4):
    if kind == "logz":
        fs.sample(wl["h"], wl["W"], seed=1, step=s, return_logprob=True)
    elif kind == "prq":
        fs.sample(wl["h"], wl["W"], seeds=seeds, step=s)
    else:
        bench.fused_step_fn(fs, wl, [s], torch.empty(B, dtype=torch.int32, device=dev))()
torch.cuda.synchronize()
