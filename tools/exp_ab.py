"""A/B of the fused step on selected configs (library chosen by FS_LIB_PATH)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_2603_15854_b200 as fs
dev = torch.device("cuda", 0)
cases = [("llama3_8b", 32), ("llama3_8b", 256), ("qwen25_7b", 256), ("gemma3_27b", 256), ("llama3_70b", 256)]
out = []
for name, B in cases:
    wl = bench.make_device_workload(name, B, dev)
    o = torch.empty(B, dtype=torch.int32, device=dev)
    fn = bench.fused_step_fn(fs, wl, [0], o)
    out.append(f"{name}/B{B} {1e3 * bench.time_median(fn, 60, 15):7.1f}")
    del wl
    torch.cuda.empty_cache()
print(os.environ.get("TAG", ""), " | ".join(out), flush=True)
