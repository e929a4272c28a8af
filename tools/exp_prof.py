"""Run a few fused steps with library options from FS_OPTS (json) -- target for ncu captures."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_15854_b200 as fs
B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
name = sys.argv[2] if len(sys.argv) > 2 else "llama3_8b"
for k, v in json.loads(os.environ.get("FS_OPTS", "{}")).items():
    fs.set_option(k, v)
wl = bench.make_device_workload(name, B, torch.device("cuda", 0))
out = torch.empty(B, dtype=torch.int32, device="cuda")
fn = bench.fused_step_fn(fs, wl, [0], out)
for _ in range(8):
    fn()
torch.cuda.synchronize()
