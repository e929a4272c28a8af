"""Stage-1 time at large B with the debug knobs: epilogue skipped / MMA skipped (pair and 1-CTA)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_2603_15854_b200 as fs
dev = torch.device("cuda", 0)
for name in ("llama3_8b", "qwen25_7b"):
    for B in (128, 256):
        wl = bench.make_device_workload(name, B, dev)
        o = torch.empty(B, dtype=torch.int32, device=dev)
        out = []
        for pair in (1, 0):
            for de, dm in ((0, 0), (1, 0), (0, 1), (1, 1)):
                fs.set_option("pair", pair); fs.set_option("dbg_no_epi", de); fs.set_option("dbg_no_mma", dm)
                fn = bench.fused_step_fn(fs, wl, [0], o)
                for _ in range(5): fn()
                fs.set_option("time_stage1", 1)
                for _ in range(20): fn()
                t = fs.query("stage1_ms") / 20 * 1e3
                fs.set_option("time_stage1", 0)
                out.append(f"p{pair}e{de}m{dm}={t:6.1f}")
        fs.set_option("pair", -1); fs.set_option("dbg_no_epi", 0); fs.set_option("dbg_no_mma", 0)
        print(f"{name} B={B}: " + " ".join(out), flush=True)
        del wl
