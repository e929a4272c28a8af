"""Experiment: stage-1 bandwidth vs W row stride / L2 residency (B=1 and B=32)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_15854_b200 as fs
dev = torch.device("cuda", 0)
for B in (1, 32):
    for (V, D) in [(128256, 4096), (128256, 4160), (126976, 4160), (128256, 4032), (152064, 3584), (8192, 4096), (16384, 4096)]:
        g = torch.Generator(device=dev); g.manual_seed(1)
        h = torch.randn(B, D, device=dev, generator=g).to(torch.bfloat16)
        W = (torch.randn(V, D, device=dev, generator=g) * 0.02).to(torch.bfloat16)
        out = torch.empty(B, dtype=torch.int32, device=dev)
        ctr = [0]
        def fn():
            ctr[0] += 1
            fs.sample(h, W, seed=1, step=ctr[0], out=out)
        t_end = time.time() + 0.5
        while time.time() < t_end:
            fn()
        torch.cuda.synchronize()
        fs.set_option("time_stage1", 1); fs.query("stage1_ms")
        bench.time_loop(fn, 100, 5)
        t = fs.query("stage1_ms") / 100
        fs.set_option("time_stage1", 0)
        gbs = (2 * V * D + 2 * B * D) / (t * 1e-3) / 1e9
        print(f"B={B:3d} V={V:7d} D={D:5d} stage1 {t*1e3:8.2f} us  {gbs:8.1f} GB/s", flush=True)
        del W, h
        torch.cuda.empty_cache()
