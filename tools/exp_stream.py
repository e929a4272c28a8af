"""Experiment: stage-1 time with and without MMAs (TMA ring streaming only), vs kbps."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_15854_b200 as fs
dev = torch.device("cuda", 0)
V, D = 128256, 4096
g = torch.Generator(device=dev); g.manual_seed(1)
W = (torch.randn(V, D, device=dev, generator=g) * 0.02).to(torch.bfloat16)
for B in (1, 32, 128, 256):
    h = torch.randn(B, D, device=dev, generator=g).to(torch.bfloat16)
    out = torch.empty(B, dtype=torch.int32, device=dev)
    ctr = [0]
    def fn():
        ctr[0] += 1
        fs.sample(h, W, seed=1, step=ctr[0], out=out)
    for nomma in (0, 1):
        for kbps in (1, 2, 3, 4):
            fs.set_option("dbg_no_mma", nomma); fs.set_option("kbps", kbps)
            try:
                t_end = time.time() + 0.3
                while time.time() < t_end:
                    fn()
                torch.cuda.synchronize()
                step = bench.time_loop(fn, 100, 5) * 1e3
                fs.set_option("time_stage1", 1); fs.query("stage1_ms")
                bench.time_loop(fn, 100, 5)
                t = fs.query("stage1_ms") / 100
                fs.set_option("time_stage1", 0)
                print(f"B={B:3d} no_mma={nomma} kbps={kbps} step {step:8.2f} us stage1 {t*1e3:8.2f} us  {2*V*D/(t*1e-3)/1e9:8.1f} GB/s (W only)", flush=True)
            except Exception as e:
                print(f"B={B} no_mma={nomma} kbps={kbps} error {e}")
                fs.set_option("time_stage1", 0)
    fs.set_option("dbg_no_mma", 0); fs.set_option("kbps", 0)
