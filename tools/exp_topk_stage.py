"""Fused top-k: stage-1 time (events) vs whole call, per route, Llama-3-8B head, k=50 p=0.95."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_2603_15854_b200 as fs
dev = torch.device("cuda", 0)
V, D = 128256, 4096
g = torch.Generator(device=dev).manual_seed(0)
W = (torch.randn(V, D, device=dev, generator=g) * 0.02).to(torch.bfloat16)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 50
for B in (1, 8, 32, 64, 128):
    h = torch.randn(B, D, device=dev, generator=g).to(torch.bfloat16)
    ctr = [0]
    out = []
    for mode in (1, 2):
        fs.set_option("topk_mode", mode)
        def run():
            ctr[0] += 1
            fs.sample(h, W, seed=1, step=ctr[0], top_k=K, top_p=0.95)
        try:
            t = bench.time_median(run, 30, 5) * 1e3
            fs.set_option("time_stage1", 1)
            for _ in range(20):
                run()
            s1 = fs.query("stage1_ms") / 20 * 1e3
            fs.set_option("time_stage1", 0)
            out.append(f"mode{mode} total {t:7.1f} stage1 {s1:7.1f}")
        except fs.FlashSampleError:
            out.append(f"mode{mode} n/a")
    fs.set_option("topk_mode", 0)
    print(f"B={B:4d} k={K} " + " | ".join(out), flush=True)
