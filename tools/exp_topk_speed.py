"""Top-k / top-p speed: standalone over materialised fp32 logits and fused through the LM head."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_15854_b200 as fs
dev = torch.device("cuda", 0)
V, D = 128256, 4096
g = torch.Generator(device=dev); g.manual_seed(1)
W = (torch.randn(V, D, device=dev, generator=g) * 0.02).to(torch.bfloat16)
import flashinfer.sampling as fis
for B in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,32,128,256").split(",")]:
    h = torch.randn(B, D, device=dev, generator=g).to(torch.bfloat16)
    lg = torch.matmul(h, W.t()).float()
    ctr = [0]
    def sl():
        ctr[0] += 1
        fs.sample_logits(lg, seed=1, step=ctr[0], top_k=50, top_p=0.95)
    def fused():
        ctr[0] += 1
        fs.sample(h, W, seed=1, step=ctr[0], top_k=50, top_p=0.95)
    def fi():
        fis.top_k_top_p_sampling_from_logits(lg, 50, 0.95)
    r = {n: round(bench.time_median(f, 50, 10) * 1e3, 1) for n, f in (("ours_logits", sl), ("flashinfer", fi), ("ours_fused", fused))}
    print(f"B={B}: {r}", flush=True)
