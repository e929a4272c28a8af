"""Fused top-k / top-p through the LM head vs cuBLAS + FlashInfer top_k_top_p (FI1), Llama-3-8B head."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_2603_15854_b200 as fs
import flashinfer.sampling as fis
dev = torch.device("cuda", 0)
V, D = 128256, 4096
g = torch.Generator(device=dev).manual_seed(0)
W = (torch.randn(V, D, device=dev, generator=g) * 0.02).to(torch.bfloat16)
for B in (1, 8, 32, 64, 128, 256):
    h = torch.randn(B, D, device=dev, generator=g).to(torch.bfloat16)
    ctr = [0]
    res = {}
    for name, mode in (("lists", 1), ("raw", 2), ("auto", 0)):
        fs.set_option("topk_mode", mode)
        def run():
            ctr[0] += 1
            fs.sample(h, W, seed=1, step=ctr[0], top_k=50, top_p=0.95)
        try:
            res[name] = bench.time_median(run, 50, 10) * 1e3
        except fs.FlashSampleError as e:
            res[name] = float("nan")
    fs.set_option("topk_mode", 0)
    def plain():
        ctr[0] += 1
        fs.sample(h, W, seed=1, step=ctr[0])
    res["plain"] = bench.time_median(plain, 50, 10) * 1e3
    def fi1():
        lg = h @ W.t()
        fis.top_k_top_p_sampling_from_logits(lg, 50, 0.95)
    res["fi1"] = bench.time_median(fi1, 50, 10) * 1e3
    print(f"B={B:4d} " + "  ".join(f"{k} {v:8.2f}" for k, v in res.items()), flush=True)
