import sys, os
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_2603_15854_b200 as fs
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(1)
V, D = 128256, 4096
W = (torch.randn(V, D, device=dev, generator=g) * 0.02).to(torch.bfloat16)
fs.set_option("pdl_w", 1)
for B in (1, 8, 32, 64):
    h = torch.randn(B, D, device=dev, generator=g).to(torch.bfloat16)
    ctr = [0]
    def f():
        ctr[0] += 1
        fs.sample(h, W, seed=1, step=ctr[0], return_logprob=True)
    def plain():
        ctr[0] += 1
        fs.sample(h, W, seed=1, step=ctr[0])
    r = {}
    for fuse in (0, 1):
        fs.set_option("fuse_reduce", fuse)
        r[f"logz_fuse{fuse}"] = round(bench.time_loop(f, 200, 20) * 1e3, 1)
        r[f"plain_fuse{fuse}"] = round(bench.time_loop(plain, 200, 20) * 1e3, 1)
    print(B, r, flush=True)
