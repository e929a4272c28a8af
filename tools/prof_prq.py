import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_15854_b200 as fs
dev = torch.device("cuda", 0)
V, D, B = 128256, 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 256
g = torch.Generator(device=dev); g.manual_seed(1)
W = (torch.randn(V, D, device=dev, generator=g) * 0.02).to(torch.bfloat16)
h = torch.randn(B, D, device=dev, generator=g).to(torch.bfloat16)
seeds = torch.arange(B, device=dev, dtype=torch.int64) * 7919 + 17
out = torch.empty(B, dtype=torch.int32, device=dev)
for s in range(4):
    fs.sample(h, W, seeds=seeds, step=s, out=out)
torch.cuda.synchronize()
