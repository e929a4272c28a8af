"""One configuration of the fused top-k path, for ncu: B mode k."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_15854_b200 as fs
B, mode, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dev = torch.device("cuda", 0)
V, D = 128256, 4096
g = torch.Generator(device=dev).manual_seed(0)
W = (torch.randn(V, D, device=dev, generator=g) * 0.02).to(torch.bfloat16)
h = torch.randn(B, D, device=dev, generator=g).to(torch.bfloat16)
fs.set_option("topk_mode", mode)
fs.set_option("dbg_no_mma", int(os.environ.get("DBG_NO_MMA", "0")))
for s in range(4):
    fs.sample(h, W, seed=1, step=s, top_k=K, top_p=0.95)
torch.cuda.synchronize()
