import torch, sys
B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
dev = torch.device("cuda", 0)
W = (torch.randn(128256, 4096, device=dev) * 0.02).to(torch.bfloat16)
h = torch.randn(B, 4096, device=dev).to(torch.bfloat16)
for _ in range(30):
    y = torch.matmul(h, W.t())
torch.cuda.synchronize()
