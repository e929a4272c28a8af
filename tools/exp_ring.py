"""Stage-1 time of the plain sampling kernel vs TMA ring shape (kbps x stages), Llama-3-8B head."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_2603_15854_b200 as fs
dev = torch.device("cuda", 0)
V, D = 128256, 4096
g = torch.Generator(device=dev).manual_seed(0)
W = (torch.randn(V, D, device=dev, generator=g) * 0.02).to(torch.bfloat16)
for B in (8, 32):
    h = torch.randn(B, D, device=dev, generator=g).to(torch.bfloat16)
    out = []
    for kb, st in ((4, 3), (3, 3), (2, 5), (2, 4), (3, 2), (2, 3), (1, 8), (4, 2), (5, 2)):
        fs.set_option("kbps", kb); fs.set_option("stages", st)
        ctr = [0]
        def run():
            ctr[0] += 1
            fs.sample(h, W, seed=1, step=ctr[0])
        try:
            for _ in range(5): run()
            fs.set_option("time_stage1", 1)
            for _ in range(30): run()
            s1 = fs.query("stage1_ms") / 30 * 1e3
            fs.set_option("time_stage1", 0)
            out.append(f"{kb}x{st}={s1:6.1f}")
        except fs.FlashSampleError as e:
            fs.set_option("time_stage1", 0)
            out.append(f"{kb}x{st}=n/a")
    fs.set_option("kbps", 0); fs.set_option("stages", 0)
    print(f"B={B}: " + " ".join(out), flush=True)
