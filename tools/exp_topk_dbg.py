import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_2603_15854_b200 as fs
dev = torch.device("cuda", 0)
V, D = 128256, 4096
g = torch.Generator(device=dev).manual_seed(0)
W = (torch.randn(V, D, device=dev, generator=g) * 0.02).to(torch.bfloat16)
fs.set_option("topk_mode", 1)
for B in (1, 8, 32):
    h = torch.randn(B, D, device=dev, generator=g).to(torch.bfloat16)
    out = []
    for dbg_epi, dbg_mma in ((0, 0), (1, 0), (2, 0), (0, 1), (2, 1)):
        fs.set_option("dbg_no_epi", dbg_epi); fs.set_option("dbg_no_mma", dbg_mma)
        ctr = [0]
        def run():
            ctr[0] += 1
            fs.sample(h, W, seed=1, step=ctr[0], top_k=50)
        for _ in range(5): run()
        fs.set_option("time_stage1", 1)
        for _ in range(30): run()
        s1 = fs.query("stage1_ms") / 30 * 1e3
        fs.set_option("time_stage1", 0)
        out.append(f"epi{dbg_epi}/mma{dbg_mma}={s1:6.1f}")
    fs.set_option("dbg_no_epi", 0); fs.set_option("dbg_no_mma", 0)
    print(f"B={B}: " + " ".join(out), flush=True)
