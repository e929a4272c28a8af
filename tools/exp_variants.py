"""Step time of the sampling variants (plain / temperature / per-request seeds / log-mass / grouped)
at large B, per kernel choice (pair on/off) -- where the epilogue, not the stream, sets the pace."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_15854_b200 as fs
dev = torch.device("cuda", 0)
V, D = 128256, 4096
g = torch.Generator(device=dev); g.manual_seed(1)
W = (torch.randn(V, D, device=dev, generator=g) * 0.02).to(torch.bfloat16)
fs.set_option("pdl_w", 1)
for B in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "128,256").split(",")]:
    h = torch.randn(B, D, device=dev, generator=g).to(torch.bfloat16)
    tau = torch.full((B,), 0.7, device=dev)
    seeds = torch.arange(B, device=dev, dtype=torch.int64) * 7919 + 17
    out = torch.empty(B, dtype=torch.int32, device=dev)
    ctr = [0]
    variants = {
        "plain": lambda: fs.sample(h, W, seed=1, step=ctr[0], out=out),
        "tau": lambda: fs.sample(h, W, temperature=tau, seed=1, step=ctr[0], out=out),
        "prq": lambda: fs.sample(h, W, seeds=seeds, step=ctr[0], out=out),
        "logz": lambda: fs.sample(h, W, seed=1, step=ctr[0], return_logprob=True),
        "grouped4096": lambda: fs.sample_grouped(h, W, group_size=4096, seed=1, step=ctr[0], return_groups=True),
    }
    for pair in (1, 0):
        fs.set_option("pair", pair)
        for epi in (0, 1):
            fs.set_option("dbg_no_epi", epi)
            row = []
            for name, f in variants.items():
                def fn():
                    ctr[0] += 1
                    f()
                t = bench.time_loop(fn, 50, 5) * 1e3
                row.append(f"{name} {t:7.1f}")
            print(f"B={B} pair={pair} no_epi={epi}: " + " | ".join(row), flush=True)
    fs.set_option("pair", -1)
    fs.set_option("dbg_no_epi", 0)
