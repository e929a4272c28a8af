"""Step time vs vocabulary size at fixed D and B (how the per-CTA tile remainder costs): one
kernel per step, back-to-back loop, pdl_w = 0.   python tools/v_scan.py D B V1,V2,..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_15854_b200 as fs  # noqa: E402

D, B = int(sys.argv[1]), int(sys.argv[2])
Vs = [int(x) for x in sys.argv[3].split(",")]
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(3)
Wfull = (torch.randn(max(Vs), D, device=dev, generator=g) * 0.02).to(torch.bfloat16)
h = torch.randn(B, D, device=dev, generator=g).to(torch.bfloat16)
out = torch.empty(B, dtype=torch.int32, device=dev)
fs.set_option("pdl_w", 0)
for rep in range(2):
    for V in Vs:
        W = Wfull[:V]
        ctr = [0]

        def fn():
            ctr[0] += 1
            fs.sample(h, W, seed=1, step=ctr[0], out=out)
        us = 1e3 * bench.time_loop(fn, 300, 20)
        byts = 2 * V * D + 2 * B * D
        U = (V + 15) // 16
        print(f"rep {rep} D={D} B={B} V={V:7d} units/CTA={U / 148:6.2f} tiles/CTA={V / 148 / 128:5.2f} "
              f"{us:8.2f} us  {byts / us / 1e3:7.1f} GB/s  ({byts / us / 1e3 / 6553.6:.3f} of copy peak)", flush=True)
