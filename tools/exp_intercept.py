"""Step time vs V at fixed B, D (fixed per-step overhead = intercept of the linear fit)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2603_15854_b200 as fs
dev = torch.device("cuda", 0)
D = 4096
g = torch.Generator(device=dev); g.manual_seed(1)
Wfull = (torch.randn(128256 * 2, D, device=dev, generator=g) * 0.02).to(torch.bfloat16)
for B in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,32").split(",")]:
    h = torch.randn(B, D, device=dev, generator=g).to(torch.bfloat16)
    out = torch.empty(B, dtype=torch.int32, device=dev)
    xs, ys = [], []
    for V in [148 * 128, 148 * 256, 148 * 512, 32064, 64128, 128256, 256512]:
        W = Wfull[:V]
        ctr = [0]
        def fn():
            ctr[0] += 1
            fs.sample(h, W, seed=1, step=ctr[0], out=out)
        t = bench.time_loop(fn, 200, 20) * 1e3
        xs.append(V); ys.append(t)
        print(f"B={B} V={V:6d} step {t:8.2f} us  {2*V*D/(t*1e-6)/1e9:7.1f} GB/s", flush=True)
    a = np.polyfit(np.array(xs[3:], float), np.array(ys[3:], float), 1)
    print(f"B={B} fit over V>=32064: {a[0]*1e3:.4f} us per 1000 rows ({2*D*1e3/(a[0]*1e3*1e-6)/1e9/1e3:.1f} GB/s marginal), intercept {a[1]:.2f} us", flush=True)
