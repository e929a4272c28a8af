"""Where the MMA issuer of the fused kernel waits (debug option dbg_times, slots 6 / 7): total ns per
step blocked on a drained TMEM accumulator (the epilogue is behind) and on landed operands (the TMA
ring is behind), as a share of the kernel's duration, per config and batch size.

    python tools/mma_waits.py llama3_8b 32,128,256
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_15854_b200 as fs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama3_8b"
Bs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "32,128,256").split(",")]
dev = torch.device("cuda", 0)
fs.set_option("pdl_w", 0)
for B in Bs:
    wl = bench.make_device_workload(name, B, dev)
    out = torch.empty(B, dtype=torch.int32, device=dev)
    fn = bench.fused_step_fn(fs, wl, [0], out)
    for _ in range(30):
        fn()
    torch.cuda.synchronize()
    n = 10
    bufs = [torch.zeros(148 * 8, dtype=torch.int64, device=dev) for _ in range(n)]
    for s in range(n):
        fs.set_option("dbg_times", bufs[s].data_ptr())
        fn()
    fs.set_option("dbg_times", 0)
    torch.cuda.synchronize()
    A = np.stack([b.cpu().numpy().reshape(148, 8) for b in bufs]).astype(np.float64)
    G = int((A[0, :, 0] > 0).sum())
    A = A[:, :G]
    end = np.where(A[:, :, 5] > 0, A[:, :, 5], A[:, :, 3])                 # CTA done, else last tile drained
    dur = (end.max(1) - A[:, :, 0].min(1)) / 1e3                          # kernel span, us
    mma = A[:, :, 6] + A[:, :, 7] > 0                                       # CTAs that issue MMAs
    acc = np.array([A[s, mma[s], 6].mean() for s in range(n)]) / 1e3
    dat = np.array([A[s, mma[s], 7].mean() for s in range(n)]) / 1e3
    print(f"{name} B={B:4d} grid {G}: kernel {np.median(dur):7.1f} us; MMA issuer waits on the accumulator "
          f"{np.median(acc):6.1f} us ({np.median(acc / dur):.0%}), on operands {np.median(dat):6.1f} us "
          f"({np.median(dat / dur):.0%})", flush=True)
    del wl
    torch.cuda.empty_cache()
