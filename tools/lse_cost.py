"""What the log-mass epilogue costs: the same LM head sampled plainly (fs.sample) and with per-group
log-masses (fs.sample_grouped), step loop (pdl_w = 0), interleaved A B A B so that clock drift under
the power cap hits both alike.  Also the epilogue-free bound (option dbg_no_epi) of each.

    python tools/lse_cost.py gemma3_27b 128,256 [group_size]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
import paper_2603_15854_b200 as fs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "gemma3_27b"
Bs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "32,128,256").split(",")]
G = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
REPS = int(os.environ.get("REPS", "3"))
STEPS = int(os.environ.get("STEPS", "200"))
dev = torch.device("cuda", 0)
fs.set_option("pdl_w", 0)
for B in Bs:
    wl = bench.make_device_workload(name, B, dev)
    out = torch.empty(B, dtype=torch.int32, device=dev)
    ctr = [0]

    def plain():
        ctr[0] += 1
        fs.sample(wl["h"], wl["W"], bias=wl["bias"], temperature=wl["temperature"], mask=wl["mask"],
                  seed=synth.SAMPLING_SEED, step=ctr[0], out=out)

    def grouped():
        ctr[0] += 1
        fs.sample_grouped(wl["h"], wl["W"], group_size=G, bias=wl["bias"], temperature=wl["temperature"],
                          mask=wl["mask"], seed=synth.SAMPLING_SEED, step=ctr[0], return_groups=True)

    t_end = time.time() + 1.0
    while time.time() < t_end:
        for _ in range(50):
            plain()
        torch.cuda.synchronize()
    res = {}
    for rep in range(REPS):
        for noepi in (0, 1):
            fs.set_option("dbg_no_epi", noepi)
            for tag, fn in (("plain", plain), ("grouped", grouped)):
                with bench.ClockSampler(0) as clk:
                    us = 1e3 * bench.time_loop(fn, STEPS, 10)
                res.setdefault((tag, noepi), []).append((us, clk.summary()["sm_mhz"]))
    fs.set_option("dbg_no_epi", 0)
    for (tag, noepi), runs in sorted(res.items()):
        us = sorted(r[0] for r in runs)[len(runs) // 2]
        mhz = sorted(r[1] for r in runs)[len(runs) // 2]
        print(f"{name} B={B:4d} g={G} {tag:8s} no_epi={noepi}: {us:8.2f} us  sm {mhz} MHz  runs "
              f"{[round(r[0], 1) for r in runs]}", flush=True)
