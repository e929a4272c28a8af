"""Interleaved A/B of a library option by energy per step (NVML total-energy counter over ~1.5 s of
back-to-back steps per arm) and time per step -- under the power cap the joules are the steadier
measure.

    python tools/energy_ab.py llama3_8b 128,256 epi_bar 0,1
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml as nv  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_15854_b200 as fs  # noqa: E402

name = sys.argv[1]
Bs = [int(x) for x in sys.argv[2].split(",")]
opt = sys.argv[3]
vals = [int(x) for x in sys.argv[4].split(",")]
REPS = int(os.environ.get("REPS", "4"))
SECS = float(os.environ.get("SECS", "1.5"))
nv.nvmlInit()
hnd = nv.nvmlDeviceGetHandleByIndex(0)
dev = torch.device("cuda", 0)
fs.set_option("pdl_w", 0)
for B in Bs:
    wl = bench.make_device_workload(name, B, dev)
    out = torch.empty(B, dtype=torch.int32, device=dev)
    fn = bench.fused_step_fn(fs, wl, [0], out)
    res = {v: [] for v in vals}
    for _ in range(REPS):
        for v in vals:
            fs.set_option(opt, v)
            for _ in range(20):
                fn()
            torch.cuda.synchronize()
            n = 0
            e0 = nv.nvmlDeviceGetTotalEnergyConsumption(hnd)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            t0 = time.time()
            while time.time() - t0 < SECS:
                for _ in range(50):
                    fn()
                n += 50
                torch.cuda.synchronize()
            ev1.record()
            torch.cuda.synchronize()
            e1 = nv.nvmlDeviceGetTotalEnergyConsumption(hnd)
            res[v].append((1e3 * ev0.elapsed_time(ev1) / n, (e1 - e0) / n))
    fs.set_option(opt, 0)
    for v in vals:
        us = sorted(r[0] for r in res[v])[len(res[v]) // 2]
        mj = sorted(r[1] for r in res[v])[len(res[v]) // 2]
        print(f"{name} B={B:4d} {opt}={v}: {us:8.2f} us/step  {mj:7.1f} mJ/step  runs {[(round(a, 1), round(b, 1)) for a, b in res[v]]}",
              flush=True)
    del wl
    torch.cuda.empty_cache()
