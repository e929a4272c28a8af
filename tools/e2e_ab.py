"""Interleaved A/B of a library option on the end-to-end serving step (HostStepSampler: the sampling
kernel stages the pinned host h itself, the host spins on the completion word and reads the ids
every step), wall time per step.

    python tools/e2e_ab.py llama3_8b 1,32,128 staged_prefetch 0,16
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_15854_b200 as fs  # noqa: E402

name = sys.argv[1]
Bs = [int(x) for x in sys.argv[2].split(",")]
opt = sys.argv[3]
vals = [int(x) for x in sys.argv[4].split(",")]
REPS, STEPS = int(os.environ.get("REPS", "4")), int(os.environ.get("STEPS", "400"))
dev = torch.device("cuda", 0)
for B in Bs:
    wl = bench.make_device_workload(name, B, dev)
    h_host = wl["h"].cpu().pin_memory()
    t_host = wl["temperature"].cpu().pin_memory() if wl["temperature"] is not None else None
    samplers = {}
    for v in vals:
        s = fs.HostStepSampler(h_host, wl["W"], bias=wl["bias"], temperature_host=t_host, seed=1)
        s.set_option("pdl_w", 1)
        s.set_option(opt, v)
        samplers[v] = s
    res = {v: [] for v in vals}
    for _ in range(REPS):
        for v, s in samplers.items():
            for i in range(20):
                s(i)
                s.wait()
            t0 = time.perf_counter()
            for i in range(STEPS):
                s(i)
                s.wait()
            res[v].append((time.perf_counter() - t0) / STEPS * 1e6)
    for v in vals:
        r = sorted(res[v])
        print(f"{name} B={B} {opt}={v}: e2e {r[len(r) // 2]:.1f} us/step  runs {[round(x, 1) for x in res[v]]}", flush=True)
    del samplers, wl
    torch.cuda.empty_cache()
