"""Energy per step of the fused kernel and of its parts (debug options dbg_no_epi / dbg_no_mma), from
the NVML total-energy counter over ~2 s of back-to-back steps: where the joules of a power-capped
large-batch step go.

    python tools/energy_split.py llama3_8b 128,256
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml as nv  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_15854_b200 as fs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama3_8b"
Bs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "128,256").split(",")]
SECS = float(os.environ.get("SECS", "2.0"))
VARIANTS = [("full", {}), ("no_epilogue", {"dbg_no_epi": 1}), ("no_mma", {"dbg_no_mma": 1}),
            ("no_loads", {"dbg_no_mma": 2}), ("no_mma_no_epi", {"dbg_no_mma": 1, "dbg_no_epi": 1})]
nv.nvmlInit()
hnd = nv.nvmlDeviceGetHandleByIndex(0)
dev = torch.device("cuda", 0)
fs.set_option("pdl_w", 0)
for B in Bs:
    wl = bench.make_device_workload(name, B, dev)
    out = torch.empty(B, dtype=torch.int32, device=dev)
    fn = bench.fused_step_fn(fs, wl, [0], out)
    # idle power (2 s) for the static share
    torch.cuda.synchronize()
    e0 = nv.nvmlDeviceGetTotalEnergyConsumption(hnd)
    t0 = time.time()
    time.sleep(1.0)
    idle_w = (nv.nvmlDeviceGetTotalEnergyConsumption(hnd) - e0) / 1e3 / (time.time() - t0)
    for rep in range(2):
        for label, opts in VARIANTS:
            for k in ("dbg_no_epi", "dbg_no_mma"):
                fs.set_option(k, opts.get(k, 0))
            for _ in range(20):
                fn()
            torch.cuda.synchronize()
            n = 0
            with bench.ClockSampler(0) as clk:
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
            us = 1e3 * ev0.elapsed_time(ev1) / n
            j = (e1 - e0) / 1e3 / n
            c = clk.summary()
            print(f"{name} B={B:4d} rep {rep} {label:14s} {us:8.1f} us/step  {1e3 * j:8.1f} mJ/step  "
                  f"{j / (us * 1e-6):7.1f} W  (idle {idle_w:.0f} W)  sm {c['sm_mhz']} MHz", flush=True)
    for k in ("dbg_no_epi", "dbg_no_mma"):
        fs.set_option(k, 0)
    del wl
    torch.cuda.empty_cache()
