"""Energy per step of the fused sampler next to cuBLAS doing the LM-head GEMM alone (no sampling) and
the best unfused sampler (cuBLAS GEMM -> fp32 logits -> FlashInfer Gumbel-max, "FI2"), from the NVML
total-energy counter over ~1.5 s of back-to-back steps each: at large B the B200 runs at its power
cap, where time per step ~ energy per step / cap -- a step that needs fewer joules than the GEMM
alone is as close to that bound as the GEMM is.

    python tools/energy_vs_gemm.py llama3_8b,qwen25_7b 128,256
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml as nv  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
import paper_2603_15854_b200 as fs  # noqa: E402

names = (sys.argv[1] if len(sys.argv) > 1 else "llama3_8b").split(",")
Bs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "128,256").split(",")]
SECS = float(os.environ.get("SECS", "1.5"))
REPS = int(os.environ.get("REPS", "2"))
nv.nvmlInit()
hnd = nv.nvmlDeviceGetHandleByIndex(0)
dev = torch.device("cuda", 0)
fs.set_option("pdl_w", 0)
try:
    import flashinfer.sampling as fis
except Exception:                      # noqa: BLE001
    fis = None


def measure(fn):
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
    c = clk.summary()
    return 1e3 * ev0.elapsed_time(ev1) / n, (e1 - e0) / n, c.get("sm_mhz"), c.get("power_w_median")


for name in names:
    for B in Bs:
        wl = bench.make_device_workload(name, B, dev)
        out = torch.empty(B, dtype=torch.int32, device=dev)
        ours = bench.fused_step_fn(fs, wl, [0], out)
        logits = torch.empty(B, wl["V"], dtype=torch.bfloat16, device=dev)

        def gemm():
            torch.matmul(wl["h"], wl["W"].t(), out=logits)

        arms = [("fused (ours)", ours), ("cuBLAS GEMM only", gemm)]
        if fis is not None:
            def fi2():
                lg = torch.matmul(wl["h"], wl["W"].t()).float()
                fis.sampling_from_logits(lg)
            arms.append(("cuBLAS + FlashInfer (FI2)", fi2))
        res = {a: [] for a, _ in arms}
        for _ in range(REPS):
            for label, fn in arms:
                res[label].append(measure(fn))
        for label, _ in arms:
            r = sorted(res[label])[len(res[label]) // 2]
            print(f"{name} B={B:4d} {label:26s} {r[0]:8.2f} us/step  {r[1]:7.1f} mJ/step  sm {r[2]} MHz  "
                  f"{r[3]} W  (runs {[(round(x[0], 1), round(x[1], 1)) for x in res[label]]})", flush=True)
        del wl, logits
        torch.cuda.empty_cache()
