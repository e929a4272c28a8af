"""A/B library options on the bench workload: step time (back-to-back loop, pdl_w=0), stage-1 time
and the SM clock / power sampled during each loop.  Every combination is measured `REPS` times in
interleaved order (A B A B ...) so that clock drift under the power cap hits all of them alike.

    python tools/sweep_opts.py llama3_8b 128,256 '{"dbg_no_epi": [0, 1]}'
    VDIV=8 python tools/sweep_opts.py llama3_70b 1,32 '{"whole_tiles": [0, 1]}'   # V/8 rows (a TP shard's compute)
    python tools/sweep_opts.py llama3_8b 256 '[{"h_lead": -1}, {"h_lead": 4, "kbps": 2, "h_stages": 3}]'   # explicit combos
"""
import itertools
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_15854_b200 as fs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama3_8b"
Bs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,32,128,256").split(",")]
opts = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {"kbps": [1, 2, 4]}
REPS = int(os.environ.get("REPS", "3"))
STEPS = int(os.environ.get("STEPS", "200"))
dev = torch.device("cuda", 0)
pk = bench.peaks()
fs.set_option("pdl_w", 0)
for B in Bs:
    vdiv = int(os.environ.get("VDIV", "1"))
    wl = bench.make_device_workload(name, B, dev, V=bench.synth.CONFIGS[name]["V"] // vdiv if vdiv > 1 else None)
    out = torch.empty(B, dtype=torch.int32, device=dev)
    if isinstance(opts, list):                      # explicit combinations: [{"opt": v, ...}, ...]
        keys = sorted({k for d in opts for k in d})
        combos = [tuple(d.get(k, 0) for k in keys) for d in opts]
    else:
        keys = list(opts)
        combos = list(itertools.product(*[opts[k] for k in keys]))
    fn0 = bench.fused_step_fn(fs, wl, [0], out)
    t_end = time.time() + 1.0
    while time.time() < t_end:                     # pre-heat: let clocks settle under load
        for _ in range(50):
            fn0()
        torch.cuda.synchronize()
    res = {c: [] for c in combos}
    for rep in range(REPS):
        for combo in combos:
            try:
                for k, v in zip(keys, combo):
                    fs.set_option(k, v)
                fn = bench.fused_step_fn(fs, wl, [0], out)
                with bench.ClockSampler(0) as clk:
                    us = 1e3 * bench.time_loop(fn, STEPS, 10)
                t1 = bench.stage1_time_ms(fs, fn, 50)
                c = clk.summary()
                res[combo].append((us, t1 * 1e3, c["sm_mhz"], c.get("power_w_median")))
            except Exception as e:
                print(f"B={B} {dict(zip(keys, combo))} ERROR {e}", flush=True)
    for combo in combos:
        for k, v in zip(keys, combo):
            fs.set_option(k, v)
        runs = res[combo]
        if not runs:
            continue
        us = sorted(r[0] for r in runs)[len(runs) // 2]
        t1 = sorted(r[1] for r in runs)[len(runs) // 2]
        r = bench.roofline(name, B, wl["D"], wl["V"], t1 * 1e-3, pk, wl["bias"] is not None)
        print(f"{name} B={B:4d} {dict(zip(keys, combo))} step {us:8.2f} us  stage1 {t1:8.2f} us  "
              f"frac {r['frac']:.3f} {r['bound']}  runs {[(round(a, 1), m, p) for a, _, m, p in runs]}", flush=True)
    for k in keys:
        fs.set_option(k, 0)
    del wl
    torch.cuda.empty_cache()
