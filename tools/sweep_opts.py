"""Time the fused step under library tuning options (kbps, stages, ...) on the bench workload."""
import itertools, json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_15854_b200 as fs

name = sys.argv[1] if len(sys.argv) > 1 else "llama3_8b"
Bs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,32,128,256").split(",")]
opts = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {"kbps": [1, 2, 4]}
dev = torch.device("cuda", 0)
pk = bench.peaks()
for B in Bs:
    wl = bench.make_device_workload(name, B, dev)
    out = torch.empty(B, dtype=torch.int32, device=dev)
    keys = list(opts)
    import time
    fn0 = bench.fused_step_fn(fs, wl, [0], out)
    t_end = time.time() + 1.0
    while time.time() < t_end:                     # pre-heat: let clocks settle under load
        for _ in range(50):
            fn0()
        torch.cuda.synchronize()
    for combo in itertools.product(*[opts[k] for k in keys]):
        try:
            for k, v in zip(keys, combo):
                fs.set_option(k, v)
            fn = bench.fused_step_fn(fs, wl, [0], out)
            us = 1e3 * bench.time_loop(fn, 200, 20)
            fs.set_option("time_stage1", 1); fs.query("stage1_ms")
            bench.time_loop(fn, 50, 2)
            t1 = fs.query("stage1_ms") / 50
            fs.set_option("time_stage1", 0)
            r = bench.roofline(name, B, wl["D"], wl["V"], t1, pk, wl["bias"] is not None)
            print(f"B={B:4d} {dict(zip(keys, combo))} step {us:8.2f} us  stage1 {t1*1e3:8.2f} us  frac {r['frac']:.3f} {r['bound']}", flush=True)
        except Exception as e:
            print(f"B={B} {dict(zip(keys, combo))} ERROR {e}", flush=True)
    for k in keys:
        fs.set_option(k, 0)
    del wl
    torch.cuda.empty_cache()
