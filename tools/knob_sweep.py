"""Sweep load-path knobs; prints stage-1 time and W GB/s."""
import sys, os, time, itertools, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_15854_b200 as fs
dev = torch.device("cuda", 0)
V, D = 128256, 4096
grid = json.loads(sys.argv[1])
Bs = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 32]
g = torch.Generator(device=dev); g.manual_seed(1)
W = (torch.randn(V, D, device=dev, generator=g) * 0.02).to(torch.bfloat16)
for B in Bs:
    h = torch.randn(B, D, device=dev, generator=g).to(torch.bfloat16)
    out = torch.empty(B, dtype=torch.int32, device=dev)
    ctr = [0]
    def fn():
        ctr[0] += 1
        fs.sample(h, W, seed=1, step=ctr[0], out=out)
    keys = list(grid)
    for combo in itertools.product(*[grid[k] for k in keys]):
        cfg = dict(zip(keys, combo))
        try:
            for k, v in cfg.items():
                fs.set_option(k, v)
            with bench.ClockSampler(0) as cs:
                t_end = time.time() + float(os.environ.get("KNOB_SECS", "1.0"))
                while time.time() < t_end:
                    for _ in range(20):
                        fn()
                    torch.cuda.synchronize()
            smp = cs.samples[len(cs.samples) * 2 // 5:]
            mhz = sorted(float(x[1][0]) for x in smp if x[1][0].replace(".", "").isdigit())
            pw = sorted(float(x[1][2]) for x in smp if x[1][2].replace(".", "").isdigit())
            clk = f"sm {mhz[len(mhz)//2] if mhz else -1:.0f} MHz {pw[len(pw)//2] if pw else -1:.0f} W"
            step = bench.time_loop(fn, 100, 5) * 1e3
            fs.set_option("time_stage1", 1); fs.query("stage1_ms")
            bench.time_loop(fn, 100, 5)
            t = fs.query("stage1_ms") / 100
            fs.set_option("time_stage1", 0)
            print(f"B={B:3d} {cfg} step {step:8.2f} us stage1 {t*1e3:8.2f} us {2*V*D/(t*1e-3)/1e9:8.1f} GB/s {clk}", flush=True)
        except Exception as e:
            fs.set_option("time_stage1", 0)
            print(f"B={B} {cfg} error {e}", flush=True)
    for k in keys:
        fs.set_option(k, {"l2promo": 3, "w_policy": 1}.get(k, 0))
