"""Where the end-to-end step's time goes beyond the device step (bench.py `e2e`): host cost of the
prepared call, launch-to-start latency, completion-to-host wake-up, in-kernel h staging over PCIe.

    python tools/e2e_breakdown.py [B]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
import paper_2603_15854_b200 as fs  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
dev = torch.device("cuda", 0)
wl = bench.make_device_workload("llama3_8b", B, dev)
h_host = wl["h"].cpu().pin_memory()
idx_host = torch.empty(B, dtype=torch.int32, pin_memory=True)
idx_np = idx_host.numpy()
out = torch.empty(B, dtype=torch.int32, device=dev)
stream = torch.cuda.current_stream()
N = 300


def host_us(fn, n=N):
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return 1e6 * (time.perf_counter() - t0) / n


res = {}
ctx = fs.context(0)
lib = fs._lib.lib()
import ctypes  # noqa: E402
d = ctypes.c_double()
res["ctypes_query_call_us"] = host_us(lambda: lib.fs_ctx_query(ctx, b"stage1_launches", ctypes.byref(d)))
s = fs.HostStepSampler(h_host, wl["W"], seed=synth.SAMPLING_SEED, idx_host=idx_host)
ctr = [0]


def prepared_call():
    ctr[0] += 1
    s(ctr[0])


for pdl in (0, 1):
    fs.set_option("pdl_w", pdl)
    for _ in range(20):
        prepared_call()
        s.wait()
    # host time to issue one step while the GPU is busy (queue far from full)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        prepared_call()
    res[f"pdl{pdl}_issue_us_per_call"] = 1e6 * (time.perf_counter() - t0) / 50
    torch.cuda.synchronize()
    # device-only back-to-back period of the staged kernel
    res[f"pdl{pdl}_device_loop_us"] = 1e3 * bench.time_loop(prepared_call, 200, 10)
    # serving cadence: call, wait, read -- host wall clock and device events
    t0 = time.perf_counter()
    for _ in range(N):
        prepared_call()
        s.wait()
        int(idx_np[0])
    res[f"pdl{pdl}_e2e_wall_us"] = 1e6 * (time.perf_counter() - t0) / N


# the same cadence with h already on the device (no staging): the PCIe part of the e2e gap
def dev_step():
    ctr[0] += 1
    fs.sample(wl["h"], wl["W"], seed=synth.SAMPLING_SEED, step=ctr[0], out=out)


fs.set_option("pdl_w", 0)
t0 = time.perf_counter()
for _ in range(N):
    dev_step()
    stream.synchronize()
res["device_h_call_sync_wall_us"] = 1e6 * (time.perf_counter() - t0) / N
res["device_h_loop_us"] = 1e3 * bench.time_loop(dev_step, 200, 10)
# round trip of an empty-ish kernel: launch + completion wake-up
x = torch.zeros(1, device=dev)
t0 = time.perf_counter()
for _ in range(N):
    x.add_(1)
    stream.synchronize()
res["tiny_kernel_sync_roundtrip_us"] = 1e6 * (time.perf_counter() - t0) / N
for k, v in res.items():
    print(f"{k:36s} {v:9.2f}")
