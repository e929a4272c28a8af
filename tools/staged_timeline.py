"""Per-CTA timeline of back-to-back fs_sample_staged steps (h read from pinned host memory by the
sampling kernel) next to the device-h step (debug option dbg_times): when the staged h is
released to the producers, when the loads end, when the last CTA finishes -- where the end-to-end
overhead of in-kernel staging goes.

    python tools/staged_timeline.py [B=32] [config=llama3_8b]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_15854_b200 as fs  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
name = sys.argv[2] if len(sys.argv) > 2 else "llama3_8b"
dev = torch.device("cuda", 0)
fs.set_option("pdl_w", 0)
wl = bench.make_device_workload(name, B, dev)
W, h = wl["W"], wl["h"]
h_host = h.cpu().pin_memory()
h_dev = torch.empty_like(h)
idx_host = torch.empty(B, dtype=torch.int32, pin_memory=True)
out = torch.empty(B, dtype=torch.int32, device=dev)
ctr = [0]


def staged():
    ctr[0] += 1
    fs.sample_from_host(h_host, W, seed=1, step=ctr[0], h_dev=h_dev, idx_host=idx_host)


def device():
    ctr[0] += 1
    fs.sample(h, W, seed=1, step=ctr[0], out=out)


for tag, fn in (("device", device), ("staged", staged), ("device", device), ("staged", staged)):
    for _ in range(30):
        fn()
    torch.cuda.synchronize()
    us = 1e3 * bench.time_loop(fn, 300, 10)
    n = 16
    bufs = [torch.zeros(148 * 8, dtype=torch.int64, device=dev) for _ in range(n)]
    for s in range(n):
        fs.set_option("dbg_times", bufs[s].data_ptr())
        fn()
    fs.set_option("dbg_times", 0)
    torch.cuda.synchronize()
    A = np.stack([b.cpu().numpy().reshape(148, 8) for b in bufs]).astype(np.float64)
    G = int((A[0, :, 0] > 0).sum())
    A = A[:, :G]
    rel = lambda k: (A[:, :, k] - A[:, :, 0].min(axis=1, keepdims=True)) / 1e3   # us after first CTA start
    st, wt, ld, dr, end = rel(0), rel(1), rel(2), rel(3), rel(5)
    med = lambda x: float(np.median(x))
    print(f"{name} B={B} {tag:7s} loop {us:7.2f} us/step  grid {G}  (medians over {n} steps, us after the first CTA start)")
    print(f"   start spread {med(st.max(1)):6.2f}  wait-done min/med/max {med(wt.min(1)):6.2f} {med(np.median(wt, 1)):6.2f} "
          f"{med(wt.max(1)):6.2f}  loads-done max {med(ld.max(1)):7.2f}  drained max {med(dr.max(1)):7.2f}  "
          f"last CTA end {med(end.max(1)):7.2f}", flush=True)
    steps = A[:, :, 0].min(axis=1)
    ends = A[:, :, 5].max(axis=1)
    print(f"   launch gap (previous step's last CTA end -> this step's first CTA start): "
          f"{med((steps[1:] - ends[:-1]) / 1e3):6.2f} us", flush=True)

