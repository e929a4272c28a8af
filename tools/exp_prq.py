"""Per-request RNG streams: fused step and logits sampler time vs the shared stream, Llama-3-8B head."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_2603_15854_b200 as fs
dev = torch.device("cuda", 0)
for B in (32, 128, 256):
    wl = bench.make_device_workload("llama3_8b", B, dev)
    seeds = torch.arange(B, device=dev, dtype=torch.int64) * 7919 + 17
    o = torch.empty(B, dtype=torch.int32, device=dev)
    c = [0]
    def shared():
        c[0] += 1; fs.sample(wl["h"], wl["W"], seed=1, step=c[0], out=o)
    def prq():
        c[0] += 1; fs.sample(wl["h"], wl["W"], seeds=seeds, step=c[0], out=o)
    lg = torch.matmul(wl["h"], wl["W"].t()).float()
    def lshared():
        c[0] += 1; fs.sample_logits(lg, seed=1, step=c[0])
    def lprq():
        c[0] += 1; fs.sample_logits(lg, seeds=seeds, step=c[0])
    r = [f"{n} {1e3 * bench.time_median(f, 50, 10):7.1f}" for n, f in (("shared", shared), ("prq", prq), ("logits", lshared), ("logits_prq", lprq))]
    print(f"B={B}: " + " | ".join(r), flush=True)
    del wl, lg
