import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_2603_15854_b200 as fs
import flashinfer.sampling as fis
dev = torch.device("cuda", 0)
for B in (1, 32, 128, 256):
    lg = torch.randn(B, 128256, device=dev) * 1.3
    ctr = [0]
    def ours():
        ctr[0] += 1
        fs.sample_logits(lg, seed=1, step=ctr[0])
    def seeds_():
        ctr[0] += 1
        fs.sample_logits(lg, seeds=torch.arange(B, device=dev) * 3 + 1, step=ctr[0])
    t = bench.time_median(ours, 100, 25) * 1e3
    t2 = bench.time_median(lambda: fis.sampling_from_logits(lg), 100, 25) * 1e3
    t3 = bench.time_median(seeds_, 100, 25) * 1e3
    print(f"B={B:4d} fs_sample_logits {t:8.2f} us ({lg.numel()*4/(t*1e-6)/1e9:7.1f} GB/s)  per-request {t3:8.2f}  flashinfer {t2:8.2f} us")
for B in (1, 32, 128, 256):
    lg = torch.randn(B, 128256, device=dev) * 1.3
    ctr = [0]
    def ours():
        ctr[0] += 1
        fs.sample_logits(lg, seed=1, step=ctr[0], top_k=50, top_p=0.95)
    t = bench.time_median(ours, 100, 25) * 1e3
    t2 = bench.time_median(lambda: fis.top_k_top_p_sampling_from_logits(lg, 50, 0.95), 100, 25) * 1e3
    print(f"B={B:4d} top-k 50 / top-p 0.95: fs {t:8.2f} us   flashinfer {t2:8.2f} us")
