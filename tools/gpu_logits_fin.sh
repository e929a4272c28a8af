mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_onekernel.py tests/test_gpu_logits.py -q -x -p no:cacheprovider > gpurun_out/pytest_lf.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_lf.log
python - > gpurun_out/exp15.txt 2>&1 <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_2603_15854_b200 as fs
import flashinfer.sampling as fis
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(1)
V, D = 128256, 4096
W = (torch.randn(V, D, device=dev, generator=g) * 0.02).to(torch.bfloat16)
for B in (1, 32, 128, 256):
    h = torch.randn(B, D, device=dev, generator=g).to(torch.bfloat16)
    lg = torch.matmul(h, W.t()).float()
    ctr = [0]
    def ours():
        ctr[0] += 1
        fs.sample_logits(lg, seed=1, step=ctr[0])
    r = {}
    for fuse in (0, 1):
        fs.set_option("fuse_reduce", fuse)
        r[f"ours_fuse{fuse}"] = round(bench.time_median(ours, 100, 20) * 1e3, 2)
        r[f"ours_fuse{fuse}_loop"] = round(bench.time_loop(ours, 100, 20) * 1e3, 2)
    r["flashinfer"] = round(bench.time_median(lambda: fis.sampling_from_logits(lg), 100, 20) * 1e3, 2)
    print(B, r, flush=True)
PY
