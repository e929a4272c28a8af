"""One profiled call per (config, B) for ncu: run under
    ncu --profile-from-start off --set full --clock-control none --import-source on -o gpurun_out/X \
        python tools/ncu_capture.py llama3_8b:1,32,256 qwen25_7b:1,32,256 gemma3_27b:1,32,256 llama3_70b:1,32,256 \
        llama3_70b_n8:32
Each spec is config[:B,B,...]; `<config>_n<k>` profiles rank 0's shard of a k-way vocabulary split
(fs_sample_shard).  Every call is warmed up 3 times, then exactly one call is bracketed by
cudaProfilerStart/Stop (bench.py's headline launch configuration: pdl_w = 0, fuse_reduce = 1).
The order of the profiled calls is printed (one line per call) so the ncu report can be mapped."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
import paper_2603_15854_b200 as fs  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    fs.set_option("pdl_w", 0)
    for spec in sys.argv[1:]:
        name, _, bs = spec.partition(":")
        Bs = [int(x) for x in bs.split(",")] if bs else [1, 32, 256]
        n = 1
        if "_n" in name:
            name, n = name.rsplit("_n", 1)
            n = int(n)
        V = synth.CONFIGS[name]["V"]
        for B in Bs:
            if n == 1:
                wl = bench.make_device_workload(name, B, dev)
                out = torch.empty(B, dtype=torch.int32, device=dev)
                fn = bench.fused_step_fn(fs, wl, [0], out)
            else:
                wl = bench.make_device_workload(name, B, dev, V=V, vocab_rows=(0, V // n))
                summ = fs.Summaries.empty(B, device=dev)

                def fn(wl=wl, summ=summ):
                    fs.sample_shard(wl["h"], wl["W"], 0, V, seed=synth.SAMPLING_SEED, step=1, out=summ)
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            torch.cuda.profiler.start()
            fn()
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()
            print(f"profiled {name}{'_n%d' % n if n > 1 else ''} B={B}", flush=True)
            del wl
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
