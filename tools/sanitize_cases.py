"""Small invocations of every kernel for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2603_15854_b200 as fs
dev = "cuda"
wl = synth.make_workload("qwen25_7b", 40, V=3000, D=136, with_transforms=True)
h, W, bias, tau, mask = (x.to(dev) for x in (wl.h, wl.W, wl.bias, wl.temperature, wl.mask))
for pair in (0, 1):
    fs.set_option("pair", pair)
    for fuse, pdl_w in ((0, 0), (1, 0), (1, 1)):       # stage-2 kernel / one-kernel finalize / + PDL prefetch
        fs.set_option("fuse_reduce", fuse)
        fs.set_option("pdl_w", pdl_w)
        for st in range(3):
            fs.sample(h, W, seed=1, step=st)
            fs.sample(h, W, bias=bias, temperature=tau, mask=mask, seed=1, step=2, return_score=True)
    fs.set_option("fuse_reduce", 1)
    fs.set_option("pdl_w", 0)
    fs.sample_grouped(h, W, group_size=512, bias=bias, temperature=tau, mask=mask, seed=1, step=2)
    fs.sample(h, W, seeds=torch.arange(40, device=dev), step=3, return_logprob=True)
    parts = [fs.sample_shard(h, W[a:b].contiguous(), a, 3000, seed=1, step=2).raw for a, b in ((0, 1500), (1500, 3000))]
    fs.combine_summaries(torch.stack(parts))
fs.set_option("pair", -1)
for wt in (0, 1):                                         # 16-row CTA ranges / whole tiles on the fewest CTAs
    fs.set_option("whole_tiles", wt)
    fs.sample(h, W, bias=bias, temperature=tau, mask=mask, seed=1, step=4, return_score=True)
    fs.sample(h[:8].contiguous(), W, seed=1, step=4)
# one-kernel paths added later: logZ finalize in the last CTA (B <= 16), grouped warp-per-group stage 2,
# in-kernel host staging, logits-sampler finalize, fused top-k span gather
h8, tau8, mask8 = h[:8].contiguous(), tau[:8].contiguous(), mask[:8].contiguous()
fs.sample(h8, W, bias=bias, temperature=tau8, mask=mask8, seed=1, step=2, return_logprob=True)
fs.sample_shard(h8, W[1000:2000].contiguous(), 1000, 3000, seed=1, step=2)
fs.sample_grouped(h, W, group_size=256, bias=bias, temperature=tau, mask=mask, seed=1, step=2)
for pdl_w in (0, 1):
    fs.set_option("pdl_w", pdl_w)
    out = torch.empty(40, dtype=torch.int32).pin_memory()
    for st in range(3):
        fs.sample_from_host(h.cpu().pin_memory(), W, temperature_host=tau.cpu().pin_memory(), bias=bias, seed=1,
                            step=st, h_dev=torch.empty_like(h), idx_host=out)
fs.set_option("pdl_w", 0)
fs.sample_logits(h.float() @ W.float().t(), bias=bias, temperature=tau, mask=mask, seed=1, step=3, return_score=True)
fs.set_option("topk_mode", 2)
fs.sample(h, W, temperature=tau, seed=1, step=2, top_k=30, top_p=0.9)
fs.set_option("topk_mode", 0)
fs.set_option("force_simt", 1)
fs.sample(h, W, bias=bias, temperature=tau, mask=mask, seed=1, step=2)
fs.set_option("force_simt", 0)
tiny = synth.make_workload("tiny", 4)
fs.sample(tiny.h.to(dev), tiny.W.to(dev), seed=1, step=0)
lg = (h.float() @ W.float().t())
fs.sample_logits(lg, bias=bias, temperature=tau, mask=mask, seed=1, step=1, return_all=True)
fs.sample_logits(lg, top_k=20, top_p=0.9, seed=1, step=1, return_all=True)
g = fs.sample_grouped(h, W, group_size=512, seed=1, step=0)[3]
fs.merge_summaries(fs.Summaries(g.raw[:, 0].contiguous()), fs.Summaries(g.raw[:, 1].contiguous()))
fs.gumbel_from_bits(torch.arange(1000, dtype=torch.int32, device=dev))
fs.random_bits(1, 2, torch.arange(100, device=dev), torch.arange(100, device=dev))
torch.cuda.synchronize()
print("sanitize cases ok")
# round 2: TP shard without log-mass (one-kernel records) and the one-kernel push exchange
fs.comm_init(fs.comm_unique_id(), 1, 0)
fs.sample_tp(h, W, 0, 3000, seed=1, step=5)
fs.sample_tp(h8, W, 0, 3000, seed=1, step=5)
fs.comm_destroy()
fs.comm_window_open([fs.comm_window_create(1, 0, 64)])
for st in range(3):
    fs.sample_tp_push(h, W, 0, 3000, seed=1, step=st)                   # one kernel: push + wait + combine
    fs.sample_tp_push(h8, W, 0, 3000, seed=1, step=st, return_all=True)  # log-mass shard + wait kernel
fs.comm_window_destroy()
torch.cuda.synchronize()
print("sanitize cases done")
