#!/usr/bin/env python
"""bench.py -- FlashSampling (fused LM-head + exact Gumbel-max sampling) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--config llama3_8b] [--B 32] [--impl reference]

Metric (BASELINE.json): "LM-head+sample us/step & HBM GB/s vs peak, B=1-256, V=128K-262K".
A step = one pass of the whole hot path (stage-1 fused kernel + stage-2 reduce; for N>1 also
the summary all-gather and combine) over one batch of synthetic decode hidden states.

N=1 : workload = BASELINE.json configs[1], Llama-3-8B LM head (D=4096, V=128256, bf16), B=32
      (the north-star "B<=32" target).  The JSON line also carries the B in {1,8,32,128,256}
      sweep with the unfused baselines measured on the same box.
N>1 : (torchrun, one rank per GPU, NCCL) the same workload vocabulary-sharded (Alg. A.4):
      every rank streams V/N rows and the ranks all-gather B x 12-byte summaries.
      scaling = "strong" (total work fixed).
--impl reference : the fp64 CPU oracle (oracle/), timed on the host cores on a bounded
      vocabulary sample of the same workload, scaled to a full step.

W (1.05 GB) is larger than L2 (126 MB), so successive steps stream it from HBM; no flush.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "LM-head+sample µs/step & HBM GB/s vs peak, B=1–256, V=128K–262K"
UNIT = "us/step"


# ----------------------------------------------------------------------------------------------
def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm_gbs=d["hbm_gbs"], bf16_tflops=d["bf16_tflops"],
                    bf16_tflops_sustained=d.get("bf16_tflops_sustained", d["bf16_tflops"]), source="measured")
    return dict(hbm_gbs=6650.0, bf16_tflops=1590.0, bf16_tflops_sustained=1400.0, source="fallback")


def algorithmic_bytes(B, D, V, transforms=False, n_groups=0, tp_world=1):
    """Bytes the method must move per step: W once, h, transforms,
    outputs; the [B,V] logits are never materialised.  Candidate scratch is excluded."""
    b = 2 * V * D + 2 * B * D + 4 * B
    if transforms:
        b += 4 * V + 4 * B + 4 * B * ((V + 31) // 32)
    if n_groups:
        b += 12 * B * n_groups
    if tp_world > 1:
        b += 12 * B * tp_world
    return b


def stage1_bytes(B, D, V, transforms=False):
    b = 2 * V * D + 2 * B * D
    if transforms:
        b += 4 * V + 4 * B + 4 * B * ((V + 31) // 32)
    return b


class ClockSampler:
    """SM clock / power / clock-event reasons sampled while running: NVML polled every 5 ms from a
    thread (enough samples inside a sub-second timed region); nvidia-smi every 100 ms as fallback."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device_index: int):
        self.samples = []
        self.proc = None
        try:
            uuid = str(torch.cuda.get_device_properties(device_index).uuid)
            ident = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
        except Exception:
            ident = str(device_index)
        self.cmd = ["nvidia-smi", f"--id={ident}", "--query-gpu=" + ",".join(self.FIELDS),
                    "--format=csv,noheader,nounits", "-lms", "100"]

    def _nvml_loop(self, nv, hnd):
        names = [(nv.nvmlClocksEventReasonHwSlowdown, "hw_slowdown"),
                 (nv.nvmlClocksEventReasonHwThermalSlowdown, "hw_thermal_slowdown"),
                 (nv.nvmlClocksEventReasonSwThermalSlowdown, "sw_thermal_slowdown"),
                 (nv.nvmlClocksEventReasonSwPowerCap, "sw_power_cap")]
        mx = nv.nvmlDeviceGetMaxClockInfo(hnd, nv.NVML_CLOCK_SM)
        while not self.stop:
            try:
                sm = nv.nvmlDeviceGetClockInfo(hnd, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(hnd) / 1000.0
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(hnd)
                flags = ["Active" if rs & bit else "Not Active" for bit, _ in names]
                self.samples.append((time.time(), [str(sm), str(mx), f"{pw:.1f}", *flags]))
            except Exception:
                break
            time.sleep(0.005)

    def __enter__(self):
        self.stop = False
        try:
            import pynvml as nv
            nv.nvmlInit()
            uuid = self.cmd[1].split("=", 1)[1]
            try:
                hnd = nv.nvmlDeviceGetHandleByUUID(uuid)
            except Exception:
                hnd = nv.nvmlDeviceGetHandleByIndex(0)
            self.thread = threading.Thread(target=self._nvml_loop, args=(nv, hnd), daemon=True)
            self.thread.start()
            self.source = "nvml"
            return self
        except Exception:
            pass
        self.source = "nvidia-smi"
        try:
            self.proc = subprocess.Popen(self.cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.samples.append((time.time(), parts))

    def __exit__(self, *a):
        self.stop = True
        if getattr(self, "source", "") == "nvml":
            self.thread.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(p[0]) for _, p in self.samples if p[0].replace(".", "").isdigit()]
        mx = [float(p[1]) for _, p in self.samples if p[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, p in self.samples for i in range(4) if p[3 + i].lower() == "active"})
        pw = [float(p[2]) for _, p in self.samples if p[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples), "power_w_median": statistics.median(pw) if pw else None,
                "source": getattr(self, "source", None)}


def time_loop(fn, steps, warmup, stream=None):
    """Average device ms per call over exactly `steps` calls, CUDA events on the launching stream."""
    stream = stream or torch.cuda.current_stream()
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def time_median(fn, iters, warmup):
    """Median of per-call event times (the paper's protocol: 25 warm-ups, median of 100)."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for a, b in evs:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in evs)


# ----------------------------------------------------------------------------------------------
def make_device_workload(name, B, device, seed=1234, V=None, vocab_rows=None):
    """Synthetic decode inputs of `name` drawn directly on the GPU (same recipe as synth)."""
    cfg = synth.CONFIGS[name]
    D, V = cfg["D"], V or cfg["V"]
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    h = torch.randn(B, D, device=device, generator=g).to(torch.bfloat16)
    rows = vocab_rows if vocab_rows is not None else (0, V)
    W = (torch.randn(rows[1] - rows[0], D, device=device, generator=g) * synth.W_STD).to(torch.bfloat16)
    bias = tau = mask = None
    if "temperature" in cfg:
        bias = torch.randn(rows[1] - rows[0], device=device, generator=g) * cfg["bias_std"]
        tau = torch.full((B,), cfg["temperature"], device=device)
        ban = torch.rand(B, V, device=device, generator=g) < cfg["mask_ban_frac"]
        mask = synth.pack_allowed_bits(~ban)
    return dict(h=h, W=W, bias=bias, temperature=tau, mask=mask, D=D, V=V, group_size=cfg.get("group_size"))


def fused_step_fn(fs, wl, step_ctr, out):
    def fn():
        step_ctr[0] += 1
        if wl["group_size"]:
            fs.sample_grouped(wl["h"], wl["W"], group_size=wl["group_size"], bias=wl["bias"],
                              temperature=wl["temperature"], mask=wl["mask"], seed=synth.SAMPLING_SEED,
                              step=step_ctr[0], return_groups=True)
        else:
            fs.sample(wl["h"], wl["W"], bias=wl["bias"], temperature=wl["temperature"], mask=wl["mask"],
                      seed=synth.SAMPLING_SEED, step=step_ctr[0], out=out)
    return fn


def baselines(wl, iters, warmup):
    """Unfused paths on the same inputs: cuBLAS GEMM alone; GEMM + softmax +
    torch.multinomial (eager); FlashInfer FI2 (Gumbel-max on logits) and FI1 (top-k/top-p).
    For the grouped workload the unfused path must also produce the log-normalizer and the
    per-group log-masses (torch.logsumexp over the materialised logits)."""
    h, W, bias, tau, mask = wl["h"], wl["W"], wl["bias"], wl["temperature"], wl["mask"]
    V = W.shape[0]
    g = wl["group_size"]
    res = {}

    def transformed():
        lg = torch.matmul(h, W.t()).float()
        if bias is not None:
            lg = lg + bias
        if tau is not None:
            lg = lg / tau[:, None]
        if mask is not None:
            allowed = synth.unpack_allowed_bits(mask, V)
            lg = lg.masked_fill(~allowed, float("-inf"))
        return lg

    def with_groups(sampler_fn):
        def fn():
            lg = transformed()
            out = sampler_fn(lg)
            if g:
                pad = (-V) % g
                lgp = torch.nn.functional.pad(lg, (0, pad), value=float("-inf"))
                torch.logsumexp(lgp.view(lg.shape[0], -1, g), dim=-1)
                torch.logsumexp(lg, dim=-1)
            return out
        return fn

    res["cublas_gemm_only_us"] = 1e3 * time_median(lambda: torch.matmul(h, W.t()), iters, warmup)
    res["gemm_softmax_multinomial_eager_us"] = 1e3 * time_median(
        with_groups(lambda lg: torch.multinomial(torch.softmax(lg, -1), 1)), iters, warmup)
    try:
        import flashinfer.sampling as fis
        res["fi2_gemm_sampling_from_logits_us"] = 1e3 * time_median(
            with_groups(lambda lg: fis.sampling_from_logits(lg)), iters, warmup)
        res["fi1_gemm_top_k_top_p_us"] = 1e3 * time_median(
            with_groups(lambda lg: fis.top_k_top_p_sampling_from_logits(lg, 50, 0.95)), iters, warmup)
    except Exception as e:  # pragma: no cover - FlashInfer missing or failing on this box
        res["flashinfer_error"] = repr(e)[:200]
    return res


# ----------------------------------------------------------------------------------------------
def cpu_oracle_step_us(name, B, seconds, with_tp_world=1):
    """Time the fp64 oracle (as it stands) on a bounded vocabulary slice of the workload and
    scale to a full step.  Returns (us_per_full_step, cores, sample description)."""
    import numpy as np
    from oracle import sampler
    try:
        from threadpoolctl import threadpool_info
        cores = max([d.get("num_threads", 1) for d in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    cfg = synth.CONFIGS[name]
    D, V = cfg["D"], cfg["V"]
    Vs = 4096
    wl = synth.make_workload(name, B, V=Vs, D=D)
    a = dict(h=synth.as_numpy_exact(wl.h), W=synth.as_numpy_exact(wl.W), bias=synth.as_numpy_exact(wl.bias),
             temperature=synth.as_numpy_exact(wl.temperature), mask=synth.as_numpy_exact(wl.mask))
    t0 = time.perf_counter()
    n = 0
    while True:
        sc = sampler.scores(a["h"], a["W"], seed=synth.SAMPLING_SEED, step=n, bias=a["bias"],
                            temperature=a["temperature"], mask=a["mask"])
        sampler.flat_sample(sc, want_near=False)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    per_slice = el / n
    return 1e6 * per_slice * (V / Vs), cores, (f"{n} oracle passes over a {Vs}-row vocabulary slice "
                                              f"(all {B} rows, D={D}); scaled x{V / Vs:.2f} to V={V}")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    name, B = args.config, args.B
    sec_per_step = max(0.05, min(1.0, 120.0 / max(1, args.steps + args.warmup)))
    # warm-up passes (untimed), then K timed passes, each a bounded sample of the workload
    cpu_oracle_step_us(name, B, min(2.0, sec_per_step * args.warmup))
    us, cores, sample = cpu_oracle_step_us(name, B, sec_per_step * args.steps)
    line = {"impl": "reference", "metric": METRIC, "value": round(us, 1), "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(us / 1e3, 3),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE.json shapes)",
            "config": {"workload": f"{name} LM head, B={B}", "B": B, "D": synth.CONFIGS[name]["D"],
                       "V": synth.CONFIGS[name]["V"]},
            "cpu_baseline": {"value": round(us, 1), "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": round(us, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------------
def load_traffic(name, B):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    try:
        return json.load(open(p)).get(f"{name}/B{B}")
    except Exception:
        return None


def roofline(name, B, D, V, t_stage1_ms, pk, transforms):
    byts = stage1_bytes(B, D, V, transforms)
    flops = 2.0 * B * V * D
    t_hbm = byts / (pk["hbm_gbs"] * 1e9)
    t_tc = flops / (pk["bf16_tflops"] * 1e12)
    t = t_stage1_ms * 1e-3
    traffic = load_traffic(name, B)
    # the library picks the CTA-pair kernel from MMA N >= 32 (B > 16), else the 1-CTA kernel
    kname = "fused_tc2_kernel (CTA pair, stage 1)" if B > 16 else "fused_tc_kernel (stage 1)"
    if t_tc > t_hbm:
        ach = flops / t / 1e12
        return {"bound": "tensor", "achieved": round(ach, 1), "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                "frac": round(ach / pk["bf16_tflops"], 4), "traffic": traffic,
                "kernel": kname, "kernel_us": round(t * 1e6, 2),
                "algorithmic_bytes": byts, "peak_source": pk["source"]}
    ach = byts / t / 1e9
    return {"bound": "hbm", "achieved": round(ach, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": round(ach / pk["hbm_gbs"], 4), "traffic": traffic, "kernel": kname,
            "kernel_us": round(t * 1e6, 2), "algorithmic_bytes": byts, "peak_source": pk["source"],
            "frac_of_nominal_8TBps": round(ach / 8000.0, 4)}


def run_single(args):
    import paper_2603_15854_b200 as fs
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    pk = peaks()
    name, B = args.config, args.B
    wl = make_device_workload(name, B, dev)
    D, V = wl["D"], wl["V"]
    transforms = wl["bias"] is not None
    n_groups = (V + wl["group_size"] - 1) // wl["group_size"] if wl["group_size"] else 0
    out = torch.empty(B, dtype=torch.int32, device=dev)
    ctr = [0]
    fn = fused_step_fn(fs, wl, ctr, out)
    fs.set_option("pdl_w", 1)            # serving configuration: W prefetched across steps (PDL)
    one_kernel = not wl["group_size"]   # plain / transformed sampling: stage 1 finalizes (fuse_reduce)
    for _ in range(max(3, args.warmup)):
        fn()
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        ms = time_loop(fn, args.steps, args.warmup)
    clocks = clk.summary()
    us = ms * 1e3
    # isolated stage-1 timing (CUDA events around each fused-kernel launch on its stream; PDL off)
    fs.set_option("time_stage1", 1)
    fs.query("stage1_ms")
    time_loop(fn, min(args.steps, 200), 2)
    launches = fs.query("stage1_launches")
    t1_ms = fs.query("stage1_ms") / max(1.0, launches)
    fs.set_option("time_stage1", 0)
    # one kernel per step: its average launch duration is the timed loop's events / K
    roof = roofline(name, B, D, V, ms if one_kernel else t1_ms, pk, transforms)
    roof["timing"] = ("CUDA events over the K timed steps (one fused kernel per step)" if one_kernel
                      else "CUDA events around each stage-1 launch (PDL off)")
    roof["kernel_us_isolated"] = round(t1_ms * 1e3, 2)
    # end to end through the public API with host buffers (H2D of h [+tau, mask], D2H of idx)
    h_host = wl["h"].cpu().pin_memory()
    t_host = wl["temperature"].cpu().pin_memory() if wl["temperature"] is not None else None
    m_host = wl["mask"].cpu().pin_memory() if wl["mask"] is not None else None
    h_dev = torch.empty_like(wl["h"])
    t_dev = torch.empty_like(wl["temperature"]) if t_host is not None else None
    m_dev = torch.empty_like(wl["mask"]) if m_host is not None else None
    idx_host = torch.empty(B, dtype=torch.int32, pin_memory=True)
    e_ctr = [0]

    def e2e_fn():
        e_ctr[0] += 1
        fs.sample_from_host(h_host, wl["W"], temperature_host=t_host, mask_host=m_host, bias=wl["bias"],
                            seed=synth.SAMPLING_SEED, step=e_ctr[0], h_dev=h_dev, t_dev=t_dev, m_dev=m_dev,
                            idx_dev=out, idx_host=idx_host)
    e2e_ms = time_loop(e2e_fn, args.steps, args.warmup)
    h2d = h_host.numel() * 2 + (t_host.numel() * 4 if t_host is not None else 0) + \
        (m_host.numel() * 4 if m_host is not None else 0)
    line = {"metric": METRIC, "value": round(us, 2), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded h~N(0,1), W~N(0,0.02^2), bf16; random-init LM head)",
            "config": {"workload": f"{name} LM head, B={B}" + (f", grouped g={wl['group_size']}" if n_groups else ""),
                       "B": B, "D": D, "V": V, "parallelism": "single GPU",
                       "launch": ("one fused kernel per step" if one_kernel else "stage 1 + stage-2 reduce")
                                 + ", PDL across steps (pdl_w=1)",
                       "l2": "no flush: W (%.2f GB) > L2 (126 MB) is re-streamed from HBM every step" % (2 * V * D / 1e9)},
            "hbm_gbs_achieved_step": round(algorithmic_bytes(B, D, V, transforms, n_groups) / (ms * 1e-3) / 1e9, 1),
            "roofline": roof,
            "clocks": clocks,
            "gpu_launches": (1 if one_kernel else 2) * args.steps * ((B + 255) // 256),
            "e2e": {"value": round(e2e_ms * 1e3, 2), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": B * 4,
                    "path": ("sample_from_host -> fs_sample_staged: the sampling kernel copies the pinned host h "
                             "into device memory itself (per-CTA slices + grid counter) and stores the ids into "
                             "pinned host memory -- one kernel per step" if m_host is None else
                             "sample_from_host: pinned inputs staged by fs_copy_async (PDL-chained copy kernel), "
                             "ids stored by the sampling kernel into pinned host memory")}}
    if not args.no_sweep:
        line["sweep"] = sweep(fs, name, pk, args)
        # the other BASELINE.json configs (same protocol): transforms, grouped, 70B LM head
        if name == "llama3_8b" and not args.no_configs:
            line["configs"] = {c: sweep(fs, c, pk, args, Bs=(1, 32, 256))
                               for c in ("qwen25_7b", "gemma3_27b", "llama3_70b")}
    if not args.no_cpu:
        cus, cores, sample = cpu_oracle_step_us(name, B, args.cpu_seconds)
        line["cpu_baseline"] = {"value": round(cus, 1), "unit": UNIT, "cores": cores, "kind": "oracle",
                                "sample": sample}
    print(json.dumps(line), flush=True)


def sweep(fs, name, pk, args, Bs=(1, 8, 32, 128, 256)):
    res = {}
    dev = torch.device("cuda", 0)
    for B in Bs:
        wl = make_device_workload(name, B, dev, seed=99 + B)
        D, V = wl["D"], wl["V"]
        transforms = wl["bias"] is not None
        out = torch.empty(B, dtype=torch.int32, device=dev)
        ctr = [0]
        fn = fused_step_fn(fs, wl, ctr, out)
        fs.set_option("pdl_w", 1)
        one_kernel = not wl["group_size"]
        us = 1e3 * time_median(fn, 100, 25)            # per-call events (the paper's protocol)
        loop_us = 1e3 * time_loop(fn, 100, 10)          # back-to-back steps (PDL overlap), as the headline
        fs.set_option("time_stage1", 1)
        fs.query("stage1_ms")
        time_loop(fn, 50, 2)
        t1 = fs.query("stage1_ms") / 50
        fs.set_option("time_stage1", 0)
        r = {"fused_us": round(us, 2), "fused_loop_us": round(loop_us, 2), "stage1_us": round(t1 * 1e3, 2),
             "one_kernel": one_kernel}
        r["roofline"] = roofline(name, B, D, V, us * 1e-3 if one_kernel else t1, pk, transforms)
        if name == "llama3_8b" and not wl["group_size"]:
            # SURVEY f3/f4 variants of the same step: per-request RNG streams, log-probabilities
            seeds = torch.arange(B, device=dev, dtype=torch.int64) * 7919 + 17
            vctr = [0]

            def per_request():
                vctr[0] += 1
                fs.sample(wl["h"], wl["W"], seeds=seeds, step=vctr[0], out=out)

            def with_logprob():
                vctr[0] += 1
                fs.sample(wl["h"], wl["W"], seed=synth.SAMPLING_SEED, step=vctr[0], return_logprob=True)
            def topk_fused():
                vctr[0] += 1
                fs.sample(wl["h"], wl["W"], seed=synth.SAMPLING_SEED, step=vctr[0], top_k=50, top_p=0.95, out=out)
            r["variants"] = {"per_request_seeds_us": round(1e3 * time_median(per_request, 100, 25), 2),
                             "with_logZ_logprob_us": round(1e3 * time_median(with_logprob, 100, 25), 2),
                             # SURVEY f1 through the LM head (vs baselines.fi1_gemm_top_k_top_p_us)
                             "top_k50_top_p095_fused_us": round(1e3 * time_median(topk_fused, 100, 25), 2)}
        if not args.no_baselines and not wl["group_size"]:
            # standalone sampling over the same materialised fp32 logits (§5.2):
            # fs_sample_logits vs FlashInfer's Gumbel-max sampling_from_logits (FI2's sampler)
            lg = torch.matmul(wl["h"], wl["W"].t()).float()
            sctr = [0]

            def ours_sl():
                sctr[0] += 1
                fs.sample_logits(lg, bias=wl["bias"], temperature=wl["temperature"], mask=wl["mask"],
                                 seed=synth.SAMPLING_SEED, step=sctr[0])
            def ours_topk():
                sctr[0] += 1
                fs.sample_logits(lg, bias=wl["bias"], temperature=wl["temperature"], mask=wl["mask"],
                                 seed=synth.SAMPLING_SEED, step=sctr[0], top_k=50, top_p=0.95)
            st = {"fs_sample_logits_us": round(1e3 * time_median(ours_sl, 100, 25), 2),
                  "fs_sample_logits_top_k50_top_p095_us": round(1e3 * time_median(ours_topk, 100, 25), 2),
                  "logits_bytes": lg.numel() * 4}
            st["fs_sample_logits_gbs"] = round(st["logits_bytes"] / (st["fs_sample_logits_us"] * 1e-6) / 1e9, 1)
            try:
                import flashinfer.sampling as fis
                if wl["bias"] is None:
                    st["flashinfer_sampling_from_logits_us"] = round(
                        1e3 * time_median(lambda: fis.sampling_from_logits(lg), 100, 25), 2)
                    st["flashinfer_top_k_top_p_k50_p095_us"] = round(
                        1e3 * time_median(lambda: fis.top_k_top_p_sampling_from_logits(lg, 50, 0.95), 100, 25), 2)
            except Exception as e:  # pragma: no cover
                st["flashinfer_error"] = repr(e)[:200]
            r["standalone_logits"] = st
            del lg
        if not args.no_baselines:
            bl = baselines(wl, 100, 25)
            r["baselines"] = {k: (round(v, 2) if isinstance(v, float) else v) for k, v in bl.items()}
            unfused = [v for k, v in bl.items() if k.endswith("_us") and k != "cublas_gemm_only_us"]
            if unfused:
                r["speedup_vs_best_unfused"] = round(min(unfused) / us, 3)
        res[f"B{B}"] = r
        del wl
        torch.cuda.empty_cache()
    return res


# ----------------------------------------------------------------------------------------------
def run_tp(args):
    import torch.distributed as dist
    import paper_2603_15854_b200 as fs
    from paper_2603_15854_b200 import tp
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    if os.environ.get("FS_TP_SAME_DEVICE"):       # test hook: all ranks on GPU 0 (gloo), for 1-GPU boxes
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    backend = os.environ.get("FS_TP_BACKEND", "nccl")
    dist.init_process_group(backend, **({"device_id": dev} if backend == "nccl" else {}))
    name, B = args.config, args.B
    cfg = synth.CONFIGS[name]
    D, V = cfg["D"], cfg["V"]
    a, b = tp.shard_bounds(V, world, rank)
    g = torch.Generator(device=dev)
    g.manual_seed(1234)                                   # identical h on every rank
    h = torch.randn(B, D, device=dev, generator=g).to(torch.bfloat16)
    g.manual_seed(5678 + rank)
    W = (torch.randn(b - a, D, device=dev, generator=g) * synth.W_STD).to(torch.bfloat16)
    local_s = fs.Summaries.empty(B, device=dev)
    gathered = torch.empty(world, B, 3, dtype=torch.int32, device=dev)
    ctr = [0]
    fs.set_option("pdl_w", 1)            # W of the next shard step streams before the dependency wait

    def step():
        ctr[0] += 1
        return tp.sample_tp(h, W, a, V, seed=synth.SAMPLING_SEED, step=ctr[0], workspace=(local_s, gathered))
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            idx = step()
        e1.record()
        torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    allidx = [torch.empty_like(idx) for _ in range(world)]
    dist.all_gather(allidx, idx)
    identical = all(torch.equal(allidx[0], x) for x in allidx)
    # e2e: per step H2D of h, D2H of idx, through the same public API
    h_host = h.cpu().pin_memory()
    h_dev = torch.empty_like(h)
    idx_host = torch.empty(B, dtype=torch.int32, pin_memory=True)

    def e2e():
        h_dev.copy_(h_host, non_blocking=True)
        ctr[0] += 1
        i = tp.sample_tp(h_dev, W, a, V, seed=synth.SAMPLING_SEED, step=ctr[0], workspace=(local_s, gathered))
        idx_host.copy_(i, non_blocking=True)
    for _ in range(args.warmup):
        e2e()
    torch.cuda.synchronize()
    dist.barrier()
    e0.record()
    for _ in range(args.steps):
        e2e()
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
    dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    # the same step with the library's peer-memory exchange instead of the NCCL
    # all-gather (reported beside the headline; the headline keeps the NCCL path)
    push = {}
    ok = torch.ones(1, device=dev)
    try:
        tp.PushExchange(B_max=B)
    except Exception as e:  # pragma: no cover
        ok.zero_()
        push["error"] = repr(e)[:200]
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if ok.item() == 1:
        def pstep():
            ctr[0] += 1
            return fs.sample_tp_push(h, W, a, V, seed=synth.SAMPLING_SEED, step=ctr[0])
        for _ in range(max(3, args.warmup)):
            pstep()
        torch.cuda.synchronize()
        dist.barrier()
        e0.record()
        for _ in range(args.steps):
            pidx = pstep()
        e1.record()
        torch.cuda.synchronize()
        p_ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
        dist.all_reduce(p_ms, op=dist.ReduceOp.MAX)
        ref = tp.sample_tp(h, W, a, V, seed=synth.SAMPLING_SEED, step=ctr[0], workspace=(local_s, gathered))
        same = torch.tensor([float(torch.equal(ref, pidx))], device=dev)
        dist.all_reduce(same, op=dist.ReduceOp.MIN)
        push = {"us_per_step": round(p_ms.item() * 1e3, 2), "idx_equal_nccl_path": bool(same.item() == 1),
                "timeouts": fs.query("comm_timeouts")}
    if rank == 0:
        pk = peaks()
        us = ms.item() * 1e3
        byts = algorithmic_bytes(B, D, V, tp_world=world)
        line = {"metric": METRIC, "value": round(us, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms.item(), 5), "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (seeded, random-init LM head shards)",
                "config": {"workload": f"{name} LM head, B={B}, vocab-sharded TP (Alg. A.4)", "B": B, "D": D,
                           "V": V, "parallelism": f"tp{world} (vocab)",
                           "l2": "no flush: per-rank shard %.2f GB" % (2 * (b - a) * D / 1e9)},
                "aggregate_hbm_gbs": round(byts / (ms.item() * 1e-3) / 1e9, 1),
                "per_rank_hbm_frac": round((2 * (b - a) * D / (ms.item() * 1e-3) / 1e9) / pk["hbm_gbs"], 4),
                "idx_identical_across_ranks": identical,
                "exchange_push": push,
                "clocks": clk.summary(), "gpu_launches": 3 * args.steps,
                "e2e": {"value": round(e2e_ms.item() * 1e3, 2), "unit": UNIT, "h2d_bytes_per_step": B * D * 2,
                        "d2h_bytes_per_step": B * 4}}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="llama3_8b", choices=list(synth.CONFIGS))
    ap.add_argument("--B", type=int, default=32)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-baselines", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        return run_tp(args)
    return run_single(args)


if __name__ == "__main__":
    main()
