#!/usr/bin/env python
"""bench.py -- FlashSampling (fused LM-head + exact Gumbel-max sampling) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--config llama3_8b] [--B 32] [--impl reference]

Metric (BASELINE.json): "LM-head+sample us/step & HBM GB/s vs peak, B=1-256, V=128K-262K".
A step = one pass of the whole hot path (the fused stage-1 kernel, whose last
CTA also runs stage 2 for plain sampling; for N>1 also the B x 12-byte summary all-gather and the
combine, a8) over one batch of synthetic decode hidden states.

N=1 : workload = BASELINE.json configs[1], Llama-3-8B LM head (D=4096, V=128256, bf16), B=32
      (the north-star "B<=32" target).  `value` = K back-to-back steps with NO cross-step overlap
      (pdl_w=0: every step's kernel starts after the previous one finished) -- the honest step
      latency.  The PDL-pipelined period (next step's W stream starting under the previous step's
      tail) is reported separately as `pipelined_us`, the paper's per-call median as
      `per_call_median_us`.  The JSON line also carries the B in {1,8,32,128,256} sweep of every
      BASELINE.json config (+ the paper's own D=4096, V=151936 workload) with the unfused
      baselines measured on the same box, the per-rank compute of the vocab-sharded 70B step at
      n=2/4/8, and the CPU oracle timed with 1 thread and with every host core.
N>1 : (torchrun, one rank per GPU, NCCL) the same workload vocabulary-sharded (Alg. A.4): every
      rank streams V/N rows and the library all-gathers B x 12-byte summaries (fs_sample_tp,
      its own NCCL communicator).  scaling = "strong" (total work fixed).
--impl reference : the fp64 CPU oracle (oracle/), timed on the host cores on a bounded
      vocabulary sample of the same workload, scaled to a full step; same config dict.

W (>= 1.05 GB) is larger than L2 (126 MB), so successive steps stream it from HBM; no flush
(the 70B n=8 shard, 263 MB, is also > 2x L2).
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
SWEEP_B = (1, 8, 32, 128, 256)
PAPER_B = (1, 8, 32, 64, 128, 256)
# PAPER.md Table 3, B200 column: FlashSampling speedup vs Multinomial (compiled) / FI1 / FI2
# at D=4096, V=151936 -- context for the "paper_d4096" sweep (another implementation, same GPU type).
PAPER_TABLE3_B200 = {1: (1.46, 1.51, 1.32), 2: (1.46, 1.56, 1.30), 4: (1.47, 1.61, 1.32), 8: (1.53, 1.61, 1.33),
                     16: (1.57, 1.65, 1.36), 32: (1.68, 1.68, 1.38), 64: (1.84, 1.67, 1.39),
                     128: (1.89, 1.55, 1.27), 256: (1.58, 1.32, 1.07)}


# ----------------------------------------------------------------------------------------------
def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm_gbs=d["hbm_gbs"], bf16_tflops=d["bf16_tflops"],
                    bf16_tflops_sustained=d.get("bf16_tflops_sustained", d["bf16_tflops"]), source="measured")
    return dict(hbm_gbs=6650.0, bf16_tflops=1590.0, bf16_tflops_sustained=1400.0, source="fallback")


def algorithmic_bytes(B, D, V, transforms=False, n_groups=0, tp_world=1):
    """Bytes the method must move per step: W once, h, transforms, outputs; the
    [B,V] logits are never materialised.  Candidate scratch is excluded."""
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


def config_dict(name, B, world=1):
    """The workload description both arms print (identical dicts for the same workload)."""
    cfg = synth.CONFIGS[name]
    D, V = cfg["D"], cfg["V"]
    desc = f"{name} LM head, B={B}"
    if cfg.get("group_size"):
        desc += f", grouped g={cfg['group_size']} ({(V + cfg['group_size'] - 1) // cfg['group_size']} groups)"
    if "temperature" in cfg:
        desc += f", tau={cfg['temperature']} + bias + {int(100 * cfg['mask_ban_frac'])}% mask"
    if world > 1:
        desc += ", vocab-sharded TP (Alg. A.4)"
    return {"workload": desc, "B": B, "D": D, "V": V,
            "parallelism": "single GPU" if world == 1 else f"tp{world} (vocab)",
            "l2": "no flush: W (%.2f GB%s) > L2 (126 MB), re-streamed from HBM every step"
                  % (2 * V * D / max(1, world) / 1e9, " per rank" if world > 1 else "")}


class ClockSampler:
    """SM clock / power / clock-event reasons sampled while running: NVML polled every 5 ms from a
    thread; nvidia-smi every 100 ms as fallback."""
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
        self.t_start = time.time()
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
        self.t_end = time.time()
        if getattr(self, "source", "") == "nvml":
            self.thread.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        win = round(1e3 * (getattr(self, "t_end", time.time()) - getattr(self, "t_start", time.time())), 1)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "window_ms": win}
        sm = [float(p[0]) for _, p in self.samples if p[0].replace(".", "").isdigit()]
        mx = [float(p[1]) for _, p in self.samples if p[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        counts = {names[i]: sum(1 for _, p in self.samples if p[3 + i].lower() == "active") for i in range(4)}
        pw = [float(p[2]) for _, p in self.samples if p[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(k for k, v in counts.items() if v), "reason_samples": {k: v for k, v in counts.items() if v},
                "samples": len(self.samples), "window_ms": win,
                "power_w_median": statistics.median(pw) if pw else None, "source": getattr(self, "source", None)}


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


def time_quantiles(fn, iters, warmup):
    """Per-call event times (the paper's protocol: 25 warm-ups, median of 100): (p10, p50, p90) ms."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for a, b in evs:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in evs)
    q = lambda f: t[min(len(t) - 1, int(round(f * (len(t) - 1))))]
    return q(0.1), statistics.median(t), q(0.9)


def time_median(fn, iters, warmup):
    return time_quantiles(fn, iters, warmup)[1]


def time_graph_steps(make_call, n=100, reps=3):
    """CUDA-graph replay of n consecutive steps (each captured launch has its own step number):
    device ms per step with the host launch overhead removed."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        make_call(0)()                      # this stream's library context allocates outside capture
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(n):
                make_call(i + 1)()
        g.replay()
        s.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            g.replay()
            b.record(s)
            s.synchronize()
            ts.append(a.elapsed_time(b) / n)
    torch.cuda.current_stream().wait_stream(s)
    return statistics.median(ts)


def time_graph(fn, n=50, reps=5):
    """Device time per call of a short, launch-bound call: n calls captured into one CUDA graph on
    a side stream and replayed (median of `reps` replays) -- per-call event timing of a ~3 us kernel
    would measure the host's launch overhead instead."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                fn()
        g.replay()
        s.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            g.replay()
            b.record(s)
            s.synchronize()
            ts.append(a.elapsed_time(b) / n)
    torch.cuda.current_stream().wait_stream(s)
    return statistics.median(ts)


def timed_region(fn, steps, warmup, device_index=0, clock_window_s=0.12, barrier=None, agree=None):
    """The contract's timed region: W warm-ups, then a pre-roll of the same step long enough that the
    clock sampler sees >= clock_window_s of this load, then sync (+ barrier), exactly K steps between
    CUDA events on the launching stream, sync (+ barrier).  Returns (ms per step, clocks summary)."""
    stream = torch.cuda.current_stream()
    for _ in range(max(3, warmup)):
        fn()
    torch.cuda.synchronize()
    est = time_loop(fn, 10, 0)
    n_pre = max(0, int(math.ceil(clock_window_s / max(1e-6, est * 1e-3))) - steps)
    if agree is not None:            # N > 1: every rank must run the same number of (collective) steps
        n_pre = agree(n_pre)
    with ClockSampler(device_index) as clk:
        for _ in range(n_pre):
            fn()
        torch.cuda.synchronize()
        if barrier:
            barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        if barrier:
            barrier()
        torch.cuda.synchronize()
    c = clk.summary()
    c["preroll_steps"] = n_pre
    return e0.elapsed_time(e1) / steps, c


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


_COMPILED = {}


def _multinomial_fn(transforms, groups_g, V):
    """GEMM -> fp32 -> (+bias)/tau -> masked_fill -> softmax -> torch.multinomial, plus the
    log-normaliser and per-group log-masses when the workload is the grouped one."""
    def f(h, W, bias, tau, allowed):
        lg = torch.matmul(h, W.t()).float()
        if transforms:
            lg = ((lg + bias) / tau[:, None]).masked_fill(~allowed, float("-inf"))
        out = torch.multinomial(torch.softmax(lg, -1), 1)
        if groups_g:
            pad = (-V) % groups_g
            lgp = torch.nn.functional.pad(lg, (0, pad), value=float("-inf"))
            return out, torch.logsumexp(lgp.view(lg.shape[0], -1, groups_g), dim=-1), torch.logsumexp(lg, dim=-1)
        return out
    return f


def baselines(name, wl, iters, warmup, compiled=True):
    """Unfused paths on the same inputs: cuBLAS GEMM alone; GEMM + softmax +
    torch.multinomial, eager and torch.compile'd (the paper's "Multinomial"); FlashInfer FI2
    (Gumbel-max on logits) and FI1 (top-k 50 / top-p 0.95, reading R17).  For the grouped workload the
    unfused path must also produce the log-normaliser and the per-group log-masses.  The vocabulary
    mask is handed to the baselines already unpacked to bool (their most favourable input form)."""
    h, W, bias, tau, mask = wl["h"], wl["W"], wl["bias"], wl["temperature"], wl["mask"]
    V = W.shape[0]
    g = wl["group_size"]
    transforms = bias is not None
    allowed = synth.unpack_allowed_bits(mask, V) if mask is not None else None
    res = {}

    def transformed():
        lg = torch.matmul(h, W.t()).float()
        if transforms:
            lg = ((lg + bias) / tau[:, None]).masked_fill(~allowed, float("-inf"))
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
    mfn = _multinomial_fn(transforms, g, V)
    res["multinomial_eager_us"] = 1e3 * time_median(lambda: mfn(h, W, bias, tau, allowed), iters, warmup)
    if compiled:
        try:
            key = (name, transforms, g)
            if key not in _COMPILED:
                _COMPILED[key] = torch.compile(mfn, dynamic=True)
            cf = _COMPILED[key]
            t0 = time.time()
            cf(h, W, bias, tau, allowed)
            torch.cuda.synchronize()
            res["multinomial_compiled_us"] = 1e3 * time_median(lambda: cf(h, W, bias, tau, allowed), iters, warmup)
            res["multinomial_compile_s"] = round(time.time() - t0, 1)
        except Exception as e:  # pragma: no cover - inductor unavailable on the box
            res["multinomial_compiled_error"] = repr(e)[:200]
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
def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def cpu_oracle_step_us(name, B, seconds, threads=None):
    """Time the fp64 oracle (as it stands) on a bounded vocabulary slice of the workload and scale
    to a full step.  threads=1 pins numpy's BLAS pool to one thread; None leaves every host core.
    Returns (us_per_full_step, threads used, sample description)."""
    from oracle import sampler
    try:
        from threadpoolctl import threadpool_limits
    except Exception:  # pragma: no cover
        threadpool_limits = None
    cfg = synth.CONFIGS[name]
    D, V = cfg["D"], cfg["V"]
    Vs = 4096
    wl = synth.make_workload(name, B, V=Vs, D=D)
    a = dict(h=synth.as_numpy_exact(wl.h), W=synth.as_numpy_exact(wl.W), bias=synth.as_numpy_exact(wl.bias),
             temperature=synth.as_numpy_exact(wl.temperature), mask=synth.as_numpy_exact(wl.mask))
    nthreads = 1 if threads == 1 else host_cores()
    ctxm = threadpool_limits(limits=nthreads) if threadpool_limits else None
    if ctxm:
        ctxm.__enter__()
    try:
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
    finally:
        if ctxm:
            ctxm.__exit__(None, None, None)
    per_slice = el / n
    return 1e6 * per_slice * (V / Vs), nthreads, (f"{n} oracle passes over a {Vs}-row vocabulary slice "
                                                  f"(all {B} rows, D={D}) in {el:.1f} s; scaled x{V / Vs:.2f} to V={V}")


def cpu_baseline(name, B, seconds):
    us_all, cores, sample = cpu_oracle_step_us(name, B, seconds)
    us_one, _, sample_one = cpu_oracle_step_us(name, B, seconds, threads=1)
    return {"value": round(us_all, 1), "unit": UNIT, "cores": cores, "nproc": host_cores(), "kind": "oracle",
            "sample": sample, "one_thread": {"value": round(us_one, 1), "unit": UNIT, "cores": 1, "sample": sample_one}}


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
            "data": "synthetic (seeded h~N(0,1), W~N(0,0.02^2), bf16; random-init LM head)",
            "config": config_dict(name, B, args.gpus),
            "cpu_baseline": {"value": round(us, 1), "unit": UNIT, "cores": cores, "nproc": host_cores(),
                             "kind": "oracle", "sample": sample},
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


def roofline(name, B, D, V, t_kernel_ms, pk, transforms, kname=None, traffic_key=None):
    """Roofline of the stage-1 kernel: algorithmic bytes and 2BVD flops over the
    kernel's measured launch time.  The bound is the larger of t_HBM (measured copy peak) and t_TC at
    the SUSTAINED bf16 rate (the kernel is timed inside a long loop, MEASURED_PEAKS.json)."""
    byts = stage1_bytes(B, D, V, transforms)
    flops = 2.0 * B * V * D
    t_hbm = byts / (pk["hbm_gbs"] * 1e9)
    t_tc = flops / (pk["bf16_tflops_sustained"] * 1e12)
    t = t_kernel_ms * 1e-3
    traffic = load_traffic(*(traffic_key or (name, B)))
    kname = kname or ("fused_tc2_kernel (CTA pair, stage 1)" if B > 16 else "fused_tc_kernel (stage 1)")
    common = {"traffic": traffic, "kernel": kname, "kernel_us": round(t * 1e6, 2), "algorithmic_bytes": byts,
              "flops": flops, "peak_source": pk["source"],
              "floor_us": round(1e6 * max(t_hbm, t_tc), 2), "frac_of_floor": round(max(t_hbm, t_tc) / t, 4),
              "t_hbm_us": round(1e6 * t_hbm, 2), "t_tc_sustained_us": round(1e6 * t_tc, 2)}
    if t_tc > t_hbm:
        ach = flops / t / 1e12
        return {"bound": "tensor", "achieved": round(ach, 1), "peak": pk["bf16_tflops_sustained"],
                "unit": "TFLOP/s", "frac": round(ach / pk["bf16_tflops_sustained"], 4),
                "peak_kind": "bf16_tflops_sustained", **common}
    ach = byts / t / 1e9
    return {"bound": "hbm", "achieved": round(ach, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": round(ach / pk["hbm_gbs"], 4), "peak_kind": "hbm_gbs (copy)",
            "frac_of_nominal_8TBps": round(ach / 8000.0, 4), **common}


def read_peak(fs, dev, nbytes=1 << 30, iters=20):
    """Read-only HBM peak: our bulk-TMA read ring (fs_read_probe) over a 1 GiB random
    buffer (8.5x L2), CUDA events around `iters` back-to-back launches after warm-up.  The copy peak
    of MEASURED_PEAKS.json stays the roofline denominator; this is the read-only ceiling beside it."""
    buf = torch.empty(nbytes, dtype=torch.uint8, device=dev).random_(0, 256)
    sink = torch.zeros(1, dtype=torch.int64, device=dev)
    ms = time_loop(lambda: fs.read_probe(buf, sink), iters, 3)
    del buf
    return {"gbs": round(nbytes / (ms * 1e-3) / 1e9, 1), "bytes": nbytes, "us_per_pass": round(ms * 1e3, 2),
            "kernel": "read_probe_kernel (fs_read_probe: two CTAs per SM, each a 6 x 16 KB cp.async.bulk ring)"}


def stage1_time_ms(fs, fn, n):
    """Live CUDA events around each stage-1 launch inside the library (option time_stage1, which
    also disables PDL for those launches); average launch duration."""
    fs.set_option("time_stage1", 1)
    fs.query("stage1_ms")
    time_loop(fn, n, 2)
    launches = fs.query("stage1_launches")
    t = fs.query("stage1_ms") / max(1.0, launches)
    fs.set_option("time_stage1", 0)
    return t


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
    one_kernel = not wl["group_size"]   # plain / transformed sampling: stage 1 finalizes (fuse_reduce)
    # headline: K back-to-back steps, no cross-step overlap (each kernel waits for the previous one)
    fs.set_option("pdl_w", 0)
    ms, clocks = timed_region(fn, args.steps, args.warmup)
    us = ms * 1e3
    t1_ms = stage1_time_ms(fs, fn, min(args.steps, 200))
    pc10, per_call, pc90 = (1e3 * x for x in time_quantiles(fn, 100, 25))

    def graph_call(i):
        def c():
            fs.sample(wl["h"], wl["W"], bias=wl["bias"], temperature=wl["temperature"], mask=wl["mask"],
                      seed=synth.SAMPLING_SEED, step=10**6 + i, out=out)
        return c
    graph_ms = time_graph_steps(graph_call) if one_kernel else None
    # PDL-pipelined period: step n+1's W stream starts under step n's tail (reported, not the value)
    fs.set_option("pdl_w", 1)
    pipe_ms = time_loop(fn, max(args.steps, 100), args.warmup)
    fs.set_option("pdl_w", 0)
    # one kernel per step: its average launch duration is the timed loop's events / K
    roof = roofline(name, B, D, V, ms if one_kernel else t1_ms, pk, transforms)
    roof["timing"] = ("CUDA events over the K timed steps (one fused kernel per step, no PDL overlap)" if one_kernel
                      else "CUDA events around each stage-1 launch")
    roof["kernel_us_isolated"] = round(t1_ms * 1e3, 2)
    rp = read_peak(fs, dev)
    if roof["bound"] == "hbm":
        roof["frac_of_read_peak"] = round(roof["achieved"] / rp["gbs"], 4)
    # end to end through the public API with host buffers: every step stages this step's h from pinned
    # host memory, samples, and the host reads the step's ids (stream sync per step, as a serving loop)
    h_host = wl["h"].cpu().pin_memory()
    t_host = wl["temperature"].cpu().pin_memory() if wl["temperature"] is not None else None
    m_host = wl["mask"].cpu().pin_memory() if wl["mask"] is not None else None
    h_dev = torch.empty_like(wl["h"])
    t_dev = torch.empty_like(wl["temperature"]) if t_host is not None else None
    m_dev = torch.empty_like(wl["mask"]) if m_host is not None else None
    idx_host = torch.empty(B, dtype=torch.int32, pin_memory=True)
    e_ctr = [0]
    stream = torch.cuda.current_stream()
    sink = [0]

    def e2e_generic():
        e_ctr[0] += 1
        fs.sample_from_host(h_host, wl["W"], temperature_host=t_host, mask_host=m_host, bias=wl["bias"],
                            seed=synth.SAMPLING_SEED, step=e_ctr[0], h_dev=h_dev, t_dev=t_dev, m_dev=m_dev,
                            idx_dev=out, idx_host=idx_host)
        stream.synchronize()
        sink[0] += int(idx_host[0])
    prepared = None
    if m_host is None and not wl["group_size"]:
        prepared = fs.HostStepSampler(h_host, wl["W"], bias=wl["bias"], temperature_host=t_host,
                                      seed=synth.SAMPLING_SEED, h_dev=h_dev, idx_host=idx_host)

    idx_np = idx_host.numpy()                  # host view of the pinned ids (no torch op per step)

    def e2e_prepared():
        e_ctr[0] += 1
        prepared(e_ctr[0])
        prepared.wait()
        sink[0] += int(idx_np[0])
    # the host syncs every step, so nothing overlaps across steps; pdl_w = 1 only lets this step's
    # W stream start while the kernel itself is still staging h from host memory (the prepared
    # sampler has a context of its own: the option is set on it too)
    fs.set_option("pdl_w", 1)
    if prepared is not None:
        prepared.set_option("pdl_w", 1)
    e2e_ms = time_loop(e2e_prepared if prepared else e2e_generic, args.steps, args.warmup)
    e2e_generic_ms = time_loop(e2e_generic, args.steps, args.warmup) if prepared else e2e_ms
    fs.set_option("pdl_w", 0)
    h2d = h_host.numel() * 2 + (t_host.numel() * 4 if t_host is not None else 0) + \
        (m_host.numel() * 4 if m_host is not None else 0)
    line = {"metric": METRIC, "value": round(us, 2), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded h~N(0,1), W~N(0,0.02^2), bf16; random-init LM head)",
            "config": config_dict(name, B),
            "launch": ("one fused kernel per step (stage 2 in the last CTA)" if one_kernel
                       else "stage 1 + PDL-chained stage-2 reduce") + "; no cross-step overlap (pdl_w=0)",
            "per_call_median_us": round(per_call, 2),
            "per_call_p10_p90_us": [round(pc10, 2), round(pc90, 2)],
            "graph_replay_us": round(graph_ms * 1e3, 2) if graph_ms else None,
            "pipelined_us": round(pipe_ms * 1e3, 2),
            "pipelined_note": "K back-to-back steps with pdl_w=1: the next step's W stream starts before the "
                              "previous step's kernel ends (PDL); a period, not a step latency",
            "hbm_gbs_achieved_step": round(algorithmic_bytes(B, D, V, transforms, n_groups) / (ms * 1e-3) / 1e9, 1),
            "roofline": roof,
            "read_peak": rp,
            "clocks": clocks,
            "gpu_launches": (1 if one_kernel else 2) * args.steps * ((B + 255) // 256),
            "e2e": {"value": round(e2e_ms * 1e3, 2), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": B * 4, "generic_call_us": round(e2e_generic_ms * 1e3, 2),
                    "path": ("HostStepSampler (prepared fs_sample_staged call on its own context): the sampling "
                             "kernel copies the pinned host h into device memory itself, stores the ids into pinned "
                             "host memory and then a pinned completion flag; the host spins on the flag and reads the "
                             "ids every step (generic_call_us: sample_from_host + stream sync)" if prepared else
                             "sample_from_host: pinned inputs staged by fs_copy_async (PDL-chained copy kernel), "
                             "ids stored by the sampling kernel into pinned host memory; host sync + read every step")}}
    if not args.no_sweep:
        line["sweep"] = sweep(fs, name, pk, args)
        if name == "llama3_8b" and not args.no_configs:
            # the other BASELINE.json configs (same protocol) + the paper's own B200 workload
            line["configs"] = {c: sweep(fs, c, pk, args) for c in ("qwen25_7b", "gemma3_27b", "llama3_70b")}
            line["configs"]["paper_d4096"] = sweep(fs, "paper_d4096", pk, args, Bs=PAPER_B)
            line["tp_shards"] = tp_shards(fs, pk)
            line["tp_exchange_world1"] = tp_exchange_world1(fs)
            line["tp_push_multiprocess_1gpu"] = tp_push_multiprocess()
    if not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(name, B, args.cpu_seconds)
    print(json.dumps(line), flush=True)


def sweep(fs, name, pk, args, Bs=SWEEP_B):
    res = {}
    dev = torch.device("cuda", 0)
    for B in Bs:
        wl = make_device_workload(name, B, dev, seed=99 + B)
        D, V = wl["D"], wl["V"]
        transforms = wl["bias"] is not None
        out = torch.empty(B, dtype=torch.int32, device=dev)
        ctr = [0]
        fn = fused_step_fn(fs, wl, ctr, out)
        one_kernel = not wl["group_size"]
        fs.set_option("pdl_w", 0)
        with ClockSampler(0) as clk_call:
            q10, us, q90 = (1e3 * x for x in time_quantiles(fn, 100, 25))   # per call (the paper's protocol)
        with ClockSampler(0) as clk_loop:
            loop_us = 1e3 * time_loop(fn, 100, 10)      # back-to-back steps, no overlap (as the headline)
        t1 = stage1_time_ms(fs, fn, 50)
        pipe_us = None                                  # pdl_w = 1 applies PDL only up to pdl_w_max_b = 128 rows
        if B <= 128:
            fs.set_option("pdl_w", 1)
            pipe_us = round(1e3 * time_loop(fn, 100, 10), 2)   # PDL-pipelined period
            fs.set_option("pdl_w", 0)
        r = {"fused_us": round(us, 2), "fused_p10_p90_us": [round(q10, 2), round(q90, 2)],
             "fused_loop_us": round(loop_us, 2), "pipelined_us": pipe_us,
             "stage1_us": round(t1 * 1e3, 2), "one_kernel": one_kernel,
             "clocks": {k: {"sm_mhz": c.get("sm_mhz"), "power_w": c.get("power_w_median"), "reasons": c.get("reasons")}
                        for k, c in (("call", clk_call.summary()), ("loop", clk_loop.summary()))}}
        r["roofline"] = roofline(name, B, D, V, us * 1e-3 if one_kernel else t1, pk, transforms)
        if name == "llama3_8b":
            # SURVEY f1/f3/f4 variants of the same step: per-request RNG streams, log-probabilities, top-k/p
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
                             "top_k50_top_p095_fused_us": round(1e3 * time_median(topk_fused, 100, 25), 2)}
        if not args.no_baselines and name == "llama3_8b":
            # standalone sampling over the same materialised fp32 logits (§5.2)
            lg = torch.matmul(wl["h"], wl["W"].t()).float()
            sctr = [0]

            def ours_sl():
                sctr[0] += 1
                fs.sample_logits(lg, seed=synth.SAMPLING_SEED, step=sctr[0])

            def ours_topk():
                sctr[0] += 1
                fs.sample_logits(lg, seed=synth.SAMPLING_SEED, step=sctr[0], top_k=50, top_p=0.95)
            st = {"fs_sample_logits_us": round(1e3 * time_median(ours_sl, 100, 25), 2),
                  "fs_sample_logits_top_k50_top_p095_us": round(1e3 * time_median(ours_topk, 100, 25), 2),
                  "logits_bytes": lg.numel() * 4}
            st["fs_sample_logits_gbs"] = round(st["logits_bytes"] / (st["fs_sample_logits_us"] * 1e-6) / 1e9, 1)
            try:
                import flashinfer.sampling as fis
                st["flashinfer_sampling_from_logits_us"] = round(
                    1e3 * time_median(lambda: fis.sampling_from_logits(lg), 100, 25), 2)
                st["flashinfer_top_k_top_p_k50_p095_us"] = round(
                    1e3 * time_median(lambda: fis.top_k_top_p_sampling_from_logits(lg, 50, 0.95), 100, 25), 2)
            except Exception as e:  # pragma: no cover
                st["flashinfer_error"] = repr(e)[:200]
            r["standalone_logits"] = st
            del lg
        if not args.no_baselines:
            bl = baselines(name, wl, 100, 25, compiled=not args.no_compile)
            r["baselines"] = {k: (round(v, 2) if isinstance(v, float) else v) for k, v in bl.items()}
            unfused = [v for k, v in bl.items() if k.endswith("_us") and k != "cublas_gemm_only_us"]
            if unfused:
                r["speedup_vs_best_unfused"] = round(min(unfused) / us, 3)
            r["speedup_vs_cublas_gemm_only"] = round(bl["cublas_gemm_only_us"] / us, 3)
            if name == "paper_d4096":
                mult = bl.get("multinomial_compiled_us", bl["multinomial_eager_us"])
                ours = {"vs_multinomial": round(mult / us, 3)}
                if "fi1_gemm_top_k_top_p_us" in bl:
                    ours["vs_fi1"] = round(bl["fi1_gemm_top_k_top_p_us"] / us, 3)
                    ours["vs_fi2"] = round(bl["fi2_gemm_sampling_from_logits_us"] / us, 3)
                r["paper_table3"] = {"ours": ours, "paper_triton_b200": dict(zip(
                    ("vs_multinomial", "vs_fi1", "vs_fi2"), PAPER_TABLE3_B200.get(B, (None,) * 3)))}
        res[f"B{B}"] = r
        del wl
        torch.cuda.empty_cache()
    return res


def tp_shards(fs, pk, name="llama3_70b", worlds=(2, 4, 8), Bs=(1, 32, 256)):
    """Compute half of the vocabulary-sharded step (Alg. A.4) at n = 2/4/8, measured on this one GPU:
    rank 0's shard kernel over V/n rows -- idx only (what fs_sample_tp runs without logZ; the roofline)
    and with log-mass (fs_sample_shard) -- and the outer selection over n records (fs_combine_summaries).  The exchange itself needs n GPUs (bench --gpus N).  Beside it, the naive
    TP baseline's compute half (per-rank cuBLAS GEMM [B, V/n]) and the bytes its logits all-gather
    would receive per rank."""
    dev = torch.device("cuda", 0)
    cfg = synth.CONFIGS[name]
    D, V = cfg["D"], cfg["V"]
    res = {}
    fs.set_option("pdl_w", 0)
    for n in worlds:
        lo, hi = 0, V // n
        for B in Bs:
            wl = make_device_workload(name, B, dev, seed=7 + n + B, V=V, vocab_rows=(lo, hi))
            summ = fs.Summaries.empty(B, device=dev)
            gathered = fs.Summaries.empty(n, B, device=dev)
            ctr = [0]

            def shard():
                ctr[0] += 1
                fs.sample_shard(wl["h"], wl["W"], lo, V, seed=synth.SAMPLING_SEED, step=ctr[0], out=summ)

            def shard_idx_only():
                # the kernel fs_sample_tp runs when no logZ is requested: plain epilogue, one-kernel
                # finalize (records written by the last CTA) -- the same work as fs_sample on the shard
                ctr[0] += 1
                fs.sample(wl["h"], wl["W"], seed=synth.SAMPLING_SEED, step=ctr[0], out=idx_buf)

            idx_buf = torch.empty(B, dtype=torch.int32, device=dev)
            shard()
            gathered.raw.copy_(summ.raw.unsqueeze(0).expand(n, B, 3))
            shard_us = 1e3 * time_median(shard, 100, 25)
            shard_idx_us = 1e3 * time_median(shard_idx_only, 100, 25)
            comb_us = 1e3 * time_graph(lambda: fs.combine_summaries(gathered))
            gemm_us = 1e3 * time_median(lambda: torch.matmul(wl["h"], wl["W"].t()), 100, 25)
            res[f"n{n}/B{B}"] = {
                "V_local": hi - lo, "shard_us": round(shard_us, 2), "shard_idx_only_us": round(shard_idx_us, 2),
                "combine_us": round(comb_us, 2),
                "roofline": roofline(name, B, D, hi - lo, shard_idx_us * 1e-3, pk, False,
                                     kname="idx-only shard kernel (fs_sample_tp without logZ: one kernel)",
                                     traffic_key=(f"{name}_n{n}", B)),
                "roofline_log_mass_shard": roofline(name, B, D, hi - lo, shard_us * 1e-3, pk, False,
                                                    kname="fs_sample_shard (log-mass epilogue + stage 2)"),
                "exchange_bytes_per_rank": 12 * B * n,
                "naive_tp_gemm_us": round(gemm_us, 2),
                "naive_tp_allgather_bytes_per_rank": 2 * B * (hi - lo) * (n - 1)}
            del wl
    torch.cuda.empty_cache()
    return res


def tp_push_multiprocess(world=2, steps=50, B=32):
    """SURVEY f2 across processes: tools/tp_push_procs.py runs `world` ranks of the idx-only push step
    on this one GPU (CUDA IPC windows); their kernels time-slice the GPU, so this checks the protocol
    end to end (agreement, timeouts) rather than measuring an NVLink latency."""
    try:
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "tp_push_procs.py"), str(world), str(steps),
                            str(B)], capture_output=True, text=True, timeout=300)
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        return json.loads(lines[-1]) if lines else {"error": (r.stderr or r.stdout)[-300:]}
    except Exception as e:  # pragma: no cover
        return {"error": repr(e)[:200]}


def tp_exchange_world1(fs, name="llama3_70b", n=8, Bs=(1, 32, 256)):
    """Exchange overhead of the two TP paths without a second GPU: a one-rank NCCL communicator
    (fs_comm_init world 1 -> fs_sample_tp: shard kernel + ncclAllGather of B x 12 B + combine) and a
    one-rank peer window (fs_sample_tp_push: shard kernel with the fused push + the PDL-chained
    wait/combine kernel), each against fs_sample_shard alone on the same n=8 shard.  Per-call medians.
    The transfer over NVLink itself is not in these numbers (a single GPU box)."""
    dev = torch.device("cuda", 0)
    cfg = synth.CONFIGS[name]
    D, V = cfg["D"], cfg["V"]
    lo, hi = 0, V // n
    res = {}
    fs.set_option("pdl_w", 0)
    try:
        fs.comm_init(fs.comm_unique_id(), 1, 0)
        nccl_ok = True
    except Exception as e:  # pragma: no cover - NCCL not loadable
        nccl_ok = False
        res["nccl_error"] = repr(e)[:200]
    try:
        fs.comm_window_open([fs.comm_window_create(1, 0, max(Bs))])
        push_ok = True
    except Exception as e:  # pragma: no cover
        push_ok = False
        res["push_error"] = repr(e)[:200]
    for B in Bs:
        wl = make_device_workload(name, B, dev, seed=11 + B, V=V, vocab_rows=(lo, hi))
        summ = fs.Summaries.empty(B, device=dev)
        out = torch.empty(B, dtype=torch.int32, device=dev)
        ctr = [0]

        def shard():
            ctr[0] += 1
            fs.sample_shard(wl["h"], wl["W"], lo, V, seed=synth.SAMPLING_SEED, step=ctr[0], out=summ)

        def nccl():
            ctr[0] += 1
            fs.sample_tp(wl["h"], wl["W"], lo, V, seed=synth.SAMPLING_SEED, step=ctr[0], out=out)

        def push():
            ctr[0] += 1
            fs.sample_tp_push(wl["h"], wl["W"], lo, V, seed=synth.SAMPLING_SEED, step=ctr[0])
        r = {"shard_only_us": round(1e3 * time_median(shard, 100, 25), 2)}
        if nccl_ok:
            r["nccl_world1_us"] = round(1e3 * time_median(nccl, 100, 25), 2)
            r["nccl_overhead_us"] = round(r["nccl_world1_us"] - r["shard_only_us"], 2)
        if push_ok:
            r["push_world1_us"] = round(1e3 * time_median(push, 100, 25), 2)
            r["push_overhead_us"] = round(r["push_world1_us"] - r["shard_only_us"], 2)
            r["push_timeouts"] = fs.query("comm_timeouts")
        res[f"n{n}shard/B{B}"] = r
        del wl
    if nccl_ok:
        fs.comm_destroy()
    if push_ok:
        fs.comm_window_destroy()
    torch.cuda.empty_cache()
    return res


# ----------------------------------------------------------------------------------------------
def _trace(msg):
    if os.environ.get("FS_BENCH_TRACE"):
        print(f"[rank {os.environ.get('RANK', '0')}] {time.strftime('%H:%M:%S')} {msg}", file=sys.stderr, flush=True)


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
    transport = "nccl" if backend == "nccl" else "torch"
    _trace("init")
    if transport == "nccl":
        tp.NcclComm()                                     # the library's own communicator (fs_comm_init)
    local_s = fs.Summaries.empty(B, device=dev)
    gathered = torch.empty(world, B, 3, dtype=torch.int32, device=dev)
    idx_buf = torch.empty(B, dtype=torch.int32, device=dev)
    ctr = [0]
    fs.set_option("pdl_w", 0)

    def step():
        ctr[0] += 1
        return tp.sample_tp(h, W, a, V, seed=synth.SAMPLING_SEED, step=ctr[0], workspace=(local_s, gathered),
                            transport=transport, out=idx_buf)

    def agree(n):
        t = torch.tensor([n], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return int(t.item())
    _trace("timed")
    ms_l, clocks = timed_region(step, args.steps, args.warmup, device_index=local, barrier=dist.barrier, agree=agree)
    ms = torch.tensor([ms_l], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    idx = step()
    allidx = [torch.empty_like(idx) for _ in range(world)]
    dist.all_gather(allidx, idx)
    identical = all(torch.equal(allidx[0], x) for x in allidx)
    # e2e: per step H2D of h, the sharded step, D2H of idx and a host read
    h_host = h.cpu().pin_memory()
    h_dev = torch.empty_like(h)
    idx_host = torch.empty(B, dtype=torch.int32, pin_memory=True)

    def e2e():
        h_dev.copy_(h_host, non_blocking=True)
        ctr[0] += 1
        i = tp.sample_tp(h_dev, W, a, V, seed=synth.SAMPLING_SEED, step=ctr[0], workspace=(local_s, gathered),
                         transport=transport, out=idx_buf)
        idx_host.copy_(i, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return int(idx_host[0])
    _trace("e2e")
    e2e_l, _ = timed_region(e2e, args.steps, args.warmup, device_index=local, barrier=dist.barrier,
                            clock_window_s=0.0, agree=agree)
    e2e_ms = torch.tensor([e2e_l], device=dev)
    dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    # naive TP baseline: per-rank logits [B, V/n] bf16 -> all-gather -> sampler on the full row
    _trace("naive")
    naive = {}
    try:
        lg_local = torch.empty(B, b - a, dtype=torch.bfloat16, device=dev)
        Vl = V // world
        lg_all = torch.empty(world * B, Vl, dtype=torch.bfloat16, device=dev)   # concatenated (any backend)

        def naive_step():
            torch.matmul(h, W[:Vl].t(), out=lg_local[:, :Vl])
            dist.all_gather_into_tensor(lg_all, lg_local[:, :Vl].contiguous())
            full = lg_all.view(world, B, Vl).permute(1, 0, 2).reshape(B, world * Vl).float()
            try:
                import flashinfer.sampling as fis
                return fis.sampling_from_logits(full)
            except Exception:
                return torch.multinomial(torch.softmax(full, -1), 1)
        n_ms, _ = timed_region(naive_step, args.steps, args.warmup, device_index=local, barrier=dist.barrier,
                               clock_window_s=0.0, agree=agree)
        n_t = torch.tensor([n_ms], device=dev)
        dist.all_reduce(n_t, op=dist.ReduceOp.MAX)
        naive = {"us_per_step": round(n_t.item() * 1e3, 2), "allgather_bytes_per_rank": 2 * B * Vl * (world - 1)}
    except Exception as e:  # pragma: no cover
        naive = {"error": repr(e)[:200]}
    # the same step with the library's peer-memory exchange instead of NCCL
    _trace("push")
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
        p_l, _ = timed_region(pstep, args.steps, args.warmup, device_index=local, barrier=dist.barrier,
                              clock_window_s=0.0, agree=agree)
        p_ms = torch.tensor([p_l], device=dev)
        dist.all_reduce(p_ms, op=dist.ReduceOp.MAX)
        pidx = pstep()
        ref = tp.sample_tp(h, W, a, V, seed=synth.SAMPLING_SEED, step=ctr[0], workspace=(local_s, gathered),
                           transport=transport)
        same = torch.tensor([float(torch.equal(ref, pidx))], device=dev)
        dist.all_reduce(same, op=dist.ReduceOp.MIN)
        push = {"us_per_step": round(p_ms.item() * 1e3, 2), "idx_equal_nccl_path": bool(same.item() == 1),
                "timeouts": fs.query("comm_timeouts")}
    _trace("report")
    if rank == 0:
        pk = peaks()
        us = ms.item() * 1e3
        byts = algorithmic_bytes(B, D, V, tp_world=world)
        line = {"metric": METRIC, "value": round(us, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms.item(), 5), "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (seeded h~N(0,1), W~N(0,0.02^2), bf16; random-init LM head)",
                "config": config_dict(name, B, world),
                "launch": f"fs_sample_tp ({transport}): shard kernel + all-gather of B x 12 B + combine; "
                          "no cross-step overlap (pdl_w=0)",
                "aggregate_hbm_gbs": round(byts / (ms.item() * 1e-3) / 1e9, 1),
                "per_rank_hbm_frac": round((2 * (b - a) * D / (ms.item() * 1e-3) / 1e9) / pk["hbm_gbs"], 4),
                "idx_identical_across_ranks": identical,
                "naive_tp_logits_allgather": naive,
                "exchange_push": push,
                "clocks": clocks, "gpu_launches": 3 * args.steps,
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
    ap.add_argument("--no-compile", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
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
