"""Regenerate DESIGN.md §8's results block (between the 'r02 results' marker and '## 9.') and the §1
headline numbers from profiles/r02/bench.json (the bench line of the final evidence run)."""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = json.load(open(os.path.join(ROOT, "profiles", "r02", "bench.json")))
log = "/tmp/_bench_line.log"
open(log, "w").write(json.dumps(d) + "\n")
tables = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "bench_table.py"), log], capture_output=True,
                        text=True).stdout
vv = {B: d["sweep"][f"B{B}"].get("variants", {}) for B in (1, 32, 128, 256)}
sl = {B: d["sweep"][f"B{B}"].get("standalone_logits", {}) for B in (1, 32, 128, 256)}
row = lambda k: " / ".join(f"{vv[B].get(k, 0):.0f}" for B in (1, 32, 128, 256))
srow = lambda k: " / ".join(f"{sl[B].get(k, 0):.1f}" for B in (1, 32, 128, 256))
c = d["clocks"]
ro = d["roofline"]
pk_copy = ro["peak"]
b32 = d["sweep"]["B32"]["baselines"]
fi2 = b32["fi2_gemm_sampling_from_logits_us"]
def _ratios():
    ug, uu = [], []
    for sw in [d["sweep"]] + list(d["configs"].values()):
        for v in sw.values():
            bl = v.get("baselines", {})
            if not bl:
                continue
            ug.append(bl["cublas_gemm_only_us"] / v["fused_us"])
            best = min(x for k, x in bl.items() if k.endswith("_us") and k != "cublas_gemm_only_us"
                       and isinstance(x, (int, float)))
            uu.append(best / v["fused_us"])
    return min(ug), max(ug), min(uu), max(uu)


g_lo, g_hi, u_lo, u_hi = _ratios()
block = f"""r02 results (`profiles/r02/bench.json`, the final evidence run of round 2 on one B200; `sw_power_cap`
active in {c.get('reason_samples', {}).get('sw_power_cap', 0)} of {c['samples']} clock samples of the headline window; µs per step). "per call" = median
of 100 individually event-timed calls after 25 warm-ups (the paper's protocol); "loop" = 100
back-to-back steps without cross-step overlap (the headline's protocol); "pipelined" = back-to-back
with `pdl_w` = 1 (PDL applies up to B = 128, `pdl_w_max_b`); frac = achieved / peak of the binding roofline (HBM copy peak, or sustained bf16
tensor peak), in brackets against max(t_HBM, t_TC); "×" = best unfused baseline (or cuBLAS GEMM
alone) ÷ our per-call time. Box-to-box spread under the power cap is several % (B ≥ 128 rows
especially: the loop column runs at the sustained power limit).

{tables}
Headline (Llama-3-8B, B = 32): **{d['value']:.1f} µs/step** back to back ({ro['frac']:.2f} of the {ro['peak']} GB/s copy peak,
{ro['frac_of_nominal_8TBps']:.2f} of nominal 8 TB/s), per call {d['per_call_median_us']:.1f} µs (p10–p90 {d['per_call_p10_p90_us'][0]:.1f}–{d['per_call_p10_p90_us'][1]:.1f}), CUDA-graph replay
{d['graph_replay_us']:.1f} µs, PDL-pipelined {d['pipelined_us']:.1f} µs; end to end from pinned host h with a host read of the ids
every step **{d['e2e']['value']:.1f} µs** (`sample_from_host` + stream sync: {d['e2e']['generic_call_us']:.1f} µs).

Variants at Llama-3-8B (per call, B = 1 / 32 / 128 / 256): per-request seeds {row('per_request_seeds_us')};
with logZ + log-prob {row('with_logZ_logprob_us')}; fused top-k 50 + top-p 0.95 {row('top_k50_top_p095_fused_us')}.
Standalone over materialised fp32 logits: Gumbel-max {srow('fs_sample_logits_us')} (FlashInfer
`sampling_from_logits` {srow('flashinfer_sampling_from_logits_us')}); top-k 50 + top-p 0.95
{srow('fs_sample_logits_top_k50_top_p095_us')} (FlashInfer {srow('flashinfer_top_k_top_p_k50_p095_us')}).

On the paper's own workload (D = 4096, V = 151,936) our speedups over the three unfused baselines
exceed the paper's Triton kernel's B200 ratios at every B (table above; same GPU type, different
boxes and software versions — context, not a like-for-like comparison).

Against cuBLAS GEMM alone (no sampling at all) the fused step is at parity ({g_lo:.2f}) or faster
(up to {g_hi:.2f}×) per call; the closest rows are B = 1–8, where both are at the copy peak, and grouped
Gemma (65 group summaries per row + the stage-2 group reduce). Sustained back to back at B = 128 the
power cap reverses that by 5–11% (§11 entry 32). The north star's bar, beating GEMM + sampler,
holds on every row (× best unfused {u_lo:.2f}–{u_hi:.2f}).

ncu (`profiles/r02/ncu_full_summary.json` / `.txt`, `--set full`, one call per config and B): DRAM
bytes per stage-1 launch 1.001–1.006 × the algorithmic bytes on every full-vocabulary config, 1.006–1.019 × on the
70B shards (W once; no logits
written: DRAM writes 3–12 MB); L2→SM 1.12 × W at B ≤ 32, 2.0 × W at B = 256 (h re-read per tile);
tensor pipe 5–10% active at B ≤ 32, 60–77% at B = 256 (1.34–1.51 GHz under the cap). Launch list of
the headline bench command: the fused kernel is 96% of the process's GPU time, one launch per step
(`profiles/r02/launches_b32_summary.json`).

The paper's B200 numbers are ratios only (Table 3, D=4096, V=151,936): 1.32–1.39× vs FI2 at
B ≤ 64, 1.07× at B=256 (BASELINE.md).

"""
p = os.path.join(ROOT, "DESIGN.md")
s = open(p).read()
i = s.index("r02 results (`profiles/r02/bench.json`")
j = s.index("## 9. Multi-GPU")
s = s[:i] + block + s[j:]
# §1 headline numbers
s = re.sub(r"Llama-3-8B LM head, B=32, \*\*[0-9.]+ µs per step\*\*",
           f"Llama-3-8B LM head, B=32, **{d['value']:.1f} µs per step**", s)
s = re.sub(r"now reported separately as `pipelined_us`, [0-9.]+\n",
           f"now reported separately as `pipelined_us`, {d['pipelined_us']:.1f}\n", s)
s = re.sub(r"= [0-9.]+ TB/s of algorithmic bytes = \*\*[0-9.]+ × the measured copy peak\*\*",
           f"= {ro['achieved'] / 1000:.2f} TB/s of algorithmic bytes = **{ro['frac']:.2f} × the measured copy peak**", s)
s = re.sub(r"per call [0-9.]+ µs; end to end from pinned host h with the host reading the\nids every step \*\*[0-9.]+ µs\*\*",
           f"per call {d['per_call_median_us']:.1f} µs; end to end from pinned host h with the host reading the\nids every step **{d['e2e']['value']:.1f} µs**", s)
s = re.sub(r"cuBLAS GEMM alone [0-9.]+ µs; best unfused sampler \(cuBLAS \+ FlashInfer\nGumbel-max, \"FI2\"\) [0-9.]+ µs → [0-9.]+× per call",
           f"cuBLAS GEMM alone {b32['cublas_gemm_only_us']:.1f} µs; best unfused sampler (cuBLAS + FlashInfer\nGumbel-max, \"FI2\") {fi2:.1f} µs → {fi2 / d['sweep']['B32']['fused_us']:.2f}× per call", s)
rp = d.get("read_peak", {}).get("gbs")
if rp:
    s = re.sub(r"\(6[0-9.]+ GB/s;\n0\.[0-9]+ of nominal 8 TB/s(; [0-9.]+ of the read-only peak, [0-9.]+ TB/s, §11 entry 34)?\)",
               f"({pk_copy:.1f} GB/s;\n{ro['achieved'] / 8000:.2f} of nominal 8 TB/s; {ro['achieved'] / rp:.2f} of the read-only peak, "
               f"{rp / 1000:.2f} TB/s, §11 entry 34)", s)
tc = [v["B256"]["roofline"]["frac"] for v in [d["sweep"]] + list(d["configs"].values()) if "B256" in v]
s = re.sub(r"sampler \([0-9.]+–[0-9.]+×, §8 table\)", f"sampler ({u_lo:.2f}–{u_hi:.2f}×, §8 table)", s)
s = re.sub(r"and sit at [0-9.]+–[0-9.]+ of the sustained-TC floor",
           f"and sit at {min(tc):.2f}–{max(tc):.2f} of the sustained-TC floor", s)
open(p, "w").write(s)
print("DESIGN.md results regenerated")
