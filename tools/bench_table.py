"""Markdown tables (DESIGN.md §8 results) from a bench.py JSON line: per config and B the fused step
(per call / loop / pipelined), the roofline fraction, and the unfused baselines."""
import json
import sys

_txt = open(sys.argv[1]).read().strip()
try:
    d = json.loads(_txt)                      # a pretty-printed bench.json
except json.JSONDecodeError:                  # a bench log: the last JSON line
    d = json.loads([ln for ln in _txt.splitlines() if ln.startswith("{")][-1])
print("| config | B | per call | loop | pipelined | bound, frac (of floor) | cuBLAS GEMM only | Multinomial eager / compiled | FI2 | FI1 | × best unfused | × GEMM only |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
sweeps = [("llama3_8b", d.get("sweep", {}))] + list(d.get("configs", {}).items())
for cname, sw in sweeps:
    for k, v in sw.items():
        bl = v.get("baselines", {})
        ro = v["roofline"]
        print(f"| {cname} | {k[1:]} | {v['fused_us']:.1f} | {v['fused_loop_us']:.1f} | {('%.1f' % v['pipelined_us']) if v.get('pipelined_us') is not None else '— (no PDL at B > 128)'} | "
              f"{ro['bound']} {ro['frac']:.3f} ({ro['frac_of_floor']:.3f}) | {bl.get('cublas_gemm_only_us', 0):.1f} | "
              f"{bl.get('multinomial_eager_us', 0):.1f} / {bl.get('multinomial_compiled_us', 0):.1f} | "
              f"{bl.get('fi2_gemm_sampling_from_logits_us', 0):.1f} | {bl.get('fi1_gemm_top_k_top_p_us', 0):.1f} | "
              f"{v.get('speedup_vs_best_unfused')} | {v.get('speedup_vs_cublas_gemm_only')} |")
print()
print("| paper workload B | ours vs Multinomial (compiled) / FI1 / FI2 | paper's Triton kernel on B200 (Table 3) |")
print("|---|---|---|")
for k, v in d.get("configs", {}).get("paper_d4096", {}).items():
    t = v.get("paper_table3", {})
    o, p = t.get("ours", {}), t.get("paper_triton_b200", {})
    print(f"| {k[1:]} | {o.get('vs_multinomial')} / {o.get('vs_fi1')} / {o.get('vs_fi2')} | "
          f"{p.get('vs_multinomial')} / {p.get('vs_fi1')} / {p.get('vs_fi2')} |")
print()
print("| 70B shard n / B | V_local | idx-only shard µs | frac (of floor) | log-mass shard µs | combine µs | naive per-rank GEMM µs | naive all-gather bytes/rank | summary bytes/rank |")
print("|---|---|---|---|---|---|---|---|---|")
for k, v in d.get("tp_shards", {}).items():
    ro = v["roofline"]
    print(f"| {k} | {v['V_local']} | {v.get('shard_idx_only_us', 0):.1f} | {ro['bound']} {ro['frac']:.3f} ({ro['frac_of_floor']:.3f}) | "
          f"{v['shard_us']:.1f} | {v['combine_us']:.2f} | {v['naive_tp_gemm_us']:.1f} | {v['naive_tp_allgather_bytes_per_rank']:,} | "
          f"{v['exchange_bytes_per_rank']} |")
