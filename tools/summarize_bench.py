"""Print the bench.py JSON line (last line of a log) as tables: headline, sweeps, TP shards."""
import json
import sys

d = json.loads([ln for ln in open(sys.argv[1]).read().strip().splitlines() if ln.startswith("{")][-1])
r = d.get("roofline", {})
print(f"value {d['value']} {d['unit']} | per-call {d.get('per_call_median_us')} | pipelined {d.get('pipelined_us')} | "
      f"kernel {r.get('kernel_us')} frac {r.get('frac')} {r.get('bound')} floor-frac {r.get('frac_of_floor')} | "
      f"e2e {d.get('e2e', {}).get('value')}")
print("clocks", d.get("clocks"))
print("cpu", {k: v for k, v in d.get("cpu_baseline", {}).items() if k != "sample"})
sweeps = [("llama3_8b", d.get("sweep", {}))] + list(d.get("configs", {}).items())
for cname, sw in sweeps:
    print(cname)
    for k, v in sw.items():
        bl = v.get("baselines", {})
        ro = v["roofline"]
        print(f"  {k:5s} call {v['fused_us']:8.2f} loop {v.get('fused_loop_us', 0):8.2f} pipe {v.get('pipelined_us', 0):8.2f} "
              f"st1 {v['stage1_us']:8.2f} | {ro['bound']:6s} frac {ro['frac']:.3f} floor {ro['floor_us']:7.1f} "
              f"({ro['frac_of_floor']:.3f}) | gemm {bl.get('cublas_gemm_only_us', 0):7.1f} mult {bl.get('multinomial_eager_us', 0):7.1f}"
              f"/{bl.get('multinomial_compiled_us', 0):7.1f} fi2 {bl.get('fi2_gemm_sampling_from_logits_us', 0):7.1f} "
              f"fi1 {bl.get('fi1_gemm_top_k_top_p_us', 0):7.1f} | x{v.get('speedup_vs_best_unfused')} "
              f"gemm-x{v.get('speedup_vs_cublas_gemm_only')}")
        if "variants" in v:
            print("        variants", v["variants"])
        if "standalone_logits" in v:
            print("        standalone", {k2: v2 for k2, v2 in v["standalone_logits"].items() if k2.endswith("_us")})
        if "paper_table3" in v:
            print("        table3", v["paper_table3"])
        for k2 in ("multinomial_compiled_error", "flashinfer_error"):
            if k2 in bl:
                print("        ", k2, bl[k2])
for k, v in d.get("tp_shards", {}).items():
    ro = v["roofline"]
    print(f"  tp {k:9s} Vl {v['V_local']} shard {v['shard_us']:7.2f} idx-only {v.get('shard_idx_only_us', 0):7.2f} comb {v['combine_us']:5.2f} {ro['bound']} "
          f"frac {ro['frac']:.3f} floor-frac {ro['frac_of_floor']:.3f} | naive gemm {v['naive_tp_gemm_us']:7.2f}")
for k, v in d.get("tp_exchange_world1", {}).items():
    print("  ex", k, v)
