import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d.get("roofline", {})
print("value", d["value"], d["unit"], "| stage1", r.get("kernel_us"), "us frac", r.get("frac"), r.get("bound"),
      "| e2e", d.get("e2e", {}).get("value"), "| clocks", d.get("clocks"))
def rows(sw):
    for k, v in sw.items():
        yield k, v
sweeps = [("llama3_8b", d.get("sweep", {}))] + list(d.get("configs", {}).items())
for cname, sw in sweeps:
  print(cname)
  for k, v in rows(sw):
    bl = v.get("baselines", {})
    print(f"    {k:5s} fused {v['fused_us']:8.2f} loop {v.get('fused_loop_us', float('nan')):8.2f} stage1 {v['stage1_us']:8.2f} frac {v['roofline']['frac']:.3f} "
          f"{v['roofline']['bound']:6s} gemm {bl.get('cublas_gemm_only_us', 0):8.2f} fi2 {bl.get('fi2_gemm_sampling_from_logits_us', 0):8.2f} "
          f"mult {bl.get('gemm_softmax_multinomial_eager_us', 0):8.2f} speedup {v.get('speedup_vs_best_unfused')}")
