"""Summarise ncu exports under gpurun_out/ into profiles/<round>/ (launch shares, key metrics, traffic)."""
import collections, csv, json, sys
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
rows = list(csv.reader(open("gpurun_out/launches_b32.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    agg.setdefault(d["Kernel Name"].split("(")[0][:70], []).append(float(d["Metric Value"].replace(",", "")))
out = {k: {"launches": len(v), "mean_ns": sum(v) / len(v)} for k, v in agg.items()}
st1 = [v for k, v in out.items() if "fused_tc" in k]
st2 = [v for k, v in out.items() if "reduce" in k]
summary = {"command": "ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 20 "
                      "--warmup 5 --no-sweep --no-cpu (llama3_8b, B=32)",
           "note": "cold-cache, serialised per-launch times: compare shares, not absolutes", "kernels": out}
if st1 and st2:
    summary["stage1_share_of_step"] = st1[0]["mean_ns"] / (st1[0]["mean_ns"] + st2[0]["mean_ns"])
elif st1:
    summary["stage1_share_of_step"] = 1.0
    summary["note_one_kernel"] = "plain sampling is one fused kernel per step (fuse_reduce): no stage-2 launch"
json.dump(summary, open(f"profiles/{rnd}/launches_b32_summary.json", "w"), indent=1)
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__cycles_elapsed.avg",
        "launch__grid_size", "launch__block_size", "launch__cluster_dim_x"]
allm, traffic = {}, {}
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
for B in (1, 32, 256):
    r = list(csv.reader(open(f"gpurun_out/prof_b{B}.raw.csv")))
    d, u = dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))
    allm[f"B{B}"] = {k: (d.get(k), u.get(k)) for k in keys if k in d}
    tb = lambda k: float(d[k].replace(",", "")) * scale.get(u[k], 1)
    traffic[f"llama3_8b/B{B}"] = int(tb("dram__bytes_read.sum") + tb("dram__bytes_write.sum"))
json.dump(allm, open(f"profiles/{rnd}/ncu_full_fused_tc_key_metrics.json", "w"), indent=1)
json.dump(traffic, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps({k: round(v["mean_ns"] / 1e3, 2) for k, v in out.items()}), summary.get("stage1_share_of_step"))
print(traffic)
for B, m in allm.items():
    print(B, {k.split(".")[0][-30:]: v[0] for k, v in m.items()})
