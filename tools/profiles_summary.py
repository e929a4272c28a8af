"""Summarise an ncu capture of tools/ncu_capture.py (full_raw.csv + full_capture.log) and the launch
list of the bench command (launches_b32.csv) into profiles/<round>/ and profiles/ncu_traffic.json.

    python tools/profiles_summary.py gpurun_out/r02c/prof r02
"""
import collections
import csv
import json
import os
import re
import sys

src, rnd = sys.argv[1], sys.argv[2]
out_dir = os.path.join("profiles", rnd)
os.makedirs(out_dir, exist_ok=True)

KEYS = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "l1tex__m_xbar2l1tex_read_bytes.sum": "l2_to_sm_bytes",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_lsu_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "smsp__inst_executed.sum": "inst",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3,
         "hz": 1e-9, "Khz": 1e-6, "Mhz": 1e-3, "Ghz": 1.0}

rows = list(csv.reader(open(os.path.join(src, "full_raw.csv"))))
hdr, units = rows[0], rows[1]
labels = [ln.split("profiled ", 1)[1].strip() for ln in open(os.path.join(src, "full_capture.log"))
          if ln.startswith("profiled ")]
kernels = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    rec = {"kernel": d["Kernel Name"].split("(")[0]}
    for k, short in KEYS.items():
        if k not in hdr:
            continue
        v = d[k].replace(",", "")
        try:
            x = float(v)
        except ValueError:
            continue
        u = units[hdr.index(k)]
        rec[short] = x * SCALE.get(u, 1.0)
    rec["time_us"] = rec.pop("time", None)
    if "sm_clock" in rec:
        rec["sm_clock_ghz"] = round(rec.pop("sm_clock"), 3)
    kernels.append(rec)

# map kernels to the profiled calls: each call's launches start with its stage-1 kernel ("fused_")
groups, cur = [], None
for k in kernels:
    if k["kernel"].split("<")[0].split()[-1].startswith("fused_") or cur is None:
        cur = []
        groups.append(cur)
    cur.append(k)
assert len(groups) == len(labels), (len(groups), len(labels))
summary, traffic = collections.OrderedDict(), {}
tp = os.path.join("profiles", "ncu_traffic.json")
if os.path.exists(tp):
    traffic = json.load(open(tp))
for lab, ks in zip(labels, groups):
    m = re.match(r"(\S+) B=(\d+)", lab)
    name, B = m.group(1), int(m.group(2))
    s1 = ks[0]
    entry = {"stage1": s1, "others": ks[1:],
             "stage1_dram_bytes": s1.get("dram_read", 0) + s1.get("dram_write", 0)}
    summary[f"{name}/B{B}"] = entry
    traffic[f"{name}/B{B}"] = int(entry["stage1_dram_bytes"])
json.dump({"source": "ncu --profile-from-start off --set full --clock-control none --import-source on "
                     "python tools/ncu_capture.py ... (one call per (config, B), pdl_w=0, fuse_reduce=1)",
           "note": "ncu replays each kernel ~40x with serialised launches: absolute times are cold and "
                   "unpipelined; byte counts and utilisations are per launch",
           "captures": summary}, open(os.path.join(out_dir, "ncu_full_summary.json"), "w"), indent=1)
json.dump(dict(sorted(traffic.items())), open(tp, "w"), indent=1)
print(f"{'capture':22s} {'kernel':28s} {'us':>7s} {'DRAM GB':>8s} {'L2->SM GB':>9s} {'dram%':>6s} {'tens%':>6s} "
      f"{'issue%':>6s} {'GHz':>5s} {'regs':>4s}")
for lab, e in summary.items():
    for k in [e["stage1"]] + e["others"]:
        print(f"{lab:22s} {k['kernel'][-28:]:28s} {k.get('time_us', 0):7.1f} {(k.get('dram_read', 0)) / 1e9:8.4f} "
              f"{k.get('l2_to_sm_bytes', 0) / 1e9:9.4f} {k.get('dram_pct', 0):6.1f} {k.get('tensor_pipe_pct', 0):6.1f} "
              f"{k.get('issue_active_pct', 0):6.1f} {k.get('sm_clock_ghz', 0):5.2f} {k.get('regs', 0):4.0f}")

# launch list of the headline bench command (cold, serialised: compare shares)
lp = os.path.join(src, "launches_b32.csv")
if os.path.exists(lp):
    lr = list(csv.reader(open(lp)))
    hi = [i for i, r in enumerate(lr) if "Kernel Name" in r][0]
    h2 = lr[hi]
    agg = collections.OrderedDict()
    for r in lr[hi + 1:]:
        d = dict(zip(h2, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = SCALE.get(d.get("Metric Unit", "nsecond"), 1e-3)
        agg.setdefault(d["Kernel Name"].split("(")[0][:70], []).append(float(d["Metric Value"].replace(",", "")) * scale)
    ks = {k: {"launches": len(v), "mean_us": round(sum(v) / len(v), 2)} for k, v in agg.items()}
    tot = sum(v["launches"] * v["mean_us"] for v in ks.values())
    for v in ks.values():
        v["share_of_gpu_time"] = round(v["launches"] * v["mean_us"] / tot, 4)
    json.dump({"command": "ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py "
                          "--steps 20 --warmup 5 --no-sweep --no-cpu (llama3_8b, B=32)",
               "note": "cold-cache, serialised per-launch times: compare shares, not absolutes", "kernels": ks},
              open(os.path.join(out_dir, "launches_b32_summary.json"), "w"), indent=1)
    print(json.dumps(ks, indent=1))
