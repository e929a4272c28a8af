"""Top stalled SASS instructions from an `ncu --page source --csv --print-source sass` export."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) >= len(hdr) - 1]
f = lambda x: float(x.replace(",", "")) if x and x.replace(",", "").replace(".", "").isdigit() else 0.0
key = 'Warp Stall Sampling (All Samples)'
tot = sum(f(d[key]) for d in data)
stalls = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
print("total samples", tot, "instructions", len(data))
agg = {k: sum(f(d[k]) for d in data) for k in stalls}
print("by reason:", ", ".join(f"{k[6:]}={100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for i, d in sorted(enumerate(data), key=lambda x: -f(x[1][key]))[:n]:
    top = sorted(((d[k], k[6:]) for k in stalls if f(d[k]) > 0), key=lambda x: -f(x[0]))[:2]
    print(f"{i:6d} {100*f(d[key])/tot:5.1f}% exec={f(d['Instructions Executed']):9.0f} {d['Source'].strip()[:70]:70s} {top}")
