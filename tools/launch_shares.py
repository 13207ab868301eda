"""Per-kernel share of an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv, json, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, iv, iu, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Metric Name")
tot = collections.Counter(); cnt = collections.Counter()
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    v = float(r[iv].replace(",", "")) * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0}.get(r[iu], 1.0)
    name = r[ik].split("(")[0] if not r[ik].startswith("void") else r[ik][:90]
    tot[name] += v; cnt[name] += 1
S = sum(tot.values())
out = {"command": sys.argv[2] if len(sys.argv) > 2 else "", "note": sys.argv[3] if len(sys.argv) > 3 else "",
       "kernels": {k: {"launches": cnt[k], "total_us": round(v, 1), "avg_us": round(v / cnt[k], 1), "share": round(v / S, 4)}
                   for k, v in tot.most_common()}}
print(json.dumps(out, indent=1))
