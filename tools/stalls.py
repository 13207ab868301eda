"""Per-launch stall breakdown (pc sampling) from an ncu raw CSV."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h, u, d = rows[0], rows[1], rows[2:]
ix = {k: i for i, k in enumerate(h)}
pre = "smsp__pcsamp_warps_issue_stalled_"
cols = [k for k in h if k.startswith(pre) and not k.endswith("_not_issued")]
for n, r in enumerate(d):
    vals = {}
    for k in cols:
        try: vals[k[len(pre):]] = float(r[ix[k]].replace(",", ""))
        except ValueError: pass
    tot = sum(vals.values()) or 1
    top = sorted(vals.items(), key=lambda x: -x[1])[:7]
    us = r[ix["gpu__time_duration.sum"]]
    print(n, us, " ".join(f"{k}={100*v/tot:.0f}%" for k, v in top))
