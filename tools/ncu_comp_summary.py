"""Summarise ncu raw CSVs of the companion kernels (tools/run_prof_comp.sh) into
one text table: per launch time, DRAM bytes, DRAM GB/s (fraction of the
measured peak), FP64 pipe and issue utilisation, top stalls."""
import csv, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6544.0
out = []
for name, path in zip(sys.argv[1::2], sys.argv[2::2]):
    rows = list(csv.reader(open(path)))
    h, u, d = rows[0], rows[1], rows[2:]
    ix = {k: i for i, k in enumerate(h)}
    def val(r, k):
        v = r[ix[k]].replace(",", "")
        try:
            x = float(v)
        except ValueError:
            return 0.0
        return x * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "msecond": 1e3, "nsecond": 1e-3, "us": 1, "ms": 1e3, "ns": 1e-3}.get(u[ix[k]], 1)
    pre = "smsp__pcsamp_warps_issue_stalled_"
    scols = [k for k in h if k.startswith(pre) and not k.endswith("_not_issued")]
    out.append(f"== {name} ({path})")
    for r in d:
        us = val(r, "gpu__time_duration.sum")
        dram = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        st = sorted(((val(r, k), k[len(pre):]) for k in scols), reverse=True)
        tot = sum(x for x, _ in st) or 1
        out.append(f"{r[ix['Kernel Name']][:22]:22s} us={us:9.1f} dram={dram / 1e9:7.3f}GB {dram / us / 1e3:7.0f}GB/s "
                   f"({dram / us / 1e3 / peak:.2f}) fp64={val(r, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):4.1f}% "
                   f"issue={val(r, 'sm__inst_issued.avg.pct_of_peak_sustained_active'):4.1f}% "
                   + " ".join(f"{k}={100 * x / tot:.0f}%" for x, k in st[:3]))
print("\n".join(out))
