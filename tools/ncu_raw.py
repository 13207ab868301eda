"""Print the key metrics of every launch in an `ncu --page raw --csv` dump."""
import csv, io, sys
rows = list(csv.reader(open(sys.argv[1])))
h, units, data = rows[0], rows[1], rows[2:]
col = {k: i for i, k in enumerate(h)}
def val(r, k):
    if k not in col: return float("nan")
    v = r[col[k]].replace(",", "")
    try: x = float(v)
    except ValueError: return v
    return x * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "ns": 1e-3, "us": 1, "ms": 1e3, "msecond": 1e3, "usecond": 1, "nsecond": 1e-3}.get(units[col[k]], 1)
keys = [("us", "gpu__time_duration.sum"), ("dramGB", None), ("GB/s", None),
        ("fp64%", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        ("issue%", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
        ("warps", "sm__warps_active.avg.per_cycle_active"),
        ("regs", "launch__registers_per_thread"), ("grid", "launch__grid_size"), ("blk", "launch__block_size")]
extra = sys.argv[2:]  # more metric names
for r in data:
    us = val(r, "gpu__time_duration.sum")
    dr = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    name = r[col["Kernel Name"]][:28]
    out = [name, f"us={us:.1f}", f"dram={dr/1e9:.3f}GB", f"{dr/us/1e3:.0f}GB/s"]
    for k, m in keys[3:]:
        out.append(f"{k}={val(r, m)}")
    for m in extra:
        out.append(f"{m.split('.')[0][-30:]}={val(r, m)}")
    print(" ".join(str(x) for x in out))
