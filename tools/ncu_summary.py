"""Summarise an ncu --set full report of the tile-pass launches of one
config-4 batch (B circuits per launch) into profiles/ncu_k_tile_summary.json:
per launch dram read+write bytes vs the algorithmic bytes of that pass."""
import csv, io, json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
rep, out, src = sys.argv[1], sys.argv[2], sys.argv[3]
if rep.endswith(".csv"):   # an `ncu --page raw --csv` dump made on the GPU box
    txt = open(rep).read()
else:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, units, data = rows[0], rows[1], rows[2:]
col = {k: i for i, k in enumerate(h)}
def val(r, k):
    v = r[col[k]].replace(",", "")
    x = float(v) if v else 0.0
    u = units[col[k]]
    return x * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "ns": 1e-3, "us": 1, "ms": 1e3}.get(u, 1)
import workloads as W
w = W.config4()
B = int(os.environ.get("LQ_SUMMARY_B", "4"))   # circuits per launch in the capture (lq_psr_create's batch)
# algorithmic bytes per pass of the captured plan, written on the GPU box by
# tools/prof_cfg4.py (lq_psr_pass_bytes: support tracking, write-only first
# pass, read-only and final passes)
pb = json.load(open(os.environ.get("LQ_PASS_BYTES", "gpurun_out/cfg4_pass_bytes.json")))
passes = [p for p in pb["passes"] if p["kind"] == 0]
launches = []
for i, r in enumerate(data):
    if i >= len(passes):
        break
    alg = B * passes[i]["bytes_per_circuit"]
    dr, dw = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
    launches.append({"pass": i, "us": round(val(r, "gpu__time_duration.sum"), 2), "dram_read": dr, "dram_write": dw,
                     "alg_bytes": alg, "traffic_over_alg": round((dr + dw) / alg, 4),
                     "fp64_pipe_pct": round(val(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"), 1),
                     "issue_pct": round(val(r, "sm__inst_issued.avg.pct_of_peak_sustained_active"), 1),
                     "regs": int(val(r, "launch__registers_per_thread")), "grid": int(val(r, "launch__grid_size"))})
tot_dram = sum(l["dram_read"] + l["dram_write"] for l in launches)
tot_alg = sum(l["alg_bytes"] for l in launches)
s = {"source": src, "n_qubits": w.n, "circuits_per_launch": B, "launches": len(launches),
     "dram_bytes_per_circuit_pass": tot_dram / len(launches) / B,
     "dram_bytes_per_launch": tot_dram / len(launches), "algorithmic_bytes_per_launch": tot_alg / len(launches),
     "traffic_over_algorithmic": tot_dram / tot_alg, "per_launch": launches}
json.dump(s, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in s.items() if k != "per_launch"}))
