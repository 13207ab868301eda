"""HBM-roofline companions at n = 30: every kernel class on
a 16 GiB complex128 state, timed with CUDA events (median of R reps after
warm-up), algorithmic bytes / time vs the measured HBM peak.  Writes one
JSON object to stdout."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2512_23183_b200 import lq

n = int(os.environ.get("LQ_COMP_N", "30"))
R = int(os.environ.get("LQ_COMP_REPS", "5"))
N = 1 << n
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
st = torch.cuda.current_stream()
sv = lq.StateVector(n, stream=st)
sv.init_random(1)
torch.cuda.synchronize()

def timed(fn):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(R):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)

out = {"n": n, "state_GiB": N * 16 / 2**30, "peak_gbs": peak, "reps": R, "rows": []}
def row(name, bytes_per_amp, ms, note=""):
    gbs = bytes_per_amp * N / (ms / 1e3) / 1e9
    out["rows"].append({"kernel": name, "ms": round(ms, 3), "alg_bytes_per_amp": bytes_per_amp,
                        "GBps": round(gbs, 1), "frac_measured_peak": round(gbs / peak, 3),
                        "frac_8TBps": round(gbs / 8000, 3), "note": note})
    print(json.dumps(out["rows"][-1]), flush=True)

lq.lq_set_option(lq.LQ_OPT_FUSION, 0)
for b in (0, 15, 29):
    q = n - 1 - b
    row(f"k_pair H on bit {b}", 32, timed(lambda: sv.apply([("H", q, -1, -1, 0.0)])), "unfused 1q pair pass")
row("k_pair CNOT bits (29,0)", 16, timed(lambda: sv.apply([("CNOT", 0, n - 1, -1, 0.0)])),
    "controlled permutation: only the controlled half moves (16 B/amp averaged over the state)")
row("k_diag RZ x8 (8 unfused diagonal passes)", 8 * 32, timed(lambda: sv.apply([("RZ", q, -1, -1, 0.1 * q) for q in range(8)] )),
    "unfused mode runs each diagonal op as its own k_diag pass")
lq.lq_set_option(lq.LQ_OPT_FUSION, 1)
# one fused diagonal pass: many diagonal gates
dg = [("RZ", q, -1, -1, 0.1 * q) for q in range(n)] + [("CZ", q, q + 1, -1, 0.0) for q in range(n - 1)]
npd = lq.lq_plan_describe(n, dg)[0]
row(f"tile pass: 59 diagonal gates ({npd} pass)", 32 * npd, timed(lambda: sv.apply(dg)), "FP64 pass budget splits the run")
# one tile pass of 40 random 1q/2q gates inside an 11-bit tile
rng = np.random.default_rng(3)
tq = list(range(n - 11, n))
tg = []
for _ in range(40):
    k = ["H", "RX", "RY", "RZ", "CNOT", "CZ", "T"][int(rng.integers(7))]
    a, c = [int(x) for x in rng.choice(tq, 2, replace=False)]
    tg.append((k, a, c if k in ("CNOT", "CZ") else -1, -1, float(rng.uniform(0, 6.28)) if k.startswith("R") else 0.0))
npass = lq.lq_plan_describe(n, tg)[0]
row(f"tile pass: 40 random gates ({npass} pass)", 32 * npass, timed(lambda: sv.apply(tg)))
row("tile pass: 10 RY+10 RZ layer slice", 32, timed(lambda: sv.apply(
    [("RY", q, -1, -1, 0.3 + q) for q in range(n - 10, n)] + [("RZ", q, -1, -1, 0.2 * q) for q in range(n - 10, n)])))
lq.lq_set_option(lq.LQ_OPT_KERNEL_TIMING, 1); lq.lq_kernel_timing_reset()
sv.qft(); torch.cuda.synchronize()
qp = lq.lq_kernel_timing(lq.KC_TILE)[1]   # tile passes only (not the op-table staging kernel)
lq.lq_set_option(lq.LQ_OPT_KERNEL_TIMING, 0)
row(f"QFT({n}) ({qp} tile passes, bit reversal = relabel)", 32 * qp, timed(lambda: sv.qft()))
xyz = W.xyz_terms(n)
ep = lq.lq_plan_export_json(n, [], xyz)
ne, nw = len(ep["passes"]), len(ep["wide_groups"])
row(f"expval XYZ chain ({len(xyz)} terms, {ne} read-only passes)", 16 * ne + 32 * nw, timed(lambda: sv.expval(xyz)),
    f"{len(ep['groups'])} x-mask groups in {ne} read-only tile passes, {nw} wide groups")
row("expval single Z group (read-only pass)", 16, timed(lambda: sv.expval([(1.0, 0, 1 << (n - 1))])))
row("init_random (norm pass + write pass)", 16, timed(lambda: sv.init_random(5)), "ALU-heavy: log + sincospi per amp")

# a9: one global-qubit swap in group mode (G = 2 shards in this process, the
# same swap kernel pair the NCCL path packs/unpacks): H on a global qubit =
# swap + the gate's pass; H on a local qubit = the pass alone.
sv.free(); del sv; torch.cuda.empty_cache()
sh = lq.ShardedState(n, group_world=2, stream=st)
sh.init_random(2)
def glob_q():   # the qubit currently on the global (rank) bit: the scheduler moves it after each swap
    qm = sh.qubit_map()
    return max(range(n), key=lambda q: qm[q])
def loc_q():
    qm = sh.qubit_map()
    return min(range(n), key=lambda q: qm[q])
t_loc = timed(lambda: sh.apply([("H", loc_q(), -1, -1, 0.0)]))
t_glob = timed(lambda: sh.apply([("H", glob_q(), -1, -1, 0.0)]))
row("sharded G=2: H on a local qubit (one pass)", 32, t_loc)
row("sharded G=2: global-local swap (H on the global qubit minus H on a local one)", 16, t_glob - t_loc,
    "k_swap_parts (k = 1): each shard exchanges the half of its amplitudes whose local bit differs from its rank bit, in place: "
    "16 B read + 16 B write per moved amplitude = 16 B per amplitude of the state")
print("JSON " + json.dumps(out))
