"""Config-5 shape on ONE GPU: the 1000-gate random circuit (30 % on the top
m qubits) + QFT at n (default 30), unsharded and as G in-process shards
(lq_sv_alloc_group: same schedules/kernels as the NCCL path, swaps as device
copies).  CUDA-event times per phase."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2512_23183_b200 import lq
n = int(os.environ.get("N", "30"))
st = torch.cuda.current_stream()
def ev():
    e = torch.cuda.Event(enable_timing=True); e.record(st); return e
res = []
for G in [int(g) for g in os.environ.get("GS", "1,2,4").split(",")]:
    m = max(G.bit_length() - 1, 1)
    w = W.config5(n, m, 1000)
    if G == 1:
        sv = lq.StateVector(n, stream=st)
    else:
        sv = lq.ShardedState(n, group_world=G, stream=st)
    for rep in range(2):   # first rep compiles (JIT) and warms up
        torch.cuda.synchronize()
        e0 = ev(); sv.init_random(w.seed); e1 = ev(); sv.apply(w.gates); e2 = ev(); sv.qft(); e3 = ev()
        torch.cuda.synchronize()
    r = {"n": n, "G": G, "m": m, "init_ms": e0.elapsed_time(e1), "circuit_ms": e1.elapsed_time(e2),
         "qft_ms": e2.elapsed_time(e3), "norm2": sv.norm2(), "amp0": [float(x) for x in sv.gather([0, 12345])[:1].view(np.float64)]}
    if G > 1:
        d1 = lq.lq_dist_schedule_json(n, m, w.gates)
        d2 = lq.lq_dist_schedule_json(n, m, [], qft=1)
        r["circuit_swaps"], r["qft_swaps"] = d1["n_swaps"], d2["n_swaps"]
        r["circuit_tile_passes"] = sum(len(s["plan"]["passes"]) for s in d1["steps"] if s["kind"] == "local")
        r["qft_tile_passes"] = sum(len(s["plan"]["passes"]) for s in d2["steps"] if s["kind"] == "local")
    else:
        r["circuit_tile_passes"] = lq.lq_plan_describe(n, w.gates)[0]
    print(json.dumps(r), flush=True)
    sv.free(); del sv; torch.cuda.empty_cache()
