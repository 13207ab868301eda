"""Config-1 (n = 10: init_random, 200 random gates, QFT(10), readback)
device time per run under planner variants (tile bits / register bits).
Usage: python tools/cfg1_variants.py [K:R ...]   (0 = automatic)"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2512_23183_b200 import lq
st = torch.cuda.current_stream()
w = W.config1()
ref = None
for v in (sys.argv[1:] or ["0:4", "0:3", "0:2", "8:4", "8:3", "7:3", "7:2"]):
    K, R = (int(x) for x in v.split(":"))
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, K)
    lq.lq_set_option(lq.LQ_OPT_REG_BITS, R)
    sv = lq.StateVector(w.n, stream=st)
    def run():
        sv.init_random(w.seed).apply(w.gates).qft()
        return sv.read()
    for _ in range(3):
        out = run()
    torch.cuda.synchronize()
    ds = []
    for _ in range(30):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); out = run(); b.record(st); torch.cuda.synchronize()
        ds.append(a.elapsed_time(b) * 1e3)
    if ref is None:
        ref = out
    print(json.dumps({"K": K, "R": R, "device_us": statistics.median(ds), "max_dev": float(np.abs(out - ref).max()),
                      "launches_per_run": None}), flush=True)
    sv.free()
