"""Time QFT(n), init_random and the XYZ expectation at n = LQ_COMP_N (30)
under several tile sizes (CUDA events, median of 5)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2512_23183_b200 import lq
n = int(os.environ.get("LQ_COMP_N", "30"))
N = 1 << n
st = torch.cuda.current_stream()
sv = lq.StateVector(n, stream=st)
sv.init_random(1)
def timed(fn, R=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(R):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)
peak = 6544.0
for K in [int(x) for x in os.environ.get("KS", "11 12").split()]:
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, K)
    l0 = lq.lq_launch_count(); sv.qft(); npass = lq.lq_launch_count() - l0
    ms = timed(lambda: sv.qft())
    print(f"QFT({n}) K={K}: {npass} passes {ms:.3f} ms frac={32*npass*N/(ms/1e3)/1e9/peak:.3f} (vs 3-pass floor {32*3*N/(ms/1e3)/1e9/peak:.3f})", flush=True)
lq.lq_set_option(lq.LQ_OPT_TILE_BITS, 0)
ms = timed(lambda: sv.init_random(5))
print(f"init_random: {ms:.3f} ms  write-frac={16*N/(ms/1e3)/1e9/peak:.3f}", flush=True)
xyz = W.xyz_terms(n)
ms = timed(lambda: sv.expval(xyz))
ep = lq.lq_plan_export_json(n, [], xyz)
print(f"expval xyz: {ms:.3f} ms, {len(ep['passes'])} passes frac={16*len(ep['passes'])*N/(ms/1e3)/1e9/peak:.3f}", flush=True)
