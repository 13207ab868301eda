import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np, torch
import workloads as W
from paper_2512_23183_b200 import lq
w = W.config4()
ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
def timed(f, reps=1):
    f(); torch.cuda.synchronize()
    ev0.record()
    for _ in range(reps): f()
    ev1.record(); torch.cuda.synchronize()
    return ev0.elapsed_time(ev1) / reps
for rb in (4, 3):
    lq.lq_set_option(lq.LQ_OPT_REG_BITS, rb)
    t = time.time(); g, e = lq.lq_param_shift_grad(w.n, w.gates, w.theta, w.terms); dt = time.time() - t
    print(f"rb={rb} cfg4 grad: {dt:.3f}s  E={e:.12f} |g|max={np.abs(g).max():.6f}", flush=True)
    sv = lq.StateVector(30); sv.init_random(1)
    w5 = W.config5(30, 1)
    ms = timed(lambda: sv.apply(w5.gates))
    print(f"rb={rb} n=30 1000-gate circuit {ms:.1f} ms, {lq.lq_plan_describe(30, w5.gates)[0]} passes", flush=True)
    ms = timed(lambda: sv.qft())
    print(f"rb={rb} n=30 QFT {ms:.2f} ms  {96*2**30/ms/1e6:.0f} GB/s-equiv (3 passes)", flush=True)
    sv.free(); del sv; torch.cuda.empty_cache()
lq.lq_set_option(lq.LQ_OPT_REG_BITS, 4)
sv = lq.StateVector(30); sv.init_random(1)
for kind in [("H", 0), ("H", 29), ("RZ", 3)]:
    g = [(kind[0], kind[1], -1, -1, 0.3 if kind[0] == "RZ" else 0.0)]
    ms = timed(lambda: sv.apply(g), 5)
    print(f"n=30 single {kind}: {ms:.3f} ms  {32*2**30/ms/1e6:.0f} GB/s", flush=True)
ms = timed(lambda: sv.expval(W.xyz_terms(30)))
print(f"n=30 expval xyz {ms:.2f} ms", flush=True)
