import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np, torch
import workloads as W
from paper_2512_23183_b200 import lq
w = W.config4()
torch.cuda.synchronize()
for it in range(3):
    t = time.time()
    g, e = lq.lq_param_shift_grad(w.n, w.gates, w.theta, w.terms)
    dt = time.time() - t
    print(f"cfg4 grad: {dt:.3f}s  E={e:.12f} |g|max={np.abs(g).max():.6f} launches={lq.lq_launch_count()}")
# single-pass timing at n=30
sv = lq.StateVector(30)
sv.init_random(1)
torch.cuda.synchronize()
for kind in [("H", 0), ("H", 29), ("H", 15), ("RZ", 3)]:
    for fusion in (0, 1):
        lq.lq_set_option(lq.LQ_OPT_FUSION, fusion)
        g = [(kind[0], kind[1], -1, -1, 0.3 if kind[0]=="RZ" else 0.0)]
        sv.apply(g); torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(5): sv.apply(g)
        t1.record(); torch.cuda.synchronize()
        ms = t0.elapsed_time(t1)/5
        print(f"n=30 {kind} fusion={fusion}: {ms:.3f} ms  {32*2**30/ms/1e6:.0f} GB/s")
lq.lq_set_option(lq.LQ_OPT_FUSION, 1)
w5 = W.config5(30, 1)
sv.apply(w5.gates[:50]); torch.cuda.synchronize()
t0.record(); sv.apply(w5.gates); t1.record(); torch.cuda.synchronize()
print("n=30 1000-gate circuit", t0.elapsed_time(t1), "ms", lq.lq_plan_describe(30, w5.gates)[0], "passes")
t0.record(); sv.qft(); t1.record(); torch.cuda.synchronize()
ms = t0.elapsed_time(t1); print("n=30 QFT", ms, "ms", 96*2**30/ms/1e6, "GB/s (3 passes)")
t0.record(); e = sv.expval(W.xyz_terms(30)); t1.record(); torch.cuda.synchronize()
print("n=30 expval xyz", t0.elapsed_time(t1), "ms")
