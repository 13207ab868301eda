"""Config-4 gradient timing for several tile sizes (JIT)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2512_23183_b200 import lq
w = W.config4()
npar = len(w.theta)
th = torch.tensor(w.theta, device="cuda"); g = torch.zeros(npar, dtype=torch.float64, device="cuda")
e = torch.zeros(1, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
lq.lq_set_option(lq.LQ_OPT_JIT, 2)
ref = None
cb = int(os.environ.get("LQ_COALESCE", "3"))
lq.lq_set_option(lq.LQ_OPT_PASS_BUDGET, int(os.environ.get("LQ_BUDGET", "0")))
lq.lq_set_option(lq.LQ_OPT_COALESCE_BITS, cb)
for K in [int(k) for k in os.environ.get("KS", "12,11").split(",")]:
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, K)
    t = time.time()
    P = lq.lq_psr_create(w.n, w.gates, npar, w.terms, stream=st)
    tc = time.time() - t
    lq.lq_psr_run(P, th.data_ptr(), g.data_ptr(), e.data_ptr()); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); lq.lq_psr_run(P, th.data_ptr(), g.data_ptr(), e.data_ptr()); b.record(); torch.cuda.synchronize()
    gg = g.cpu().numpy().copy()
    if ref is None: ref = gg
    print(f"budget={lq.lq_get_option(lq.LQ_OPT_PASS_BUDGET)} coalesce={cb} K={K}: create {tc:.1f}s  passes {lq.lq_psr_stats(P)[3]}  gradient {a.elapsed_time(b):.1f} ms  "
          f"E={e.item():.15f}  max|dg| vs first {np.abs(gg-ref).max():.2e}", flush=True)
    lq.lq_psr_free(P)
print("jit stats", lq.lq_jit_stats())
