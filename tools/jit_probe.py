"""Config-4 gradient timing: interpreter vs JIT (CUDA events), plus JIT compile stats."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2512_23183_b200 import lq
w = W.config4()
layers = int(os.environ.get("LQ_PROF_LAYERS", "10"))
gates = w.gates[: layers * 3 * w.n]; npar = layers * 2 * w.n
th = torch.tensor(w.theta[:npar], device="cuda"); g = torch.zeros(npar, dtype=torch.float64, device="cuda")
e = torch.zeros(1, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
res = {}
for mode in (0, 2):
    lq.lq_set_option(lq.LQ_OPT_JIT, mode)
    t = time.time()
    P = lq.lq_psr_create(w.n, gates, npar, w.terms, stream=st)
    tc = time.time() - t
    lq.lq_psr_run(P, th.data_ptr(), g.data_ptr(), e.data_ptr()); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); lq.lq_psr_run(P, th.data_ptr(), g.data_ptr(), e.data_ptr()); b.record(); torch.cuda.synchronize()
    res[mode] = (g.cpu().numpy().copy(), float(e.item()))
    print(f"jit={mode}: create {tc:.1f}s  gradient {a.elapsed_time(b):.1f} ms  E={e.item():.15f}", flush=True)
    lq.lq_psr_free(P)
print("max |g_jit - g_interp| =", np.abs(res[0][0] - res[2][0]).max(), " dE =", abs(res[0][1] - res[2][1]))
print("jit stats", lq.lq_jit_stats(), "nproc", os.cpu_count())
