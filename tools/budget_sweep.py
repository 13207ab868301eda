"""Config-4 gradient time vs the planner's FP64 pass budget
(LQ_OPT_PASS_BUDGET); arguments are budgets."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2512_23183_b200 import lq
w = W.config4()
npar = len(w.theta)
th = torch.tensor(w.theta, device="cuda"); g = torch.zeros(npar, dtype=torch.float64, device="cuda")
e = torch.zeros(1, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
for spec in sys.argv[1:]:
    b = int(spec.split(":")[0])
    lq.lq_set_option(lq.LQ_OPT_PASS_BUDGET, b)
    P = lq.lq_psr_create(w.n, w.gates, npar, w.terms, stream=st)
    lq.lq_psr_run(P, th.data_ptr(), g.data_ptr(), e.data_ptr()); torch.cuda.synchronize()
    ts = []
    for _ in range(2):
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); lq.lq_psr_run(P, th.data_ptr(), g.data_ptr(), e.data_ptr()); c.record(st); torch.cuda.synchronize()
        ts.append(a.elapsed_time(c))
    print(f"budget={b}: passes {lq.lq_psr_stats(P)[3]} gradient {min(ts):.1f} ms E={e.item():.15f}", flush=True)
    lq.lq_psr_free(P)
