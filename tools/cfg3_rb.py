"""Config-3 gradient device time per register-tile size (LQ_OPT_REG_BITS)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2512_23183_b200 import lq
st = torch.cuda.current_stream()
w = W.config3()
npar = len(w.theta)
th = torch.tensor(w.theta, device="cuda")
ref = None
for rb in [int(x) for x in os.environ.get("RBS", "4,3,2").split(",")]:
    lq.lq_set_option(lq.LQ_OPT_REG_BITS, rb)
    P = lq.lq_psr_create(w.n, w.gates, npar, w.terms, stream=st)
    g = torch.zeros(npar, dtype=torch.float64, device="cuda")
    e = torch.zeros(1, dtype=torch.float64, device="cuda")
    for _ in range(3):
        lq.lq_psr_run(P, th.data_ptr(), g.data_ptr(), e.data_ptr())
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(200):
        lq.lq_psr_run(P, th.data_ptr(), g.data_ptr(), e.data_ptr())
    b.record(st); torch.cuda.synchronize()
    gg = g.cpu().numpy()
    if ref is None:
        ref = gg
    print(json.dumps({"reg_bits": rb, "us_per_gradient": a.elapsed_time(b) / 200 * 1e3, "passes": lq.lq_psr_stats(P)[3],
                      "max_dev_vs_rb4": float(np.abs(gg - ref).max())}), flush=True)
    lq.lq_psr_free(P)
