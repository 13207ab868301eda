"""Per-pass view of one config-4 gradient (for ncu per-launch metrics): runs
the gradient once with LQ_OPT_RELABEL_STORES = $RELABEL (default: library
default) and writes the plan's per-pass tiles / store frames / algorithmic
bytes to gpurun_out/pass_plan_<relabel>.json."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_2512_23183_b200 import lq
w = W.config4()
if os.environ.get("RELABEL"):
    lq.lq_set_option(lq.LQ_OPT_RELABEL_STORES, int(os.environ["RELABEL"]))
rl = lq.lq_get_option(lq.LQ_OPT_RELABEL_STORES)
npar = len(w.theta)
th = torch.tensor(w.theta, device="cuda")
g = torch.zeros(npar, dtype=torch.float64, device="cuda")
e = torch.zeros(1, dtype=torch.float64, device="cuda")
P = lq.lq_psr_create(w.n, w.gates, npar, w.terms, stream=torch.cuda.current_stream())
lq.lq_psr_run(P, th.data_ptr(), g.data_ptr(), e.data_ptr())
torch.cuda.synchronize()
lq.lq_set_option(lq.LQ_OPT_EXPORT_PSR, 1)
plan = lq.lq_plan_export_json(w.n, w.gates, w.terms)
os.makedirs("gpurun_out", exist_ok=True)
json.dump({"relabel": rl, "pass_bytes": lq.lq_psr_pass_bytes(P),
           "passes": [{k: p[k] for k in ("kind", "T", "Sstore", "oop", "spos", "flags")} for p in plan["passes"]]},
          open("gpurun_out/pass_plan_%d.json" % rl, "w"))
print("E", e.item())
