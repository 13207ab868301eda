"""One config-4 parameter-shift gradient (for ncu launch lists / captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2512_23183_b200 import lq
w = W.config4()
layers = int(os.environ.get("LQ_PROF_LAYERS", "10"))
gates = w.gates[: layers * 3 * w.n]
npar = layers * 2 * w.n
g, e = lq.lq_param_shift_grad(w.n, gates, w.theta[:npar], w.terms)
torch.cuda.synchronize()
print("E", e, "launches", lq.lq_launch_count())
# per-pass algorithmic bytes of the same plan (tools/ncu_summary.py)
import json
P = lq.lq_psr_create(w.n, gates, npar, w.terms, stream=torch.cuda.current_stream())
os.makedirs("gpurun_out", exist_ok=True)
json.dump({"n": w.n, "passes": [{"kind": k, "bytes_per_circuit": b} for k, b in lq.lq_psr_pass_bytes(P)]},
          open("gpurun_out/cfg4_pass_bytes.json", "w"))
lq.lq_psr_free(P)
