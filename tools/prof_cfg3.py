"""Config-3 gradients through the cached plan (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_2512_23183_b200 import lq
w = W.config3()
for _ in range(int(os.environ.get("REPS", "4"))):
    lq.lq_param_shift_grad(w.n, w.gates, w.theta, w.terms)
torch.cuda.synchronize()
