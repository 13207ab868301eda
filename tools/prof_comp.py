"""One invocation of a companion kernel class at n = LQ_COMP_N (default 28)
for ncu captures: mode qft | expv | init | diag | rand40."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2512_23183_b200 import lq
mode = sys.argv[1]
n = int(os.environ.get("LQ_COMP_N", "28"))
sv = lq.StateVector(n)
sv.init_random(1)
if mode == "qft":
    sv.qft()
elif mode == "expv":
    print(sv.expval(W.xyz_terms(n)))
elif mode == "init":
    sv.init_random(5)
elif mode == "diag":
    sv.apply([("RZ", q, -1, -1, 0.1 * q) for q in range(n)] + [("CZ", q, q + 1, -1, 0.0) for q in range(n - 1)])
torch.cuda.synchronize()
print("ok", mode, lq.lq_launch_count())
