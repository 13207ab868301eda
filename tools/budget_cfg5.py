"""Config-5 circuit (1000 gates, m = 1) + QFT at n = LQ_CFG5_N (30) on one
GPU vs the planner's FP64 pass budget (arguments: budgets; 0 = no limit):
median of 3 reps from init_random, tile passes per step."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2512_23183_b200 import lq  # noqa: E402

n = int(os.environ.get("LQ_CFG5_N", 30))
w = W.config5(n, 1)
sv = lq.StateVector(n)
for b in [int(x) for x in sys.argv[1:]]:
    lq.lq_set_option(lq.LQ_OPT_STATE_PASS_BUDGET, b)
    lq.lq_psr_cache_clear()
    ts = []
    for r in range(4):
        sv.init_random(w.seed)
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sv.apply(w.gates)
        sv.qft()
        c.record()
        torch.cuda.synchronize()
        if r:
            ts.append(a.elapsed_time(c))
    lq.lq_kernel_timing_reset()
    lq.lq_set_option(lq.LQ_OPT_KERNEL_TIMING, 1)
    sv.init_random(w.seed)
    sv.apply(w.gates)
    sv.qft()
    torch.cuda.synchronize()
    lq.lq_set_option(lq.LQ_OPT_KERNEL_TIMING, 0)
    print(json.dumps({"n": n, "budget": b, "ms": statistics.median(ts),
                      "tile_passes": lq.lq_kernel_timing(lq.KC_TILE)[1]}), flush=True)
lq.lq_set_option(lq.LQ_OPT_STATE_PASS_BUDGET, 800)
