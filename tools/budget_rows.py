"""FP64 pass budget sweep (LQ_OPT_STATE_PASS_BUDGET; arguments: budgets) on the
single-state workloads: Trotter XYZ step at n = 30 (f1), the config-1 random
alphabet (200 gates) and the config-5 circuit at n = 30, each from a fresh
state, median of 3 warm reps.  One JSON object per line."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2512_23183_b200 import lq  # noqa: E402

n = int(os.environ.get("LQ_BUDGET_N", 30))
sv = lq.StateVector(n)
rand = W.random_circuit(n, 200, np.random.default_rng(1), np.random.default_rng(2))
cfg5 = W.config5(n, 1).gates


def tm(fn, init):
    ts = []
    for r in range(4):
        init()
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        c.record()
        torch.cuda.synchronize()
        if r:
            ts.append(a.elapsed_time(c))
    return statistics.median(ts)


K = int(os.environ.get("LQ_BUDGET_K", 0))   # tile bits (0 = automatic)
lq.lq_set_option(lq.LQ_OPT_TILE_BITS, K)
for b in [int(x) for x in sys.argv[1:]]:
    lq.lq_set_option(lq.LQ_OPT_STATE_PASS_BUDGET, b)
    lq.lq_psr_cache_clear()
    out = {"budget": b, "n": n, "K": K}
    out["trotter_8_steps_ms"] = tm(lambda: sv.trotter_xyz(1.0, 0.7, 0.4, 2.0, 1.0, 0.0, 0.01, 8, 8),
                                   lambda: sv.init_basis((1 << n) - 1))
    out["random200_ms"] = tm(lambda: sv.apply(rand), lambda: sv.init_random(3))
    out["cfg5_1000_ms"] = tm(lambda: sv.apply(cfg5), lambda: sv.init_random(3))
    print(json.dumps(out), flush=True)
lq.lq_set_option(lq.LQ_OPT_STATE_PASS_BUDGET, 800)
lq.lq_set_option(lq.LQ_OPT_TILE_BITS, 0)
