"""Config-3 VQE loop (200 Adam iterations) and one-shot gradient device time
with CUDA graphs off / on (LQ_OPT_GRAPHS), interleaved A/B
(profiles/r02/graphs_config3.jsonl)."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import workloads as W
from paper_2512_23183_b200 import lq
st = torch.cuda.current_stream()
w = W.config3()
for graphs in (0, 1, 0, 1):
    lq.lq_set_option(lq.LQ_OPT_GRAPHS, graphs)
    lq.lq_vqe_adam(w.n, w.gates, w.theta, w.terms, max_iter=3)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    th, tr, T = lq.lq_vqe_adam(w.n, w.gates, w.theta, w.terms, max_iter=200, tol=0.0)
    b.record(st); torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    # one-shot gradients through the cached plan (config 3)
    for _ in range(5): lq.lq_param_shift_grad(w.n, w.gates, w.theta, w.terms)
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    for _ in range(200): lq.lq_param_shift_grad(w.n, w.gates, w.theta, w.terms)
    wall = (time.perf_counter() - t0) / 200 * 1e6
    print(json.dumps({"graphs": graphs, "vqe_ms_per_iter": ms / (T + 1), "iters": T, "grad_wall_us": wall, "E_last": tr[-1]}), flush=True)
