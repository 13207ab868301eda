"""Register-tile size / occupancy probe: QFT(30), XYZ expectation at n=30 and
the config-4 gradient under LQ_OPT_REG_BITS = RB and LQ_JIT_MINBLOCKS (env)."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2512_23183_b200 import lq
rb = int(os.environ.get("RB", "4"))
lq.lq_set_option(lq.LQ_OPT_REG_BITS, rb)
st = torch.cuda.current_stream()
def timed(fn, R=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(R):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)
tag = f"RB={rb} MB={os.environ.get('LQ_JIT_MINBLOCKS', 'auto')}"
n = 30
if "qft" in sys.argv:
    sv = lq.StateVector(n, stream=st); sv.init_random(1)
    print(tag, f"QFT(30) {timed(lambda: sv.qft()):.2f} ms", flush=True)
    print(tag, f"expval xyz(30) {timed(lambda: sv.expval(W.xyz_terms(n))):.2f} ms", flush=True)
    sv.free(); del sv; torch.cuda.empty_cache()
if "cfg4" in sys.argv:
    w = W.config4()
    npar = len(w.theta)
    th = torch.tensor(w.theta, device="cuda"); g = torch.zeros(npar, dtype=torch.float64, device="cuda")
    e = torch.zeros(1, dtype=torch.float64, device="cuda")
    P = lq.lq_psr_create(w.n, w.gates, npar, w.terms, stream=st)
    ms = timed(lambda: lq.lq_psr_run(P, th.data_ptr(), g.data_ptr(), e.data_ptr()), 1)
    print(tag, f"cfg4 gradient {ms:.1f} ms passes {lq.lq_psr_stats(P)[3]} E={e.item():.15f}", flush=True)
    lq.lq_psr_free(P)
