"""Quick timing probe: QFT(30) (automatic and 11-bit tiles) and the config-4
gradient at tile bits KS (env), CUDA events, min of 3."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2512_23183_b200 import lq
st = torch.cuda.current_stream()
tag = "probe"
if "FF" in os.environ: lq.lq_set_option(lq.LQ_OPT_FIRST_PASS_FREE, int(os.environ["FF"]))
if "RB" in os.environ: lq.lq_set_option(lq.LQ_OPT_REG_BITS, int(os.environ["RB"]))
if "CO" in os.environ: lq.lq_set_option(lq.LQ_OPT_COALESCE_BITS, int(os.environ["CO"]))
if "BUDGET" in os.environ: lq.lq_set_option(lq.LQ_OPT_PASS_BUDGET, int(os.environ["BUDGET"]))
def timed(fn, R=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(R):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)
if "qft" in sys.argv:
    sv = lq.StateVector(30, stream=st); sv.init_random(1)
    for K in (0, 11):
        lq.lq_set_option(lq.LQ_OPT_TILE_BITS, K)
        print(tag, f"QFT(30) K={K}: {timed(lambda: sv.qft()):.2f} ms", flush=True)
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, 0)
    sv.free(); del sv; torch.cuda.empty_cache()
if "cfg4" in sys.argv:
    w = W.config4()
    npar = len(w.theta)
    th = torch.tensor(w.theta, device="cuda"); g = torch.zeros(npar, dtype=torch.float64, device="cuda")
    e = torch.zeros(1, dtype=torch.float64, device="cuda")
    for K in [int(k) for k in os.environ.get("KS", "12").split()]:
        lq.lq_set_option(lq.LQ_OPT_TILE_BITS, K)
        P = lq.lq_psr_create(w.n, w.gates, npar, w.terms, stream=st)
        ms = timed(lambda: lq.lq_psr_run(P, th.data_ptr(), g.data_ptr(), e.data_ptr()), 1)
        print(tag, f"cfg4 K={K} gradient {ms:.1f} ms passes {lq.lq_psr_stats(P)[3]} E={e.item():.15f}", flush=True)
        lq.lq_psr_free(P)
