"""Standalone calls at n=30: CUDA-event time of the whole call vs the sum of
its kernels' event times (LQ_OPT_KERNEL_TIMING) -> host overhead per call."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2512_23183_b200 import lq
n = int(os.environ.get("LQ_COMP_N", "30"))
st = torch.cuda.current_stream()
sv = lq.StateVector(n, stream=st); sv.init_random(1)
xyz = W.xyz_terms(n)
w5 = W.config5(n, 1)
def measure(name, fn, R=5):
    fn(); torch.cuda.synchronize()
    walls, kern, hosts = [], [], []
    for _ in range(R):
        lq.lq_set_option(lq.LQ_OPT_KERNEL_TIMING, 0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(st); t0 = time.perf_counter(); fn(); t1 = time.perf_counter(); b.record(st); torch.cuda.synchronize()
        walls.append(a.elapsed_time(b)); hosts.append((t1 - t0) * 1e3)
        lq.lq_set_option(lq.LQ_OPT_KERNEL_TIMING, 1); lq.lq_kernel_timing_reset()
        fn(); torch.cuda.synchronize()
        kern.append(sum(lq.lq_kernel_timing(c)[0] for c in range(5)))
    lq.lq_set_option(lq.LQ_OPT_KERNEL_TIMING, 0)
    print(f"{name}: event {statistics.median(walls):.2f} ms, kernels {statistics.median(kern):.2f} ms, host call {statistics.median(hosts):.2f} ms", flush=True)
measure("QFT", lambda: sv.qft())
measure("expval xyz", lambda: sv.expval(xyz))
measure("expval Z0", lambda: sv.expval([(1.0, 0, 1)]))
measure("cfg5 1000 gates", lambda: sv.apply(w5.gates), 3)
measure("init_random", lambda: sv.init_random(3))
