"""BASELINE configs 1-3 on one B200 (latency-bound shapes):
config 1 = init_random(n=10) + 200 random gates + QFT(10) + full readback,
config 2 = QFT(20) of the seeded random state and of 16 basis states,
config 3 = one n=4 parameter-shift gradient (97 circuits).  CUDA events
(device time of the calls) and wall time per run, median of R runs."""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2512_23183_b200 import lq
st = torch.cuda.current_stream()
R = int(os.environ.get("R", "50"))
def measure(fn):
    fn(); torch.cuda.synchronize()
    dev, wall = [], []
    for _ in range(R):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter(); a.record(st); fn(); b.record(st); torch.cuda.synchronize()
        wall.append((time.perf_counter() - t0) * 1e3); dev.append(a.elapsed_time(b))
    return statistics.median(dev), statistics.median(wall)
out = []
w1 = W.config1()
sv = lq.StateVector(w1.n, stream=st)
def c1():
    sv.init_random(w1.seed).apply(w1.gates).qft()
    return sv.read()
d, wl = measure(c1)
upd = (len(w1.gates) + W.qft_gate_count(w1.n)) * 2 ** w1.n
out.append({"config": 1, "n": w1.n, "gates": len(w1.gates) + W.qft_gate_count(w1.n), "device_us": 1e3 * d,
            "wall_us": 1e3 * wl, "updates_per_s": upd / (wl / 1e3), "note": "incl. init_random and the 16 KiB readback"})
sv.free()
w2 = W.config2()
sv = lq.StateVector(w2.n, stream=st)
def c2():
    sv.init_random(w2.seed).qft()
    for k in w2.basis:
        sv.init_basis(int(k)).qft()
d, wl = measure(c2)
upd = 17 * W.qft_gate_count(w2.n) * 2 ** w2.n
out.append({"config": 2, "n": w2.n, "states": 17, "device_ms": d, "wall_ms": wl, "updates_per_s": upd / (d / 1e3),
            "note": "17 QFT(20) incl. state preparation; 16 MiB states stay L2-resident"})
sv.free()
w3 = W.config3()
d, wl = measure(lambda: lq.lq_param_shift_grad(w3.n, w3.gates, w3.theta, w3.terms))
upd = (2 * len(w3.theta) + 1) * len(w3.gates) * 2 ** w3.n
out.append({"config": 3, "n": w3.n, "circuits": 2 * len(w3.theta) + 1, "device_us": 1e3 * d, "wall_us": 1e3 * wl,
            "updates_per_s": upd / (wl / 1e3), "note": "host theta in, gradient out (lq_param_shift_grad, cached plan)"})
for o in out:
    print(json.dumps(o), flush=True)
