"""Measurements of the §8(f) rows on one B200 (CUDA events on the launch
stream): VQE outer loop (f2) iterations at config-3 and config-4 sizes,
Trotterised XYZ evolution (f1) at n = LQ_TROT_N (30), CRY four-term PSR
(f3) at n = 24.  One JSON object per line."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2512_23183_b200 import lq
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
st = torch.cuda.current_stream()
def ev():
    return torch.cuda.Event(enable_timing=True)
def emit(d):
    print(json.dumps(d), flush=True)

# f2: VQE iterations (one batched PSR gradient + device Adam + 8-byte readback each)
for cfg, iters in ((3, 200), (4, 2)):
    w = W.config3() if cfg == 3 else W.config4()
    lq.lq_vqe_adam(w.n, w.gates, w.theta, w.terms, max_iter=1)   # plan + JIT warm-up
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record(st)
    th, tr, T = lq.lq_vqe_adam(w.n, w.gates, w.theta, w.terms, max_iter=iters, tol=0.0)
    b.record(st); torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    ncirc = 2 * len(w.theta) + 1
    emit({"row": "f2 VQE (Adam on PSR gradients)", "config": cfg, "n": w.n, "params": len(w.theta),
          "iterations": T, "ms_per_iteration": ms / (T + 1), "E0": tr[0], "E_last": tr[-1],
          "gate_amp_updates_per_s": ncirc * len(w.gates) * 2 ** w.n * (T + 1) / (ms / 1e3)})

# f1: Trotter steps at n (state resident; 3(n-1) + n gates per step)
n = int(os.environ.get("LQ_TROT_N", "30"))
steps = int(os.environ.get("LQ_TROT_STEPS", "64"))
sv = lq.StateVector(n, stream=st).init_basis((1 << n) - 1)
sv.trotter_xyz(1.0, 0.7, 0.4, 2.0, 1.0, 0.0, 0.01, 8, 8)   # plan + JIT warm-up
torch.cuda.synchronize()
lq.lq_set_option(lq.LQ_OPT_KERNEL_TIMING, 1); lq.lq_kernel_timing_reset()
l0 = lq.lq_launch_count()
a, b = ev(), ev()
a.record(st)
E = sv.trotter_xyz(1.0, 0.7, 0.4, 2.0, 1.0, 0.0, 0.01, steps, steps)
b.record(st); torch.cuda.synchronize()
ms = a.elapsed_time(b)
tile_ms, tile_n = lq.lq_kernel_timing(0)
lq.lq_set_option(lq.LQ_OPT_KERNEL_TIMING, 0)
gps = 4 * n - 3

emit({"row": "f1 Trotter XYZ", "n": n, "steps": steps, "gates_per_step": gps, "ms": ms, "ms_per_step": ms / steps,
      "tile_launches": tile_n, "tile_ms": tile_ms,
      "tile_frac_of_peak_if_32B_per_amp": (tile_n * 32 * 2 ** n / (tile_ms / 1e3) / 1e9) / peak if tile_ms else None,
      "gate_amp_updates_per_s": steps * gps * 2 ** n / (ms / 1e3), "E_first_last": [E[0], E[-1]],
      "note": "includes the two final expectation evaluations; tile fraction assumes every tile pass reads and writes"})
sv.free(); del sv; torch.cuda.empty_cache()

# f3: a config-4-size ansatz whose entangler is CRY (4-term rule) instead of CNOT
n = 24
gates, p = [], 0
for layer in range(4):
    for q in range(n):
        gates.append(("RY", q, -1, p, 0.0)); p += 1
    for q in range(n - 1):
        gates.append(("CRY", q, q + 1, p, 0.0)); p += 1
theta = np.random.default_rng(5).uniform(0, 2 * np.pi, p)
terms = W.xyz_terms(n)
lq.lq_param_shift_grad(n, gates, theta, terms)
torch.cuda.synchronize()
a, b = ev(), ev()
a.record(st)
g, e = lq.lq_param_shift_grad(n, gates, theta, terms)
b.record(st); torch.cuda.synchronize()
ms = a.elapsed_time(b)
ncry = 4 * (n - 1)
ncirc = 2 * (p - ncry) + 4 * ncry + 1
emit({"row": "f3 CRY four-term PSR", "n": n, "params": p, "cry_params": ncry, "circuits": ncirc, "ms": ms,
      "gate_amp_updates_per_s": ncirc * len(gates) * 2 ** n / (ms / 1e3)})
