"""Write the oracle-computed fixtures of the full-size parity tests.

Every value written here comes from ``oracle/`` (the plain C oracle, fp64,
Neumaier sums) on inputs drawn by ``workloads``; nothing comes from the CUDA
path.  The GPU tests (tests/test_gpu_fullsize.py) recompute the same quantities
through liblq and compare against these files, so the slow oracle runs happen
once here instead of on the GPU box.

  tests/golden/cfg4_oracle.json   configs[3] (n=24, 480 params): E(theta)
       and the 8 seeded components of
      ``W.config4().meta['oracle_params']`` by the parameter-shift rule
      (PAPER.md:374-377, 501-539): 17 circuits of 720 gates on 2^24 amplitudes.
  tests/golden/cfg5_twin_n{24,26}_m{1,2,3}.json   the config-5 generator at
      the reduced sizes n=24 and 26 with the configured m:
      init_random(seed), the 1000-gate circuit
      (reading A13), then the QFT (Alg. 3).  Stored: the
      amplitudes at 4096 seeded indices and three seeded full-state
      projections  P_r = sum_j w_r[j] * a_j  with w_r[j] = +-1 from
      ``twin_weights`` (a plain counter hash, no arithmetic of the method),
      so every amplitude enters the comparison.

Run:  python tools/make_golden.py [cfg4] [cfg5] [cfg5n26]   (about 5 min on 8 cores;
      the n = 26 twins about 8 min more)
"""
from __future__ import annotations

import json
import math
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import workloads as W  # noqa: E402
from twin_samples import TWIN_N, TWIN_NS, TWIN_SAMPLES, twin_indices, twin_weights  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def cfg4(threads: int):
    w = W.config4()
    sample = list(w.meta["oracle_params"])
    t0 = time.time()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        fe = ex.submit(oracle.energy, w.n, w.gates, w.theta, w.terms)
        fg = [ex.submit(oracle.param_shift_grad, w.n, w.gates, w.theta, w.terms, [p]) for p in sample]
        e = fe.result()
        g = [float(f.result()[0]) for f in fg]
    out = {
        "source": "tools/make_golden.py (oracle/oracle.c only)",
        "cite": "configs[3]: PAPER.md:733-734 (energy), PAPER.md:374-377 and 501-539 (parameter shift)",
        "workload": w.name, "n": w.n, "n_params": int(w.theta.size),
        "energy": e, "params": sample, "grad": g,
        "oracle_seconds": round(time.time() - t0, 1),
    }
    with open(os.path.join(GOLD, "cfg4_oracle.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("cfg4", out["energy"], out["grad"], out["oracle_seconds"], "s")


def twin(m: int, n: int = TWIN_N):
    w = W.config5(n=n, m=m)
    t0 = time.time()
    psi = oracle.init_random(n, w.seed)
    oracle.apply_circuit(psi, w.gates)
    oracle.qft(psi)
    idx = twin_indices(n, m)
    wts = twin_weights(n)
    proj = [complex(np.sum(wr * psi)) for wr in wts]   # library dot (plain sum), three projections
    out = {
        "source": "tools/make_golden.py (oracle/oracle.c only)",
        "cite": "SURVEY.md §8(c) c.4 (iv); init_random c.1 step 2; circuit reading A13; QFT PAPER.md:599-603",
        "workload": w.name, "n": n, "m": m, "seed": w.seed, "n_gates": len(w.gates),
        "norm2": oracle.norm2(psi),
        "idx": [int(i) for i in idx],
        "re": [float(v) for v in psi[idx].real], "im": [float(v) for v in psi[idx].imag],
        "proj_re": [p.real for p in proj], "proj_im": [p.imag for p in proj],
        "oracle_seconds": round(time.time() - t0, 1),
    }
    with open(os.path.join(GOLD, f"cfg5_twin_n{n}_m{m}.json"), "w") as f:
        json.dump(out, f)
    print("twin", m, out["norm2"], out["oracle_seconds"], "s")


def main():
    what = set(sys.argv[1:]) or {"cfg4", "cfg5"}
    threads = os.cpu_count() or 1
    with ThreadPoolExecutor(max_workers=4) as ex:
        futs = []
        if "cfg5" in what:
            futs += [ex.submit(twin, m) for m in (1, 2, 3)]
        if "cfg5n26" in what:
            futs += [ex.submit(twin, m, 26) for m in (1, 2, 3)]
        if "cfg4" in what:
            futs.append(ex.submit(cfg4, max(1, threads - 3)))
        for f in futs:
            f.result()


if __name__ == "__main__":
    main()
