"""Same-box A/B of QFT(n) time (default n = 30) under environment variants
(AB_PRE_SWAP="q0-q1": apply that SWAP before each timed QFT -- a relabel of
the layout, so the QFT takes the permuted-layout path).

Each argument is a variant "name" or "name:VAR=val,VAR2=val"; every variant
runs in its own child process (plans read their experiment switches at plan
time), interleaved over AB_ROUNDS rounds.  Prints one JSON object per variant:
median / min ms, and a checksum of 4096 sampled amplitudes (variants that only
move data differently must agree bit for bit)."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import os, sys, json
sys.path.insert(0, %r)
import numpy as np, torch
from paper_2512_23183_b200 import lq
n = int(os.environ.get("AB_N", "30"))
if os.environ.get("AB_TILE_BITS"):   # LQ_OPT_TILE_BITS for this variant (0 = automatic)
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, int(os.environ["AB_TILE_BITS"]))
st = torch.cuda.current_stream()
sv = lq.StateVector(n, stream=st)
ts = []
for r in range(int(os.environ.get("AB_REPS", "5")) + 1):
    sv.init_random(7)
    if os.environ.get("AB_PRE_SWAP"):   # relabel the layout first (a folded SWAP): the generic QFT path
        q0, q1 = (int(x) for x in os.environ["AB_PRE_SWAP"].split("-"))
        sv.apply([("SWAP", q0, q1, -1, 0.0)])
    torch.cuda.synchronize()
    a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st); sv.qft(); c.record(st); torch.cuda.synchronize()
    if r: ts.append(a.elapsed_time(c))
idx = np.random.default_rng(1).choice(1 << n, 4096, replace=False)
v = sv.gather(idx)
print("AB", json.dumps({"ms": ts, "chk": [float(np.sum(v.real)), float(np.sum(v.imag))]}), flush=True)
""" % ROOT


def main():
    variants = []
    for a in sys.argv[1:]:
        name, _, envs = a.partition(":")
        env = dict(kv.split("=", 1) for kv in envs.split(",") if kv)
        variants.append((name, env))
    res = {name: [] for name, _ in variants}
    chk = {}
    for _ in range(int(os.environ.get("AB_ROUNDS", "2"))):
        for name, env in variants:
            r = subprocess.run([sys.executable, "-c", CHILD], capture_output=True, text=True,
                               env={**os.environ, **env}, timeout=900)
            line = [l for l in r.stdout.splitlines() if l.startswith("AB ")]
            if not line:
                print(json.dumps({"variant": name, "error": r.stderr[-800:]}), flush=True)
                continue
            d = json.loads(line[0][3:])
            res[name] += d["ms"]
            chk[name] = d["chk"]
    for name, env in variants:
        if res[name]:
            print(json.dumps({"variant": name, "env": env, "median_ms": statistics.median(res[name]),
                              "min_ms": min(res[name]), "chk": chk[name]}), flush=True)


if __name__ == "__main__":
    main()
