"""Same-box A/B of the QFT on a sharded state in group mode (all G shards in
one process) under environment variants, e.g. the balanced stage packing of
the local QFT runs against the greedy one (LQ_QFT_GREEDY=1).  Arguments as
tools/ab_qft.py ("name" or "name:VAR=val"); AB_N qubits, AB_G shards.  The
QFT starts from init_random in the identity layout; prints median / min ms
and a checksum of 4096 sampled amplitudes per variant."""
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
n, G = int(os.environ.get("AB_N", "31")), int(os.environ.get("AB_G", "2"))
sv = lq.ShardedState(n, group_world=G)
ts = []
for r in range(int(os.environ.get("AB_REPS", "4")) + 1):
    sv.init_random(7)
    torch.cuda.synchronize()
    a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); sv.qft(); c.record(); torch.cuda.synchronize()
    if r: ts.append(a.elapsed_time(c))
idx = np.random.default_rng(1).choice(1 << n, 4096, replace=False)
v = sv.gather(idx)
print("AB", json.dumps({"ms": ts, "chk": [float(np.sum(v.real)), float(np.sum(v.imag))]}), flush=True)
""" % ROOT


def main():
    variants = []
    for a in sys.argv[1:]:
        name, _, envs = a.partition(":")
        variants.append((name, dict(kv.split("=", 1) for kv in envs.split(",") if kv)))
    for name, env in variants:
        r = subprocess.run([sys.executable, "-c", CHILD], capture_output=True, text=True,
                           env={**os.environ, **env}, timeout=1200)
        line = [l for l in r.stdout.splitlines() if l.startswith("AB ")]
        if not line:
            print(json.dumps({"variant": name, "error": r.stderr[-800:]}), flush=True)
            continue
        d = json.loads(line[0][3:])
        print(json.dumps({"n": int(os.environ.get("AB_N", "31")), "G": int(os.environ.get("AB_G", "2")),
                          "variant": name, "env": env, "median_ms": statistics.median(d["ms"]),
                          "min_ms": min(d["ms"]), "chk": d["chk"]}), flush=True)


if __name__ == "__main__":
    main()
