"""Same-box A/B of config-4 gradient time under environment variants.

Each argument is a variant: "name" or "name:VAR=val,VAR2=val" (empty env =
the default build; AB_TILE_BITS / AB_COALESCE_BITS / AB_REG_BITS /
AB_PASS_BUDGET / AB_FIRST_PASS_FREE set the library options).  Every variant runs in its own child process (the
planner reads its experiment switches at plan time); variants are
interleaved over R rounds so clock drift hits all of them alike.
Prints one JSON object per variant: median / min gradient ms, passes, E."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import os, sys, json
sys.path.insert(0, %r)
import torch
import workloads as W
from paper_2512_23183_b200 import lq
for name in ("TILE_BITS", "COALESCE_BITS", "REG_BITS", "PASS_BUDGET", "FIRST_PASS_FREE", "RELABEL_STORES"):
    if os.environ.get("AB_" + name):
        lq.lq_set_option(getattr(lq, "LQ_OPT_" + name), int(os.environ["AB_" + name]))
w = W.config4()
npar = len(w.theta)
th = torch.tensor(w.theta, device="cuda"); g = torch.zeros(npar, dtype=torch.float64, device="cuda")
e = torch.zeros(1, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
P = lq.lq_psr_create(w.n, w.gates, npar, w.terms, stream=st)
lq.lq_psr_run(P, th.data_ptr(), g.data_ptr(), e.data_ptr()); torch.cuda.synchronize()
ts = []
for _ in range(int(os.environ.get("AB_REPS", "3"))):
    a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st); lq.lq_psr_run(P, th.data_ptr(), g.data_ptr(), e.data_ptr()); c.record(st); torch.cuda.synchronize()
    ts.append(a.elapsed_time(c))
print("AB", json.dumps({"ms": ts, "passes": lq.lq_psr_stats(P)[3], "E": e.item(), "g0": g[0].item()}), flush=True)
""" % ROOT


def main():
    variants = []
    for a in sys.argv[1:]:
        name, _, envs = a.partition(":")
        env = dict(kv.split("=", 1) for kv in envs.split(",") if kv)
        variants.append((name, env))
    rounds = int(os.environ.get("AB_ROUNDS", "2"))
    res = {name: [] for name, _ in variants}
    info = {}
    for _ in range(rounds):
        for name, env in variants:
            r = subprocess.run([sys.executable, "-c", CHILD], capture_output=True, text=True,
                               env={**os.environ, **env}, timeout=900)
            line = [l for l in r.stdout.splitlines() if l.startswith("AB ")]
            if not line:
                print(json.dumps({"variant": name, "error": r.stderr[-800:]}), flush=True)
                continue
            d = json.loads(line[0][3:])
            res[name] += d["ms"]
            info[name] = d
    for name, env in variants:
        if res[name]:
            print(json.dumps({"variant": name, "env": env, "median_ms": statistics.median(res[name]),
                              "min_ms": min(res[name]), "passes": info[name]["passes"], "E": info[name]["E"],
                              "g0": info[name]["g0"]}), flush=True)


if __name__ == "__main__":
    main()
