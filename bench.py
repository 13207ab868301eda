#!/usr/bin/env python
"""bench.py -- one JSON line for the driver.

Workload (BASELINE.json configs[3], the largest single-GPU config; the
metric's "1/2/4/8 B200" scaling applies to it): n=24 XYZ-Heisenberg
parameter-shift gradient, RY/RZ + CNOT-ring ansatz of depth 10 (720 gates,
480 parameters), 93-term Pauli sum; one step = one full gradient = 961
circuits (960 shifted + the base circuit for E(theta)) from |0...0>.
With N GPUs the 961 circuits are sharded by parameter (p % N == rank) and
the gradient is summed with one NCCL all-reduce ("scaling": "strong": the
job is the configured gradient).

value  = gate-amplitude updates/s over all ranks: circuits x 720 x 2^24 /
         max-over-ranks device time (CUDA events on the launch stream),
         inputs (theta) already in HBM.
e2e    = the same metric through lq_param_shift_grad with HOST buffers
         (pinned theta in, gradient out), plan upload and copies included.
roofline = the dominant kernel (k_tile, the fused gate pass): algorithmic
         HBM bytes / its CUDA-event time inside the timed region.
cpu_baseline = the CPU oracle (oracle/, test infrastructure) on a bounded
         sample of the same workload, rank 0, N=1 only.

`--impl reference` times the oracle itself (this tier's reference arm).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "gate-amplitude updates/s & achieved HBM GB/s (frac. of peak) at 1/2/4/8 B200"
UNIT = "gate-amplitude updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def workload():
    import workloads as W
    w = W.config4()
    return w


def workload_config(w, extra=None):
    cfg = {"workload": "BASELINE configs[3]: n=24 XYZ Heisenberg open chain (Jx=1.0, Jy=0.7, Jz=0.4, "
                       "hz=0.3; 93 terms), RY/RZ + CNOT-ring ansatz depth 10 (720 gates, 480 params); "
                       "one step = full parameter-shift gradient (960 shifted + 1 base circuit)",
           "n_qubits": w.n, "gates_per_circuit": len(w.gates), "n_params": int(w.theta.size),
           "circuits_per_step": 2 * int(w.theta.size) + 1, "pauli_terms": len(w.terms),
           "l2": "no flush needed: each step streams >= 961 x 256 MiB states through HBM (> 126 MB L2)",
           "seed": "SeedSequence(251223183 + 4)"}
    if extra:
        cfg.update(extra)
    return cfg


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.proc = None
        self.dev = device_index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.dev)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per k_tile launch from the
    committed ncu --set full capture summary (profiles/), normalised per
    circuit-state in the launch."""
    p = os.path.join(ROOT, "profiles", "ncu_k_tile_summary.json")
    if not os.path.exists(p):
        return None
    try:
        d = json.load(open(p))
        return d
    except Exception:
        return None


def cpu_oracle_sample(w, n_gates):
    """The oracle (plain single-thread C) applying the first n_gates of the
    first shifted circuit (theta + pi/2 e_0) from |0...0> at n = 24."""
    import numpy as np
    import oracle
    th = w.theta.copy()
    th[0] += math.pi / 2
    psi = oracle.zeros(w.n)
    t0 = time.perf_counter()
    oracle.apply_circuit(psi, w.gates[:n_gates], th)
    dt = time.perf_counter() - t0
    return n_gates * (1 << w.n) / dt, dt


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    w = workload()
    n_gates = 72   # one ansatz layer per step (bounded sample, ~5 s of single-core work)
    for _ in range(args.warmup):
        cpu_oracle_sample(w, n_gates)
    rates, times = [], []
    for _ in range(args.steps):
        r, dt = cpu_oracle_sample(w, n_gates)
        rates.append(r)
        times.append(dt)
    tot_updates = args.steps * n_gates * (1 << w.n)
    value = tot_updates / sum(times)
    sample = (f"oracle (plain single-thread C, oracle/oracle.c) applying one ansatz layer "
              f"({n_gates} gates) of the first shifted circuit at n={w.n} per step")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(w, {"sample": sample}),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2512_23183_b200 import lq

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    w = workload()
    n, P = w.n, int(w.theta.size)
    stream = torch.cuda.current_stream()
    plan = lq.lq_psr_create(n, w.gates, P, w.terms, rank, world, stream)
    n_circ, _, plan_bytes, tile_passes = lq.lq_psr_stats(plan)
    total_circ = 2 * P + 1
    theta = torch.tensor(w.theta, dtype=torch.float64, device=dev)
    grad = torch.zeros(P, dtype=torch.float64, device=dev)
    energy = torch.zeros(1, dtype=torch.float64, device=dev)

    def step():
        lq.lq_psr_run(plan, theta.data_ptr(), grad.data_ptr(), energy.data_ptr())
        if world > 1:
            dist.all_reduce(grad)
            dist.all_reduce(energy)

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    g_check = grad.cpu().numpy().copy()

    def timed_region(instrumented):
        """K steps between a barrier + synchronize on both sides; with
        `instrumented`, every launch is bracketed by CUDA events on its
        stream (lq_kernel_timing) for the roofline -- that costs ~2 % of step
        time, so `value` comes from the plain region."""
        lq.lq_kernel_timing_reset()
        lq.lq_set_option(lq.LQ_OPT_KERNEL_TIMING, 1 if instrumented else 0)
        l0 = lq.lq_launch_count()
        clocks = ClockSampler(local)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clocks.start()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clk = clocks.stop()
        lq.lq_set_option(lq.LQ_OPT_KERNEL_TIMING, 0)
        return ev0.elapsed_time(ev1), lq.lq_launch_count() - l0, clk

    ms, launches, clk = timed_region(False)
    ms_inst, _, clk_inst = timed_region(True)
    tile_ms, tile_cnt = lq.lq_kernel_timing(lq.KC_TILE)
    pauli_ms, pauli_cnt = lq.lq_kernel_timing(lq.KC_PAULI)
    t = torch.tensor([ms, launches, tile_ms, tile_cnt, pauli_ms], dtype=torch.float64, device=dev)
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum)
        ms_max = float(tmax[0])
        launches_all = int(tsum[1])
    else:
        ms_max, launches_all = ms, launches
    updates_per_step = total_circ * len(w.gates) * (1 << n)
    value = updates_per_step * args.steps / (ms_max / 1e3)

    # roofline of the dominant kernel on this rank: algorithmic bytes / event time.
    # Each circuit streams the state through `tile_passes` tile passes: 16 B/amp
    # per load and per store; the first pass synthesises |0...0> (no load),
    # read-only and final passes skip the store (lq_psr_traffic, exact per plan).
    tile_bytes_circ, _other = lq.lq_psr_traffic(plan)
    alg_bytes = args.steps * n_circ * tile_bytes_circ
    peak, peak_src = peaks()
    achieved = alg_bytes / (tile_ms / 1e3) / 1e9 if tile_ms > 0 else None
    tr = ncu_traffic()
    traffic = None
    alg_per_launch = alg_bytes / max(tile_cnt, 1)
    if tr and tr.get("n_qubits") == n:
        # the capture's DRAM bytes per launch, rescaled by the ratio of
        # algorithmic bytes per launch (the capture may batch differently)
        traffic = tr["dram_bytes_per_launch"] * alg_per_launch / tr["algorithmic_bytes_per_launch"]
    roof = {"kernel": "k_tile (fused tile pass)", "bound": "hbm", "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "algorithmic_bytes_per_launch": alg_per_launch, "launches": int(tile_cnt),
            "avg_launch_ms": tile_ms / max(tile_cnt, 1), "peak_source": peak_src,
            "kernel_share_of_step": tile_ms / ms_inst if ms_inst > 0 else None,
            "pauli_share_of_step": pauli_ms / ms_inst if ms_inst > 0 else None,
            "timing": "separate instrumented region of the same K steps (per-launch CUDA events); "
                      f"its step time {ms_inst / args.steps:.1f} ms vs {ms / args.steps:.1f} ms uninstrumented",
            "clocks_instrumented_region": clk_inst,
            "traffic_source": (tr or {}).get("source")}

    # ---- e2e: host buffers through the public API ------------------------------------------
    e2e_steps = args.e2e_steps or max(1, min(args.steps, 3))
    th_pin = torch.tensor(w.theta, dtype=torch.float64).pin_memory()
    g_pin = torch.zeros(P, dtype=torch.float64).pin_memory()
    e_pin = torch.zeros(1, dtype=torch.float64).pin_memory()
    ga, ta = lq.GateArray(w.gates), lq.TermArray(w.terms)
    DP = ctypes.POINTER(ctypes.c_double)

    def e2e_step():
        st = lq._lib.lq_param_shift_grad(n, ga.ptr, ga.n, ctypes.cast(th_pin.data_ptr(), DP), P, ta.ptr, ta.n,
                                         rank, world, stream.cuda_stream, ctypes.cast(g_pin.data_ptr(), DP),
                                         ctypes.cast(e_pin.data_ptr(), DP))
        lq._chk(st)
        if world > 1:
            gd = g_pin.to(dev, non_blocking=True)
            dist.all_reduce(gd)
            g_pin.copy_(gd)
        return g_pin

    e2e_step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    dtt = torch.tensor([dt], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(dtt, op=dist.ReduceOp.MAX)
    dt = float(dtt[0])
    e2e_value = updates_per_step * e2e_steps / dt
    # theta in; the plan is built and uploaded once (lq_param_shift_grad's plan cache, warm-up call)
    h2d = 8 * P + (8 * P if world > 1 else 0)
    d2h = 8 * P + 8 + (8 * P if world > 1 else 0)
    g_e2e = g_pin.numpy().copy()
    if not np.allclose(g_e2e, g_check, rtol=0, atol=1e-12):
        raise RuntimeError("e2e gradient differs from the device-resident gradient")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_gates = 144
        rate, secs = cpu_oracle_sample(w, n_gates)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"oracle (single-thread C) applying the first {n_gates} gates (2 ansatz layers) "
                         f"of one shifted circuit at n={n}: {secs:.1f} s"}
    # support tracking: the first passes run only the tiles that
    # can be nonzero.  The counted updates stay nominal (every gate on all 2^n
    # amplitudes); this is the share of the plan's ops x
    # amplitudes that fall on provably-zero amplitudes and are not executed.
    ps = lq.lq_psr_pass_bytes(plan, with_support=True)
    N = 1 << n
    tot_ops = sum(o for _, _, _, o in ps) or 1
    zero_share = sum(o * (N - a) for _, _, a, o in ps) / (tot_ops * N)
    lq.lq_psr_free(plan)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": workload_config(w, {"parallelism": f"psr-shard{world}" if world > 1 else "single",
                                              "circuits_this_rank": int(n_circ),
                                              "tile_passes_per_circuit": int(tile_passes),
                                              "updates_counted": "nominal: gates x 2^n per circuit",
                                              "nominal_share_on_provably_zero_amplitudes": round(zero_share, 4)}),
                "roofline": roof, "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                        "d2h_bytes_per_step": int(d2h), "steps": e2e_steps},
                "gpu_launches": launches_all, "clocks": clk,
                "energy": float(energy.cpu()[0]), "grad_inf_norm": float(np.abs(g_check).max())}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
