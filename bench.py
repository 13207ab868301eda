#!/usr/bin/env python
"""bench.py -- one JSON line for the driver.

Default workload (--workload cfg4; BASELINE.json configs[3], the largest
single-GPU config; the metric's "1/2/4/8 B200" applies to it): n=24
XYZ-Heisenberg parameter-shift gradient, RY/RZ + CNOT-ring ansatz of depth 10
(720 gates, 480 parameters), 93-term Pauli sum; one step = one full gradient
= 961 circuits (960 shifted + the base circuit for E(theta)) from |0...0>.
With N GPUs the circuits are sharded by parameter (p % N == rank) and the
library all-reduces the gradient and E over NCCL inside lq_psr_run
("scaling": "strong": the job is the configured gradient).

--workload cfg5 (BASELINE.json configs[4], weak scaling): n = 33 + log2 N
(2^33 amplitudes = 128 GiB per GPU), init_random, the config-5 generator's
1000 gates (30 % on the m = max(1, log2 N) top qubits), then the full QFT;
N > 1 shards the state over the ranks (global-qubit exchanges over NCCL).

value  = gate-amplitude updates/s over all ranks: user-level gates x 2^n /
         max-over-ranks device time (CUDA events on the launch stream),
         inputs already in HBM.
e2e    = the same metric through the public C-ABI call with HOST buffers
         (cfg4: lq_param_shift_grad, pinned theta in, gradient out; cfg5:
         host gate list in, 2^16 sampled amplitudes out), copies included.
roofline = the dominant kernel (the fused tile pass): algorithmic HBM bytes /
         its CUDA-event time inside an instrumented copy of the timed region.
cpu_baseline = the CPU oracle (oracle/, test infrastructure) on a bounded
         sample of the same workload, rank 0, N=1 only: one core, and all
         host cores over independent circuits.

`--gpus N` without torchrun re-launches itself under torch.distributed.run
with N ranks; it fails (exit 2) if fewer than N GPUs are visible or if the
launcher's WORLD_SIZE differs from N.  `--impl reference` times the oracle
(this tier's reference arm).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "gate-amplitude updates/s & achieved HBM GB/s (frac. of peak) at 1/2/4/8 B200"
UNIT = "gate-amplitude updates/s"
NVLINK_GBS = 900.0   # NVLink 5 per direction per GPU (task statement)
PAPER_CONTEXT = {
    "note": "the paper reports no GPU or absolute gate throughput; its CPU-library speedups, quoted as context "
            "only (Intel Core i9-10980XE, 18 cores, PAPER.md:50)",
    "vqe": "VQE wall-clock 2-5x faster than Qiskit / PennyLane, 4-qubit H2 (PAPER.md:762)",
    "qft": "QFT 120-900x vs PennyLane / Qiskit, 6-22x vs Yao.jl; 0.72 us at n=1 (dense path) "
           "(PAPER.md:648, 670)",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=["cfg4", "cfg5"])
    ap.add_argument("--n", type=int, default=None, help="cfg5: override n (default 33 + log2 N)")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def die(msg):
    sys.stderr.write(f"bench.py: {msg}\n")
    sys.exit(2)


def launch_or_check(args):
    """--gpus N: re-exec under torchrun when no launcher set WORLD_SIZE;
    refuse a world size that differs from N."""
    if args.gpus < 1 or (args.gpus & (args.gpus - 1)):
        die(f"--gpus must be a power of two >= 1, got {args.gpus}")
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            die(f"launched with WORLD_SIZE={world} but --gpus {args.gpus}")
        return
    if args.gpus == 1:
        return
    if args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            die(f"--gpus {args.gpus} needs {args.gpus} visible GPUs, this box has {have}")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


# ------------------------------------------------------------------ workloads
def cfg4_workload():
    import workloads as W
    return W.config4()


def cfg4_config(w, extra=None):
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


def cfg5_shape(args, world):
    m_sh = world.bit_length() - 1            # log2 of the ranks the state is sharded over
    n = args.n if args.n else 33 + m_sh
    m_gen = max(1, m_sh)                     # the generator's "global" qubits (reading A13)
    return n, m_sh, m_gen


def cfg5_config(n, m_sh, m_gen, n_gates, qft_gates, extra=None):
    cfg = {"workload": f"BASELINE configs[4] (weak scaling): n={n} = 33 + log2 N, init_random, {n_gates} gates "
                       f"from the config-5 generator (30 % on the top m={m_gen} qubits), then the full QFT "
                       f"({qft_gates} Alg. 3 gates); one step = init + circuit + QFT",
           "n_qubits": n, "state_bytes_per_gpu": 16 << (n - m_sh), "sharded_over": 1 << m_sh,
           "gates_per_step": n_gates + qft_gates,
           "l2": "no flush needed: a 2^33-amplitude shard (128 GiB) per GPU streams through HBM every pass",
           "seed": "SeedSequence(251223183 + 5)"}
    if extra:
        cfg.update(extra)
    return cfg


# ------------------------------------------------------------------ measurement helpers
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
    """dram__bytes_read.sum + dram__bytes_write.sum per tile-pass launch from
    the committed ncu --set full capture summary (profiles/)."""
    p = os.path.join(ROOT, "profiles", "ncu_k_tile_summary.json")
    if not os.path.exists(p):
        return None
    try:
        return json.load(open(p))
    except Exception:
        return None


def host_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count() or 1


def oracle_gate_sample(n, gates, theta, n_threads=1):
    """The oracle (plain single-thread C) applying `gates` from |0...0> at n
    qubits, on n_threads independent circuits at once (one state each; the
    oracle releases the GIL): returns (aggregate updates/s, wall seconds)."""
    import oracle
    states = [oracle.zeros(n) for _ in range(n_threads)]
    t0 = time.perf_counter()
    if n_threads == 1:
        oracle.apply_circuit(states[0], gates, theta)
    else:
        ts = [threading.Thread(target=oracle.apply_circuit, args=(s, gates, theta)) for s in states]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    dt = time.perf_counter() - t0
    return n_threads * len(gates) * (1 << n) / dt, dt


def cfg4_oracle_sample(w, n_gates, n_threads=1):
    """first n_gates of the first shifted circuit (theta + pi/2 e_0) at n=24"""
    th = w.theta.copy()
    th[0] += math.pi / 2
    return oracle_gate_sample(w.n, w.gates[:n_gates], th, n_threads)


def cpu_baseline_block(sample_fn, desc_1, desc_all):
    model, ncpu = host_info()
    r1, s1 = sample_fn(1)
    threads = max(1, min(ncpu, 32))
    out = {"value": r1, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": f"{desc_1}: {s1:.1f} s",
           "cpu_model": model, "os_cpu_count": ncpu}
    if threads > 1:
        ra, sa = sample_fn(threads)
        out["all_core"] = {"value": ra, "unit": UNIT, "cores": threads,
                           "sample": f"{desc_all} on {threads} threads (one independent circuit each): {sa:.1f} s"}
    return out


# ------------------------------------------------------------------ reference arm (the oracle)
def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    model, ncpu = host_info()
    if args.workload == "cfg4":
        w = cfg4_workload()
        n_gates = 72   # one ansatz layer per step (bounded sample, ~5 s of single-core work)
        fn = lambda: cfg4_oracle_sample(w, n_gates)   # noqa: E731
        sample = (f"oracle (plain single-thread C, oracle/oracle.c) applying one ansatz layer "
                  f"({n_gates} gates) of the first shifted circuit at n={w.n} per step")
        cfg = cfg4_config(w, {"sample": sample})
        scaling = "strong"
    else:
        import workloads as W
        n, m_sh, m_gen = cfg5_shape(args, world)
        tw = W.config5(n=24, m=m_gen)
        n_gates = 60
        fn = lambda: oracle_gate_sample(24, tw.gates[:n_gates], None)   # noqa: E731
        sample = (f"oracle (plain single-thread C) applying the first {n_gates} gates of the config-5 generator "
                  f"(m={m_gen}) to a 2^24-amplitude state per step (the n={n} state does not fit host memory)")
        cfg = cfg5_config(n, m_sh, m_gen, 1000, W.qft_gate_count(n), {"sample": sample})
        scaling = "weak"
    for _ in range(args.warmup):
        fn()
    rates, times = [], []
    for _ in range(args.steps):
        r, dt = fn()
        rates.append(r)
        times.append(dt)
    value = statistics.mean(rates)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / args.steps,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             "cpu_model": model, "os_cpu_count": ncpu},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def timed(args, world, local, stream, step, lq):
    """K steps between a barrier + synchronize on both sides; returns
    (plain ms, instrumented ms, launches, clocks, per-class event timings).
    The instrumented copy brackets every launch with CUDA events on its
    stream (the roofline's per-launch time; ~2 % overhead), so `value`
    comes from the plain region."""
    import torch
    import torch.distributed as dist

    def region(instrumented):
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

    ms, launches, clk = region(False)
    ms_inst, _, clk_inst = region(True)
    cls = {k: lq.lq_kernel_timing(getattr(lq, k)) for k in ("KC_TILE", "KC_PAULI", "KC_SWAP")}
    return ms, ms_inst, launches, clk, clk_inst, cls


def reduce_max_sum(vals, world, dev):
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    if world == 1:
        return t.tolist(), t.tolist()
    tmax, tsum = t.clone(), t.clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(tsum)
    return tmax.tolist(), tsum.tolist()


def run_cfg4(args, lq, rank, local, world, dev, comm):
    import numpy as np
    import torch
    import torch.distributed as dist
    w = cfg4_workload()
    n, P = w.n, int(w.theta.size)
    stream = torch.cuda.current_stream()
    plan = lq.lq_psr_create(n, w.gates, P, w.terms, comm=comm, stream=stream)
    n_circ, _, plan_bytes, tile_passes = lq.lq_psr_stats(plan)
    total_circ = 2 * P + 1
    theta = torch.tensor(w.theta, dtype=torch.float64, device=dev)
    grad = torch.zeros(P, dtype=torch.float64, device=dev)
    energy = torch.zeros(1, dtype=torch.float64, device=dev)

    def step():   # one full gradient; with N ranks the all-reduce runs inside lq_psr_run
        lq.lq_psr_run(plan, theta.data_ptr(), grad.data_ptr(), energy.data_ptr())

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    g_check = grad.cpu().numpy().copy()
    ms, ms_inst, launches, clk, clk_inst, cls = timed(args, world, local, stream, step, lq)
    tile_ms, tile_cnt = cls["KC_TILE"]
    pauli_ms, _ = cls["KC_PAULI"]
    mx, sm = reduce_max_sum([ms, launches], world, dev)
    ms_max, launches_all = mx[0], int(sm[1])
    updates_per_step = total_circ * len(w.gates) * (1 << n)
    value = updates_per_step * args.steps / (ms_max / 1e3)

    # roofline of the dominant kernel on this rank: algorithmic bytes / event time.
    tile_bytes_circ, _other = lq.lq_psr_traffic(plan)
    alg_bytes = args.steps * n_circ * tile_bytes_circ
    peak, peak_src = peaks()
    achieved = alg_bytes / (tile_ms / 1e3) / 1e9 if tile_ms > 0 else None
    tr = ncu_traffic()
    traffic = None
    alg_per_launch = alg_bytes / max(tile_cnt, 1)
    if tr and tr.get("n_qubits") == n:
        traffic = tr["dram_bytes_per_launch"] * alg_per_launch / tr["algorithmic_bytes_per_launch"]
    roof = {"kernel": "lqj tile pass (fused gates + Pauli groups)", "bound": "hbm", "achieved": achieved,
            "peak": peak, "unit": "GB/s", "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "algorithmic_bytes_per_launch": alg_per_launch, "launches": int(tile_cnt),
            "avg_launch_ms": tile_ms / max(tile_cnt, 1), "peak_source": peak_src,
            "frac_of_nominal_8tbs": (achieved / 8000.0) if achieved else None,
            "kernel_share_of_step": tile_ms / ms_inst if ms_inst > 0 else None,
            "pauli_share_of_step": pauli_ms / ms_inst if ms_inst > 0 else None,
            "timing": "separate instrumented region of the same K steps (per-launch CUDA events); "
                      f"its step time {ms_inst / args.steps:.1f} ms vs {ms / args.steps:.1f} ms uninstrumented",
            "clocks_instrumented_region": clk_inst,
            "traffic_source": (tr or {}).get("source")}

    # access-pattern ceiling: each pass's tile set swept without arithmetic
    # (lq_tile_sweep) over one launch's circuits; a pass that moves fewer
    # bytes (support tracking, read-only) is scaled by its byte fraction
    masks = lq.lq_psr_pass_tiles(plan)
    pbytes = lq.lq_psr_pass_bytes(plan)
    batches = tile_cnt / max(1, args.steps * tile_passes)
    B = max(1, round(n_circ / batches)) if batches else 1
    nb = n + max(0, (B - 1).bit_length())
    buf = torch.empty(1 << nb, dtype=torch.complex128, device=dev)
    sweep_cache, ceil_ms_batch = {}, 0.0
    for m, (kind, byts) in zip(masks, pbytes):
        if kind != 0 or m == 0:
            continue
        if m not in sweep_cache:
            sweep_cache[m] = lq.lq_tile_sweep(buf.data_ptr(), buf.numel() * 16, nb, m, 3, stream)
        ceil_ms_batch += sweep_cache[m] * byts / (32.0 * (1 << n))
    del buf
    torch.cuda.empty_cache()
    ceil_ms_step = ceil_ms_batch * batches
    roof["access_pattern_ceiling"] = {
        "tile_ms_per_step": ceil_ms_step, "tile_ms_per_step_measured": tile_ms / args.steps,
        "frac": ceil_ms_step / (tile_ms / args.steps) if tile_ms > 0 else None,
        "ceiling_GBps": (alg_bytes / args.steps) / (ceil_ms_step / 1e3) / 1e9 if ceil_ms_step else None,
        "source": "lq_tile_sweep: each pass's tile bit set swept in place (16 B read + 16 B write per amplitude, "
                  "no arithmetic) over one launch's circuits, x its algorithmic byte fraction; HBM3e serves "
                  "128-byte runs at large strides below the copy rate (DESIGN.md §5)"}

    # ---- e2e: host buffers through the public API (collective with N ranks) -----------------
    e2e_steps = args.e2e_steps or max(1, min(args.steps, 3))
    th_pin = torch.tensor(w.theta, dtype=torch.float64).pin_memory()
    g_pin = torch.zeros(P, dtype=torch.float64).pin_memory()
    e_pin = torch.zeros(1, dtype=torch.float64).pin_memory()
    ga, ta = lq.GateArray(w.gates), lq.TermArray(w.terms)
    DP = ctypes.POINTER(ctypes.c_double)

    def e2e_step():
        lq._chk(lq._lib.lq_param_shift_grad(n, ga.ptr, ga.n, ctypes.cast(th_pin.data_ptr(), DP), P, ta.ptr, ta.n,
                                            comm, stream.cuda_stream, ctypes.cast(g_pin.data_ptr(), DP),
                                            ctypes.cast(e_pin.data_ptr(), DP)))

    e2e_step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    dt = reduce_max_sum([time.perf_counter() - t0], world, dev)[0][0]
    e2e_value = updates_per_step * e2e_steps / dt
    h2d = 8 * P                 # theta in (the plan is built and uploaded once: the warm-up call)
    d2h = 8 * P + 8             # gradient + E out
    g_e2e = g_pin.numpy().copy()
    if not np.array_equal(g_e2e, g_check):
        raise RuntimeError("e2e gradient differs from the device-resident gradient")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_gates = 144
        cpu = cpu_baseline_block(lambda t: cfg4_oracle_sample(w, n_gates if t == 1 else 72, t),
                                 f"oracle (single-thread C) applying the first {n_gates} gates (2 ansatz layers) "
                                 f"of one shifted circuit at n={n}",
                                 "the same oracle applying one ansatz layer (72 gates)")
    # support tracking: counted updates stay nominal (every gate
    # on all 2^n amplitudes); this is the share of the plan's ops
    # x amplitudes that fall on provably-zero amplitudes and are not executed.
    ps = lq.lq_psr_pass_bytes(plan, with_support=True)
    N = 1 << n
    tot_ops = sum(o for _, _, _, o in ps) or 1
    zero_share = sum(o * (N - a) for _, _, a, o in ps) / (tot_ops * N)
    lq.lq_psr_free(plan)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "executed_value": value * (1.0 - zero_share),
                "executed_value_note": "value x (1 - nominal_share_on_provably_zero_amplitudes): the updates "
                                       "that actually execute (support tracking skips provably-zero amplitudes)",
                "config": cfg4_config(w, {"parallelism": f"psr-shard{world} + NCCL all-reduce in lq_psr_run"
                                          if world > 1 else "single",
                                          "circuits_this_rank": int(n_circ),
                                          "tile_passes_per_circuit": int(tile_passes),
                                          "updates_counted": "nominal: gates x 2^n per circuit",
                                          "nominal_share_on_provably_zero_amplitudes": round(zero_share, 4)}),
                "roofline": roof, "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                        "d2h_bytes_per_step": int(d2h), "steps": e2e_steps, "api": "lq_param_shift_grad"},
                "gpu_launches": launches_all, "clocks": clk, "paper_context": PAPER_CONTEXT,
                "energy": float(energy.cpu()[0]), "grad_inf_norm": float(np.abs(g_check).max())}
        print(json.dumps(line), flush=True)


def run_cfg5(args, lq, rank, local, world, dev, comm):
    import numpy as np
    import torch
    import workloads as W
    n, m_sh, m_gen = cfg5_shape(args, world)
    w = W.config5(n=n, m=m_gen)
    qg = W.qft_gate_count(n)
    stream = torch.cuda.current_stream()
    if world > 1:
        sv = lq.ShardedState(n, comm=comm, stream=stream)
    else:
        sv = lq.StateVector(n, stream=stream)
    ga = lq.GateArray(w.gates)

    def step():
        sv.init_random(w.seed)
        sv.apply(ga)
        sv.qft()

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    ex0 = lq.lq_sv_exchange_stats(sv.h)
    ms, ms_inst, launches, clk, clk_inst, cls = timed(args, world, local, stream, step, lq)
    ex1 = lq.lq_sv_exchange_stats(sv.h)
    tile_ms, tile_cnt = cls["KC_TILE"]
    swap_ms, swap_cnt = cls["KC_SWAP"]
    mx, sm = reduce_max_sum([ms, launches, swap_ms], world, dev)
    ms_max, launches_all, swap_ms_max = mx[0], int(sm[1]), mx[2]
    updates_per_step = (len(w.gates) + qg) * (1 << n)
    value = updates_per_step * args.steps / (ms_max / 1e3)
    nloc = 1 << (n - m_sh)
    # tile passes of circuit and QFT plans read and write every local
    # amplitude once: 32 B per amplitude per launch
    alg_per_launch = 32 * nloc
    peak, peak_src = peaks()
    achieved = alg_per_launch * tile_cnt / (tile_ms / 1e3) / 1e9 if tile_ms > 0 else None
    roof = {"kernel": "lqj tile pass (fused gates / QFT butterflies)", "bound": "hbm", "achieved": achieved,
            "peak": peak, "unit": "GB/s", "frac": (achieved / peak) if achieved else None, "traffic": None,
            "algorithmic_bytes_per_launch": alg_per_launch, "launches": int(tile_cnt),
            "avg_launch_ms": tile_ms / max(tile_cnt, 1), "peak_source": peak_src,
            "frac_of_nominal_8tbs": (achieved / 8000.0) if achieved else None,
            "kernel_share_of_step": tile_ms / ms_inst if ms_inst > 0 else None,
            "clocks_instrumented_region": clk_inst,
            "note": "single-state plans take the 800 FP64 pass budget (LQ_OPT_STATE_PASS_BUDGET): fewer, "
                    "arithmetic-heavier passes; the update rate rises (1.84 -> 1.65 s per step at n=33) while "
                    "the pass's HBM fraction falls (0.72 -> 0.51), DESIGN.md §5"}
    exchanges = (ex1[0] - ex0[0]) // 2          # two timed regions
    sent = (ex1[1] - ex0[1]) // 2
    nvl = None
    if world > 1:
        nvl = {"exchanges_per_step": exchanges / args.steps, "bytes_sent_per_rank_per_step": sent / args.steps,
               "exchange_ms_per_step": swap_ms_max / args.steps,
               "achieved_gbs": (sent / args.steps) / (swap_ms_max / args.steps / 1e3) / 1e9 if swap_ms_max else None,
               "peak_gbs": NVLINK_GBS, "unit": "GB/s (bytes sent per GPU / exchange time, pack + unpack included)"}
        if nvl["achieved_gbs"]:
            nvl["frac"] = nvl["achieved_gbs"] / NVLINK_GBS

    # e2e: host gate list in, sampled amplitudes out, through the public API
    e2e_steps = args.e2e_steps or 1
    idx = np.unique(np.random.default_rng(5).integers(0, 1 << n, size=1 << 16, dtype=np.uint64))

    def e2e_step():
        sv.init_random(w.seed)
        sv.apply(w.gates)
        sv.qft()
        return sv.gather(idx)

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        amps = e2e_step()
    torch.cuda.synchronize()
    dt = reduce_max_sum([time.perf_counter() - t0], world, dev)[0][0]
    e2e_value = updates_per_step * e2e_steps / dt
    norm = sv.norm2()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        tw = W.config5(n=24, m=m_gen)
        cpu = cpu_baseline_block(lambda t: oracle_gate_sample(24, tw.gates[:60 if t == 1 else 30], None, t),
                                 f"oracle (single-thread C) applying the first 60 config-5 gates (m={m_gen}) to a "
                                 "2^24-amplitude state (the 2^33 state exceeds host memory)",
                                 "the same oracle applying 30 gates")
    sv.free()
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": cfg5_config(n, m_sh, m_gen, len(w.gates), qg,
                                      {"parallelism": f"state sharded on {m_sh} global qubits over NCCL"
                                       if world > 1 else "single"}),
                "roofline": roof, "nvlink": nvl, "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(ga.n * 40 + idx.size * 8),
                        "d2h_bytes_per_step": int(idx.size * 16), "steps": e2e_steps,
                        "api": "lq_sv_init_random + lq_apply_circuit + lq_qft + lq_sv_gather"},
                "gpu_launches": launches_all, "clocks": clk, "paper_context": PAPER_CONTEXT,
                "norm2": norm, "sample_abs_max": float(np.abs(amps).max())}
        print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2512_23183_b200 import lq

    rank, local, world = dist_env()
    if not torch.cuda.is_available():
        die("no CUDA device: liblq has no CPU path")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        comm = lq.comm_from_torch()
    try:
        (run_cfg4 if args.workload == "cfg4" else run_cfg5)(args, lq, rank, local, world, dev, comm)
    finally:
        if comm is not None:
            lq.lq_psr_cache_clear()
            lq.lq_comm_free(comm)
        if world > 1:
            dist.destroy_process_group()


def main():
    args = parse()
    launch_or_check(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
