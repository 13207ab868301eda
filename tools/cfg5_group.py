"""Config-5 shape on ONE GPU in group mode (all G shards in this process,
device-copy exchanges): the 1000-gate config-5 circuit
(30 % on the m = log2 G top qubits) and the QFT at n = LQ_CFG5_N (30), each rep
from init_random (identity layout, as the bench step), timed with CUDA
events (median of 3 reps after a warm-up) for G = 1 (unsharded),
2, 4, 8 and exchange caps k = 1 (pairwise swaps) and 4 (all-to-all).
One JSON object per line."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2512_23183_b200 import lq  # noqa: E402


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def run(sv, w, reps=3):
    """reps of init_random -> circuit -> QFT from the identity layout (the
    bench step); medians of the circuit and QFT event times"""
    tc, tq = [], []
    for _ in range(reps):
        sv.init_random(w.seed)
        a = ev()
        sv.apply(w.gates)
        b = ev()
        sv.qft()
        c = ev()
        torch.cuda.synchronize()
        tc.append(a.elapsed_time(b))
        tq.append(b.elapsed_time(c))
    return statistics.median(tc), statistics.median(tq)


def main():
    n = int(os.environ.get("LQ_CFG5_N", 30))
    for G in (1, 2, 4, 8):
        m = G.bit_length() - 1
        w = W.config5(n, max(m, 1))
        for k in ((4,) if G == 1 else (1, 4)):
            lq.lq_set_option(lq.LQ_OPT_SWAP_QUBITS, k)
            sv = lq.StateVector(n) if G == 1 else lq.ShardedState(n, group_world=G)
            run(sv, w, 1)                      # warm-up: schedules, plans, JIT kernels
            ex0 = lq.lq_sv_exchange_stats(sv.h)
            t_circ, t_qft = run(sv, w)
            ex1 = lq.lq_sv_exchange_stats(sv.h)
            lq.lq_kernel_timing_reset()
            lq.lq_set_option(lq.LQ_OPT_KERNEL_TIMING, 1)
            sv.init_random(w.seed)
            sv.apply(w.gates)
            torch.cuda.synchronize()
            lq.lq_set_option(lq.LQ_OPT_KERNEL_TIMING, 0)
            swap_ms, swap_n = lq.lq_kernel_timing(lq.KC_SWAP)
            tile_ms, tile_n = lq.lq_kernel_timing(lq.KC_TILE)
            sched = lq.lq_dist_schedule_json(n, m, w.gates) if G > 1 else {"n_swaps": 0}
            qs = lq.lq_dist_schedule_json(n, m, [], qft=1) if G > 1 else {"n_swaps": 0}
            print(json.dumps({"n": n, "G": G, "swap_qubits_cap": k, "circuit_ms": t_circ, "qft_ms": t_qft,
                              "circuit_exchanges": sched["n_swaps"], "qft_exchanges": qs["n_swaps"],
                              "circuit_exchange_ms": swap_ms, "circuit_tile_ms": tile_ms,
                              "circuit_tile_passes": tile_n,
                              "bytes_sent_per_rank_step": (ex1[1] - ex0[1]) / 3}), flush=True)
            sv.free()
            del sv
            torch.cuda.empty_cache()
    lq.lq_set_option(lq.LQ_OPT_SWAP_QUBITS, 4)


if __name__ == "__main__":
    main()
