"""CPU emulator of liblq's distributed schedules (test infrastructure).

Executes the JSON schedule of ``lq_dist_schedule_json`` (dist.cpp) for one
rank: LOCAL steps run the rank's shard through ``plan_emulator.run`` with
the shard's global bits (gofs) in the logic index, SWAP steps trade the half
of the shard whose l-bit differs from the rank's g-bit with the partner
rank, through a caller-supplied ``exchange(send, peer) -> recv`` (in-process
lists, or torch.distributed gloo send/recv).  Shares no code with oracle/
or with the CUDA sources.
"""
from __future__ import annotations

import numpy as np

import plan_emulator as PE


def half_positions(nl: int, l: int, v: int) -> np.ndarray:
    """Local positions with bit l == v, in ascending order of the other bits."""
    i = np.arange(1 << (nl - 1), dtype=np.int64)
    lo = i & ((1 << l) - 1)
    return ((i ^ lo) << 1) | (v << l) | lo


def run_step(sched, st, psi, rank, theta=None, exchange=None):
    nl = sched["nl"]
    if st["kind"] == "local":
        gofs = (rank ^ st["xmask"]) << nl
        return PE.run(st["plan"], psi, theta, gofs=gofs)
    j = st["g"] - nl
    peer = rank ^ (1 << j)
    b = ((rank ^ st["xmask"]) >> j) & 1
    pos = half_positions(nl, st["l"], 1 - b)
    psi[pos] = exchange(psi[pos].copy(), peer)
    return 0.0


def logical_to_shard(sched, x):
    """Logical index -> (rank, local index) under the schedule's final layout."""
    n, nl = sched["n"], sched["nl"]
    phys = 0
    for q in range(n):
        if (x >> (n - 1 - q)) & 1:
            phys |= 1 << sched["qmap"][q]
    return (phys >> nl) ^ sched["xmask"], phys & ((1 << nl) - 1)


def assemble(sched, shards):
    """Logical-order full state from the final shards."""
    n = sched["n"]
    out = np.zeros(1 << n, np.complex128)
    for x in range(1 << n):
        r, li = logical_to_shard(sched, x)
        out[x] = shards[r][li]
    return out


def run_group(sched, psi_logical, theta=None):
    """All ranks in this process (the schedule starts in the identity layout,
    so physical index = logical index).  Returns (final logical state, E)."""
    nl, G = sched["nl"], 1 << sched["m"]
    shards = [psi_logical[r << nl:(r + 1) << nl].copy() for r in range(G)]
    E = 0.0
    for st in sched["steps"]:
        if st["kind"] == "local":
            for r in range(G):
                E += run_step(sched, st, shards[r], r, theta)
        else:
            outbox = {}
            for r in range(G):
                b = ((r ^ st["xmask"]) >> (st["g"] - nl)) & 1
                outbox[r] = shards[r][half_positions(nl, st["l"], 1 - b)].copy()
            for r in range(G):
                run_step(sched, st, shards[r], r, theta,
                         exchange=lambda send, peer: outbox[peer])
    return assemble(sched, shards), E
