"""CPU emulator of liblq's distributed schedules (test infrastructure).

Executes the JSON schedule of ``lq_dist_schedule_json`` (dist.cpp) for one
rank: LOCAL steps run the rank's shard through ``plan_emulator.run`` with
the shard's global bits (gofs) in the logic index, SWAP steps exchange k
global with k local bits: the rank sends every part of its shard whose
l-bits differ from its own g-bits to the rank whose g-bits they spell and
receives that rank's matching part into the same positions (k = 1: the
pairwise half-shard swap; k > 1: an all-to-all among 2^k ranks), through a
caller-supplied ``exchange(sends) -> recvs`` (in-process dicts, or
torch.distributed gloo send/recv).  Shares no code with oracle/
or with the CUDA sources.
"""
from __future__ import annotations

import numpy as np

import plan_emulator as PE


def part_positions(nl: int, ls, b: int) -> np.ndarray:
    """Local positions whose bits at ls (ascending) spell b (bit j <-> ls[j]),
    in ascending order of the other bits."""
    k = len(ls)
    pos = np.arange(1 << (nl - k), dtype=np.int64)
    for j, l in enumerate(ls):                 # deposit, lowest position first
        lo = pos & ((1 << l) - 1)
        pos = ((pos ^ lo) << 1) | (((b >> j) & 1) << l) | lo
    return pos


def swap_plan(sched, st, rank):
    """A k-qubit exchange from rank's side: [(peer, local positions)] for
    every part that leaves (part b goes to the rank whose g-bits are b and
    comes back from it into the same positions; part a = own g-bits stays)."""
    nl = sched["nl"]
    gs, ls = st["g"], st["l"]
    R = rank ^ st["xmask"]
    a = sum((((R >> (g - nl)) & 1) << j) for j, g in enumerate(gs))
    out = []
    for b in range(1 << len(gs)):
        if b == a:
            continue
        d = a ^ b
        peer = rank
        for j, g in enumerate(gs):
            if (d >> j) & 1:
                peer ^= 1 << (g - nl)
        out.append((peer, part_positions(nl, ls, b)))
    return out


def run_step(sched, st, psi, rank, theta=None, exchange=None):
    """exchange(sends: {peer: array}) -> {peer: array} (all of this rank's
    messages of one exchange step at once)."""
    nl = sched["nl"]
    if st["kind"] == "local":
        gofs = (rank ^ st["xmask"]) << nl
        return PE.run(st["plan"], psi, theta, gofs=gofs)
    plan = swap_plan(sched, st, rank)
    recv = exchange({peer: psi[pos].copy() for peer, pos in plan})
    for peer, pos in plan:
        psi[pos] = recv[peer]
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
            outbox = {r: {p: shards[r][pos].copy() for p, pos in swap_plan(sched, st, r)} for r in range(G)}
            for r in range(G):
                run_step(sched, st, shards[r], r, theta,
                         exchange=lambda sends, r=r: {p: outbox[p][r] for p in sends})
    return assemble(sched, shards), E
