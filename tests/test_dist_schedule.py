"""Distributed (sharded-state) host logic on CPU: the schedules of dist.cpp
executed by a per-rank emulator -- in one process over G shards, and over
two processes with torch.distributed gloo (global/local
classification, rank relabels, Belady swaps, expectation on shards) --
against the CPU oracle.  No GPU involved."""
import os
import socket

import numpy as np
import pytest

import dist_emulator as DE
import workloads as W
from test_gpu_parity import rich_circuit


@pytest.fixture(scope="module")
def lq():
    from paper_2512_23183_b200 import lq as _lq
    return _lq


TOL = 1e-12


@pytest.mark.parametrize("n,m", [(6, 1), (8, 2), (9, 3)])
def test_group_rich_circuit(lq, oracle, n, m):
    rng = np.random.default_rng(40 + n)
    gates = [g for g in rich_circuit(n, 80, rng)]
    sched = lq.lq_dist_schedule_json(n, m, gates)
    psi0 = oracle.init_random(n, 11 + n)
    got, _ = DE.run_group(sched, psi0.copy())
    ref = oracle.init_random(n, 11 + n)
    oracle.apply_circuit(ref, gates)
    assert np.abs(got - ref).max() <= TOL
    assert sched["n_swaps"] > 0


@pytest.mark.parametrize("m", [1, 2])
def test_group_config5_twin_with_qft(lq, oracle, m):
    """The config-5 generator (30 % of gates on global qubits) + full QFT."""
    n = 10
    w = W.config5(n, m, 200)
    for qft in (1, -1):
        sched = lq.lq_dist_schedule_json(n, m, w.gates, qft=qft)
        psi0 = oracle.init_random(n, w.seed)
        got, _ = DE.run_group(sched, psi0.copy())
        ref = oracle.init_random(n, w.seed)
        oracle.apply_circuit(ref, w.gates)
        oracle.qft(ref, inverse=qft < 0)
        assert np.abs(got - ref).max() <= TOL


def test_expval_rejects_too_wide_x(lq):
    from paper_2512_23183_b200.lq import LQError
    with pytest.raises(LQError):
        lq.lq_dist_schedule_json(4, 2, [], terms=[(1.0, 0b111, 0)])


def test_global_x_and_y_are_relabels(lq, oracle):
    n, m = 6, 2
    gates = [("H", 3, -1, -1, 0.0), ("X", 0, -1, -1, 0.0), ("Y", 1, -1, -1, 0.0), ("CNOT", 0, 4, -1, 0.0),
             ("RZ", 1, -1, -1, 0.7), ("CZ", 0, 1, -1, 0.0), ("X", 1, -1, -1, 0.0)]
    sched = lq.lq_dist_schedule_json(n, m, gates)
    assert sched["n_relabels"] == 3 and sched["n_swaps"] == 0 and sched["xmask"] != 0
    psi0 = oracle.init_random(n, 5)
    got, _ = DE.run_group(sched, psi0.copy())
    ref = oracle.init_random(n, 5)
    oracle.apply_circuit(ref, gates)
    assert np.abs(got - ref).max() <= TOL


def test_group_expval(lq, oracle):
    n, m = 9, 2
    rng = np.random.default_rng(8)
    gates = rich_circuit(n, 40, rng)
    # a term may act with X/Y on at most n - m qubits (a shard's worth: its
    # pairs (j, j ^ x) must fit on one rank after swaps)
    terms = [t for t in W.random_pauli_sum(n, 40, rng) if bin(t[1]).count("1") <= n - m][:25]
    assert any(t[1] & ((1 << m) - 1) for t in terms)   # some X/Y on global qubits (q < m)
    sched = lq.lq_dist_schedule_json(n, m, gates, terms=terms)
    psi0 = oracle.init_random(n, 21)
    _, E = DE.run_group(sched, psi0.copy())
    ref = oracle.init_random(n, 21)
    oracle.apply_circuit(ref, gates)
    eo = oracle.expval(ref, terms)
    assert abs(E - eo) <= 1e-10 * max(1.0, abs(eo))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, n, m, seed, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2512_23183_b200 import lq
    w = W.config5(n, m, 150)
    terms = W.xyz_terms(n)
    sched = lq.lq_dist_schedule_json(n, m, w.gates, qft=1, terms=terms)
    nl = sched["nl"]
    psi = oracle.init_random(n, w.seed)[rank << nl:(rank + 1) << nl].copy()

    def exchange(sends):
        reqs, recvs = [], {}
        for peer, send in sorted(sends.items()):
            t_send = torch.from_numpy(send.view(np.float64).copy())
            t_recv = torch.empty_like(t_send)
            reqs += [dist.isend(t_send, peer), dist.irecv(t_recv, peer)]
            recvs[peer] = t_recv
        for r in reqs:
            r.wait()
        return {p: t.numpy().view(np.complex128) for p, t in recvs.items()}

    E = 0.0
    for st in sched["steps"]:
        E += DE.run_step(sched, st, psi, rank, exchange=exchange)
    e = torch.tensor([E], dtype=torch.float64)
    dist.all_reduce(e)
    shards = [torch.empty(2 << nl, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(shards, torch.from_numpy(psi.view(np.float64).copy()))
    if rank == 0:
        full = DE.assemble(sched, [s.numpy().view(np.complex128) for s in shards])
        q.put((full, float(e[0])))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_ranks_config5_twin_qft_expval(oracle, world):
    """world_size 2 and 4 over gloo: each process runs its shard; exchanges
    are real point-to-point messages (world 4: 2-qubit all-to-alls among the
    4 ranks); the energy is an all-reduce."""
    import torch.multiprocessing as mp
    n, m = 9, world.bit_length() - 1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, n, m, 0, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, E = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = W.config5(n, m, 150)
    ref = oracle.init_random(n, w.seed)
    oracle.apply_circuit(ref, w.gates)
    oracle.qft(ref)
    assert np.abs(full - ref).max() <= TOL
    if world == 4:
        from paper_2512_23183_b200 import lq
        sched = lq.lq_dist_schedule_json(n, m, w.gates, qft=1)
        assert any(len(st["g"]) == 2 for st in sched["steps"] if st["kind"] == "swap")
    eo = oracle.expval(ref, W.xyz_terms(n))
    assert abs(E - eo) <= 1e-10 * max(1.0, abs(eo))


@pytest.mark.parametrize("K", [4, 6])
def test_group_small_tiles_single_op_passes(lq, oracle, K):
    """Tiles much smaller than a shard: LOCAL steps with a lone QFT stage or
    gate must become tile passes (k_pair runs only 1q/2q matrix gates)."""
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, K)
    try:
        n, m = 11, 2
        w = W.config5(n, m, 120)
        sched = lq.lq_dist_schedule_json(n, m, w.gates, qft=1)
        kinds = {p["kind"] for s in sched["steps"] if s["kind"] == "local" for p in s["plan"]["passes"]}
        psi0 = oracle.init_random(n, w.seed)
        got, _ = DE.run_group(sched, psi0.copy())
    finally:
        lq.lq_set_option(lq.LQ_OPT_TILE_BITS, 0)
    ref = oracle.init_random(n, w.seed)
    oracle.apply_circuit(ref, w.gates)
    oracle.qft(ref)
    assert np.abs(got - ref).max() <= TOL
    assert 0 in kinds


@pytest.mark.parametrize("n,m", [(4, 1), (5, 2), (6, 3), (7, 4)])
def test_minimal_shards_every_gate_qft_expval(lq, oracle, n, m):
    """Shards of 3 qubits (the minimum: a Toffoli's three qubits must fit):
    every gate kind, QFT and a Pauli sum."""
    rng = np.random.default_rng(n)
    gates = rich_circuit(n, 40, rng)
    terms = [t for t in W.random_pauli_sum(n, 8, rng) if bin(t[1]).count("1") <= n - m]
    sched = lq.lq_dist_schedule_json(n, m, gates, qft=1, terms=terms)
    got, E = DE.run_group(sched, oracle.init_random(n, 3))
    ref = oracle.init_random(n, 3)
    oracle.apply_circuit(ref, gates)
    oracle.qft(ref)
    assert np.abs(got - ref).max() <= TOL
    eo = oracle.expval(ref, terms)
    assert abs(E - eo) <= 1e-10 * max(1.0, abs(eo))


def test_shards_smaller_than_three_qubits_rejected(lq):
    from paper_2512_23183_b200.lq import LQError
    for n, m in [(3, 1), (4, 2), (2, 1)]:
        with pytest.raises(LQError):
            lq.lq_dist_schedule_json(n, m, [])


@pytest.mark.parametrize("k", [1, 2, 3])
def test_exchange_group_size_option(lq, oracle, k):
    """LQ_OPT_SWAP_QUBITS caps the qubits per exchange (1 = pairwise swaps);
    every cap gives the same state, and the distributed QFT on 2^3 ranks
    needs exactly two 3-qubit all-to-alls when the cap allows them (SURVEY
    §8(e): stages 0..m-1, then n-m..n-1; the SWAP layer is a relabel)."""
    n, m = 10, 3
    w = W.config5(n, m, 200)
    lq.lq_set_option(lq.LQ_OPT_SWAP_QUBITS, k)
    try:
        sched = lq.lq_dist_schedule_json(n, m, w.gates, qft=1)
        qft_only = lq.lq_dist_schedule_json(n, m, [], qft=1)
    finally:
        lq.lq_set_option(lq.LQ_OPT_SWAP_QUBITS, 4)
    assert all(len(st["g"]) <= k for st in sched["steps"] if st["kind"] == "swap")
    if k == 3:
        sw = [st for st in qft_only["steps"] if st["kind"] == "swap"]
        assert len(sw) == 2 and all(len(st["g"]) == 3 for st in sw)
        assert abs(qft_only["shard_fraction_sent"] - 2 * 7 / 8) < 1e-12
    # exchanges avoid the coalescing bits 0..2 when they can
    assert all(min(st["l"]) >= 3 for st in sched["steps"] if st["kind"] == "swap")
    got, _ = DE.run_group(sched, oracle.init_random(n, w.seed))
    ref = oracle.init_random(n, w.seed)
    oracle.apply_circuit(ref, w.gates)
    oracle.qft(ref)
    assert np.abs(got - ref).max() <= TOL


def test_comm_local_partition_handles(lq):
    """lq_comm_init_local: rank/world without transport (no device needed)."""
    c = lq.lq_comm_init_local(2, 4)
    assert lq.lq_comm_info(c) == (2, 4, False)
    lq.lq_comm_free(c)
    from paper_2512_23183_b200.lq import LQError
    with pytest.raises(LQError):
        lq.lq_comm_init_local(4, 4)


def test_bench_refuses_more_gpus_than_visible():
    """bench.py --gpus 2 on a box with fewer GPUs fails loudly (exit 2)
    instead of measuring one rank and reporting n_gpus: 1."""
    import subprocess
    import sys
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("this box has >= 2 GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2 and "visible GPUs" in r.stderr
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env={**env, "WORLD_SIZE": "1", "RANK": "0"}, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr


@pytest.mark.parametrize("m", [1, 2, 3])
def test_sharded_qft_schedule_is_pass_aligned(lq, m):
    """The distributed QFT at n = 30 on 2^m ranks (host schedule only): two
    exchanges -- stages 0..m-1 need the global qubits; the qubits swapped
    out are those needed right after the first tile pass (9 stages with
    12-bit tiles), and the second exchange trades them back for finished
    qubits -- and the same three 12-bit local passes as the unsharded QFT
    (9 + 9 + 12 stages; Alg. 3)."""
    s = lq.lq_dist_schedule_json(30, m, [], qft=1)
    kinds = [st["kind"] for st in s["steps"]]
    assert kinds == ["swap", "local", "swap", "local"]
    assert all(len(st["g"]) == m for st in s["steps"] if st["kind"] == "swap")
    local = [st["plan"]["passes"] for st in s["steps"] if st["kind"] == "local"]
    assert len(local[0]) == 1 and sum(len(p) for p in local) == 3
    assert all(p["K"] == 12 for ps in local for p in ps)


def _qft_pass_shapes(sched):
    """(stages, low contiguous tile bits, tile bits) of every local tile pass."""
    out = []
    for st in sched["steps"]:
        if st["kind"] != "local":
            continue
        pl = st["plan"]
        for ps in pl["passes"]:
            ns = sum(1 for sb in pl["subs"][ps["sub_begin"]:ps["sub_end"]]
                     for k in pl["kops"][sb["op_begin"]:sb["op_end"]] if k["type"] == 6)   # K_QFT
            run = 0
            while run in ps["T"]:
                run += 1
            out.append((ns, run, len(ps["T"])))
    return out


@pytest.mark.parametrize("K,n,m", [(4, 12, 1), (6, 10, 2), (6, 14, 3), (5, 13, 2)])
def test_group_qft_only_balanced_runs_emulated(lq, oracle, K, n, m):
    """QFT-only schedules with tiles small enough that the balanced caps of
    the local runs bite, executed by the emulator against the oracle, forward
    and inverse."""
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, K)
    try:
        for qft in (1, -1):
            sched = lq.lq_dist_schedule_json(n, m, [], qft=qft)
            got, _ = DE.run_group(sched, oracle.init_random(n, 21 + n))
            ref = oracle.init_random(n, 21 + n)
            oracle.qft(ref, inverse=qft < 0)
            assert np.abs(got - ref).max() <= TOL
    finally:
        lq.lq_set_option(lq.LQ_OPT_TILE_BITS, 0)


def test_sharded_qft_local_runs_pack_balanced(lq):
    """The local QFT runs of a sharded state pack like plan_qft: same pass
    count as the greedy packing, the pass over the low bits takes K stages
    and the strided passes share the rest, their spare tile bits going to the
    coalescing run (config 5 at n = 34 on 2 ranks: 9 | 7 + 7 + 11 with 256-byte
    runs instead of 9 | 8 + 8 + 9 with 128-byte runs).  n = 30 and n = 36
    fill their tiles exactly and are unchanged."""
    assert _qft_pass_shapes(lq.lq_dist_schedule_json(34, 1, [], qft=1)) == \
        [(9, 3, 12), (7, 4, 11), (7, 4, 11), (11, 11, 11)]
    assert _qft_pass_shapes(lq.lq_dist_schedule_json(36, 3, [], qft=1)) == \
        [(9, 3, 12), (8, 3, 11), (8, 3, 11), (11, 11, 11)]
    assert _qft_pass_shapes(lq.lq_dist_schedule_json(30, 3, [], qft=1)) == \
        [(9, 3, 12), (9, 3, 12), (12, 12, 12)]
    for n, m in ((29, 1), (31, 3), (32, 2), (33, 3), (35, 2)):
        sh = _qft_pass_shapes(lq.lq_dist_schedule_json(n, m, [], qft=-1))
        assert sum(s[0] for s in sh) == n and all(s[1] >= 3 for s in sh)
        assert sh[-1][0] == sh[-1][2]          # the last pass is all stages


def test_bench_gpus2_relaunches_under_torchrun_reference_arm():
    """bench.py --gpus 2 without a launcher re-executes itself under
    torch.distributed.run with two ranks (127.0.0.1 rendezvous); on the
    reference arm (the oracle; no GPU needed) rank 0 alone prints the line
    and the other rank exits 0."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
