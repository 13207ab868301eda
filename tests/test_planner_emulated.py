"""Host planner checked on CPU: liblq's exported plans executed by the
test-side plan emulator (tests/plan_emulator.py) must reproduce the oracle.
Covers tiling, register sub-blocks, folded permutations, 1q fusion and the
Pauli-group (expectation) ops without a GPU."""
import numpy as np
import pytest

import workloads as W
import plan_emulator as EM
from test_gpu_parity import rich_circuit


@pytest.fixture(scope="module")
def lq():
    from paper_2512_23183_b200 import build
    build.build()
    from paper_2512_23183_b200 import lq as _lq
    yield _lq
    _lq.lq_set_option(_lq.LQ_OPT_TILE_BITS, 0)
    _lq.lq_set_option(_lq.LQ_OPT_REG_BITS, 4)


def emulate(lq, n, gates, psi0, theta=None, terms=(), shift=None):
    plan = lq.lq_plan_export_json(n, gates, terms)
    psi = psi0.copy()
    E = EM.run(plan, psi, theta, shift)
    return EM.logical_state(plan["qmap"], psi), E, plan


@pytest.mark.parametrize("K,rb", [(0, 4), (5, 4), (6, 3), (3, 3)])
@pytest.mark.parametrize("n", [3, 9, 14])
def test_emulated_rich_circuits(lq, oracle, n, K, rb):
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, K)
    lq.lq_set_option(lq.LQ_OPT_REG_BITS, rb)
    rng = np.random.default_rng(7000 + 31 * n + K)
    gates = rich_circuit(n, 120, rng)
    psi0 = oracle.init_random(n, 5 + n)
    got, _, _ = emulate(lq, n, gates, psi0)
    ref = oracle.apply_circuit(psi0.copy(), gates)
    assert np.abs(got - ref).max() <= 1e-10


@pytest.mark.parametrize("K", [0, 5])
@pytest.mark.parametrize("n", [6, 14])
def test_emulated_psr_energy(lq, oracle, n, K):
    """Gates + Pauli groups planned together (the parameter-shift path)."""
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, K)
    gates = W.hea_ansatz(n, 2, "ring")
    theta = np.random.default_rng(n).uniform(0, 2 * np.pi, 4 * n)
    for terms in (W.xyz_terms(n), W.random_pauli_sum(n, 20, np.random.default_rng(n + 1))):
        psi0 = oracle.zeros(n)
        _, E, plan = emulate(lq, n, gates, psi0, theta, terms)
        assert E == pytest.approx(oracle.energy(n, gates, theta, terms), abs=1e-10)


@pytest.mark.parametrize("n", [5, 13])
def test_emulated_expval_only(lq, oracle, n):
    rng = np.random.default_rng(n)
    terms = W.random_pauli_sum(n, 30, rng)
    psi0 = oracle.init_random(n, 9)
    _, E, plan = emulate(lq, n, [], psi0, None, terms)
    assert E == pytest.approx(oracle.expval(psi0, terms), abs=1e-10)


@pytest.mark.parametrize("relabel", [3, 4, 5])
@pytest.mark.parametrize("n", [12, 14])
def test_emulated_psr_relabel_stores(lq, oracle, n, relabel):
    """The parameter-shift planner with relabelling out-of-place stores
    (LQ_OPT_RELABEL_STORES): every storing tile pass writes the
    state in the next pass's frame.  The plan's energy and final state (in the
    exported final layout) match the oracle; every pass after the first reads
    its tile as the contiguous low bits, and every store's lowest `relabel`
    lane bits land on the new frame's lowest bits."""
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, 7 if n == 12 else 0)
    lq.lq_set_option(lq.LQ_OPT_EXPORT_PSR, 1)
    lq.lq_set_option(lq.LQ_OPT_RELABEL_STORES, relabel)
    try:
        gates = W.hea_ansatz(n, 3, "ring")
        theta = np.random.default_rng(n).uniform(0, 2 * np.pi, 6 * n)
        terms = W.xyz_terms(n)
        psi0 = oracle.zeros(n)
        got, E, plan = emulate(lq, n, gates, psi0, theta, terms)
        assert E == pytest.approx(oracle.energy(n, gates, theta, terms), abs=1e-10)
        tiles = [p for p in plan["passes"] if p["kind"] == EM.PASS_TILE]
        assert all(p["oop"] for p in tiles if not (p["flags"] & EM.PF_NO_STORE))
        K = plan["K"]
        for a, b in zip(tiles, tiles[1:]):
            if a["oop"]:
                assert sorted(b["T"]) == list(range(K))       # contiguous reads
                sm = set(a["Sstore"][:plan["Rr"]])
                lanes = [a["T"][l] for l in range(K) if l not in sm][:relabel]
                assert [a["spos"][x] for x in lanes] == list(range(len(lanes)))
        # the final state, read through the exported final layout
        ref = oracle.apply_circuit(oracle.zeros(n), gates, theta)
        if not (tiles[-1]["flags"] & EM.PF_NO_STORE):
            assert np.abs(got - ref).max() <= 1e-10
    finally:
        lq.lq_set_option(lq.LQ_OPT_EXPORT_PSR, 0)
        lq.lq_set_option(lq.LQ_OPT_RELABEL_STORES, 0)


@pytest.mark.parametrize("K,rb", [(0, 4), (6, 4), (5, 3), (7, 2)])
@pytest.mark.parametrize("n", [4, 9, 10, 13, 14])
def test_emulated_qft_plans(lq, oracle, n, K, rb):
    """plan_qft (the single-state QFT planner: balanced stage packing, register
    twiddle tables, per-pass scale, bit reversal and the last pass's store
    relabel folded into the qubit map) executed by the plan emulator against
    the oracle's QFT, forward and inverse, from the identity
    layout and from the layout a forward QFT leaves."""
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, K)
    lq.lq_set_option(lq.LQ_OPT_REG_BITS, rb)
    psi_log = oracle.init_random(n, 77 + n)
    x = np.arange(psi_log.size, dtype=np.int64)
    for inverse in (False, True):
        ref = psi_log.copy()
        oracle.qft(ref, inverse=inverse)
        for rev in (False, True):
            plan = lq.lq_qft_plan_export_json(n, inverse, rev)
            stages = [sum(1 for k in plan["kops"][sb["op_begin"]:sb["op_end"]] if k["type"] == EM.K_QFT)
                      for ps in plan["passes"] for sb in plan["subs"][ps["sub_begin"]:ps["sub_end"]]]
            assert sum(stages) == n
            # physical-layout input: logical bit n-1-q sits on physical bit qmap_in[q]
            g = np.zeros_like(x)
            for q in range(n):
                g |= ((x >> (n - 1 - q)) & 1) << plan["qmap_in"][q]
            psi = np.empty_like(psi_log)
            psi[g] = psi_log
            EM.run(plan, psi)
            got = EM.logical_state(plan["qmap"], psi)
            assert np.abs(got - ref).max() <= 1e-12


def test_qft_plan_balanced_stage_packing(lq):
    """The strided passes share n - K stages evenly and fill their spare tile
    bits with low bits (longer coalescing runs); the contiguous pass takes K
    stages; the pass count is the greedy packing's."""
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, 0)
    lq.lq_set_option(lq.LQ_OPT_REG_BITS, 4)

    def shape(n, inverse=False, rev=False):
        plan = lq.lq_qft_plan_export_json(n, inverse, rev)
        out = []
        for ps in plan["passes"]:
            ns = sum(1 for sb in plan["subs"][ps["sub_begin"]:ps["sub_end"]]
                     for k in plan["kops"][sb["op_begin"]:sb["op_end"]] if k["type"] == EM.K_QFT)
            run = 0
            while run in ps["T"]:
                run += 1
            out.append((ns, run, len(ps["T"])))
        return out

    assert [s[0] for s in shape(30)] == [9, 9, 12]
    assert [s[0] for s in shape(28)] == [8, 8, 12]
    assert [s[1] for s in shape(28)] == [4, 4, 12]          # 256-byte runs
    # QFT^-1 of the layout a forward QFT leaves starts with the contiguous pass
    assert [s[0] for s in shape(28, True, True)] == [12, 8, 8]
    assert [s[1] for s in shape(28, True, True)] == [12, 4, 4]
    s31 = shape(31)
    assert [s[0] for s in s31] == [7, 7, 6, 11] and [s[1] for s in s31] == [4, 4, 5, 11]
    # at equal pass counts the automatic tile size takes 12 bits when 11 would
    # leave a strided pass on 128-byte runs (n = 27, 33), else 11 (n = 25, 31, 32)
    assert [s[0] for s in shape(33)] == [7, 7, 7, 12] and [s[1] for s in shape(33)] == [5, 5, 5, 12]
    assert [s[0] for s in shape(27)] == [8, 7, 12]
    assert [s[2] for s in shape(25)] == [11] * 3 and [s[2] for s in shape(32)] == [11] * 4
    for n in range(13, 41):
        sh = shape(n)
        assert sum(s[0] for s in sh) == n and all(s[2] == sh[0][2] for s in sh)
        assert all(s[1] >= 3 for s in sh)
