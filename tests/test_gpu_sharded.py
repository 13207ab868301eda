"""GPU parity of sharded states on ONE GPU:
lq_sv_alloc_group holds all G shards in this process and swaps halves with
device copies, running the same schedules, local tile plans (with the
shard's global bits as logic constants) and pack/swap kernels as the NCCL
path; results against the CPU oracle."""
import numpy as np
import pytest

import workloads as W
from test_gpu_parity import AMP_TOL, rich_circuit

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lq():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_23183_b200 import lq as _lq
    return _lq


@pytest.fixture(autouse=True)
def _opts(lq):
    yield
    lq.lq_set_option(lq.LQ_OPT_JIT, 1)
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, 0)


@pytest.mark.parametrize("n,G", [(6, 2), (11, 2), (14, 4), (17, 8)])
def test_sharded_init_random_norm_read(lq, oracle, n, G):
    sv = lq.ShardedState(n, group_world=G)
    sv.init_random(77 + n)
    ref = oracle.init_random(n, 77 + n)
    assert np.abs(sv.read() - ref).max() <= 1e-13
    assert abs(sv.norm2() - 1.0) <= 1e-12
    idx = [0, (1 << n) - 1, 5, (1 << (n - 1)) + 3]
    np.testing.assert_array_equal(sv.gather(idx), sv.read()[idx])
    sv.init_basis((1 << n) - 2)
    a = sv.read()
    assert a[(1 << n) - 2] == 1 and np.count_nonzero(a) == 1
    sv.free()


@pytest.mark.parametrize("n,G,jit", [(10, 2, 0), (13, 4, 0), (16, 2, 2), (18, 8, 0), (6, 8, 0), (5, 4, 2)])
def test_sharded_rich_circuit(lq, oracle, n, G, jit):
    lq.lq_set_option(lq.LQ_OPT_JIT, jit)
    rng = np.random.default_rng(900 + n)
    gates = rich_circuit(n, 120, rng)
    sv = lq.ShardedState(n, group_world=G)
    sv.init_random(3 + n).apply(gates)
    ref = oracle.init_random(n, 3 + n)
    oracle.apply_circuit(ref, gates)
    assert np.abs(sv.read() - ref).max() <= AMP_TOL
    sv.free()


@pytest.mark.parametrize("n,G", [(12, 2), (15, 8)])
def test_sharded_config5_twin_qft_roundtrip(lq, oracle, n, G):
    """Config-5 generator (30 % global, m = log2 G) + QFT, then the inverse."""
    m = G.bit_length() - 1
    w = W.config5(n, m, 300)
    sv = lq.ShardedState(n, group_world=G)
    sv.init_random(w.seed).apply(w.gates).qft()
    ref = oracle.init_random(n, w.seed)
    oracle.apply_circuit(ref, w.gates)
    oracle.qft(ref)
    assert np.abs(sv.read() - ref).max() <= AMP_TOL
    sv.qft(inverse=True)
    oracle.qft(ref, inverse=True)
    assert np.abs(sv.read() - ref).max() <= AMP_TOL
    sv.free()


def test_sharded_expval_xyz_and_random(lq, oracle):
    n, G = 14, 4
    rng = np.random.default_rng(12)
    gates = rich_circuit(n, 60, rng)
    sv = lq.ShardedState(n, group_world=G)
    sv.init_random(19).apply(gates)
    ref = oracle.init_random(n, 19)
    oracle.apply_circuit(ref, gates)
    for terms in (W.xyz_terms(n), [t for t in W.random_pauli_sum(n, 30, rng) if bin(t[1]).count("1") <= n - 2]):
        e, eo = sv.expval(terms), oracle.expval(ref, terms)
        assert abs(e - eo) <= 1e-10 * max(1.0, abs(eo))
    # the swaps done for the expectation left the state intact (logical reads)
    assert np.abs(sv.read() - ref).max() <= AMP_TOL
    sv.free()


def test_sharded_matches_unsharded_bitwise_layout_free(lq):
    """Same circuit on 1 and on 4 shards: equal up to rounding order."""
    n = 16
    w = W.config5(n, 2, 200)
    a = lq.StateVector(n)
    a.init_random(w.seed).apply(w.gates)
    b = lq.ShardedState(n, group_world=4)
    b.init_random(w.seed).apply(w.gates)
    assert np.abs(a.read() - b.read()).max() <= 1e-13
    a.free()
    b.free()


def test_group_rejects_too_small_shards(lq):
    with pytest.raises(lq.LQError):
        lq.ShardedState(4, group_world=4)


def test_nccl_loads_and_single_rank_comm(lq):
    uid = lq.lq_comm_unique_id()
    assert len(uid) == 128
    c = lq.lq_comm_init(uid, 0, 1)
    sv = lq.ShardedState(8, comm=c)      # world 1: an ordinary state
    assert sv.shard_info()[0] == 0
    sv.init_basis(3)
    assert sv.read()[3] == 1
    sv.free()
    lq.lq_comm_free(c)


# ---------------------------------------------------------------- full-scale sharded runs (c.4)

def _big(lq, n, G):
    import torch
    torch.cuda.empty_cache()
    return lq.ShardedState(n, group_world=G)


def test_sharded_n32_monomial_qft_closed_form_and_roundtrip(lq):
    """SURVEY c.4 (i)+(ii)+(iii) at n = 32 on G = 2 shards (64 GiB): a
    1000-gate monomial circuit (30 % on the global qubit) from a basis state,
    then the full QFT; 2^20 sampled amplitudes against the closed form
    e^{i phi} N^-1/2 e^{2 pi i j k' / N}; then QFT^-1 and the inverse circuit
    return the basis state; the norm stays 1."""
    from closed_forms import monomial_forward, monomial_inverse, qft_of_basis
    n, G = 32, 2
    rng = np.random.default_rng(3232)
    gates = W.monomial_circuit(n, 1000, rng, global_qubits=1, p_global=0.3)
    k = int(rng.integers(0, 1 << n))
    kp, ph = monomial_forward(n, gates, k)
    sv = _big(lq, n, G)
    sv.init_basis(k).apply(gates).qft()
    idx = np.unique(rng.integers(0, 1 << n, size=1 << 20, dtype=np.uint64))
    got = sv.gather(idx)
    want = ph * qft_of_basis(n, kp, idx)
    assert np.abs(got - want).max() <= 1e-12
    assert abs(sv.norm2() - 1.0) <= 1e-11
    sv.qft(inverse=True).apply(monomial_inverse(gates))
    back = sv.gather(np.array([k, k ^ 1, (k + 12345) % (1 << n)], dtype=np.uint64))
    assert abs(back[0] - 1.0) <= 1e-11 and np.abs(back[1:]).max() <= 1e-11
    sv.free()


def test_sharded_n32_single_qubit_layer_monomial_tail(lq):
    """SURVEY c.4 (vi) at n = 32, G = 2: an H/RX/RY on every qubit from
    |0...0> (H/RX/RY on the global qubit force real swaps), then a monomial
    tail (30 % global); any amplitude j = phase(j) prod_q (U_q|0>)_{b_q(k(j))}
    by walking the tail backwards; 2^16 sampled indices."""
    from closed_forms import monomial_backward
    n, G = 32, 2
    rng = np.random.default_rng(3233)
    layer, col = [], []
    for q in range(n):
        kind = ["H", "RX", "RY"][int(rng.integers(0, 3))]
        t = float(rng.uniform(0, 2 * np.pi))
        layer.append((kind, q, -1, -1, t if kind != "H" else 0.0))
        c, s = np.cos(t / 2), np.sin(t / 2)
        col.append({"H": (1 / np.sqrt(2), 1 / np.sqrt(2)), "RX": (c, -1j * s), "RY": (c, s)}[kind])
    tail = W.monomial_circuit(n, 600, rng, global_qubits=1, p_global=0.3)
    sv = _big(lq, n, G)
    sv.init_basis(0).apply(layer + tail)
    idx = np.unique(rng.integers(0, 1 << n, size=1 << 16, dtype=np.uint64))
    got = sv.gather(idx)
    want = np.empty(idx.size, np.complex128)
    for i, j in enumerate(idx.tolist()):
        kk, ph = monomial_backward(n, tail, j)
        a = ph
        for q in range(n):
            a *= col[q][(kk >> (n - 1 - q)) & 1]
        want[i] = a
    assert np.abs(got - want).max() <= 1e-12
    sv.free()


# ---------------------------------------------------------------- k-qubit exchanges (all-to-all)

@pytest.mark.parametrize("n,G", [(12, 4), (18, 8), (20, 8)])
def test_group_alltoall_matches_pairwise_and_oracle(lq, oracle, n, G):
    """The config-5 generator + QFT on G shards with k-qubit all-to-all
    exchanges (LQ_OPT_SWAP_QUBITS = 4: the distributed QFT takes two
    exchanges) and with pairwise swaps only (= 1): both equal the oracle;
    exchange statistics count (2^k - 1) / 2^k of a shard per exchange."""
    m = G.bit_length() - 1
    w = W.config5(n, m, 400)
    ref = oracle.init_random(n, w.seed)
    oracle.apply_circuit(ref, w.gates)
    oracle.qft(ref)
    stats = {}
    for k in (1, 4):
        lq.lq_set_option(lq.LQ_OPT_SWAP_QUBITS, k)
        try:
            sv = lq.ShardedState(n, group_world=G)
            sv.init_random(w.seed).apply(w.gates).qft()
            assert np.abs(sv.read() - ref).max() <= AMP_TOL
            stats[k] = lq.lq_sv_exchange_stats(sv.h)
            sv.free()
        finally:
            lq.lq_set_option(lq.LQ_OPT_SWAP_QUBITS, 4)
    sched1 = None
    lq.lq_set_option(lq.LQ_OPT_SWAP_QUBITS, 1)
    try:
        sched1 = lq.lq_dist_schedule_json(n, m, w.gates, qft=1)
    finally:
        lq.lq_set_option(lq.LQ_OPT_SWAP_QUBITS, 4)
    sched4 = lq.lq_dist_schedule_json(n, m, w.gates, qft=1)
    shard_bytes = 16 << (n - m)
    for k, sc in ((1, sched1), (4, sched4)):
        assert stats[k][0] == sc["n_swaps"]
        assert abs(stats[k][1] - sc["shard_fraction_sent"] * shard_bytes) <= 1
    if G > 2:
        assert sched4["n_swaps"] < sched1["n_swaps"] and stats[4][1] <= stats[1][1]


def test_nccl_world1_exchange_free_path(lq):
    """A world-1 NCCL communicator: the sharded allocation degenerates to an
    ordinary state (no exchange), lq_sv_exchange_stats reports none."""
    c = lq.lq_comm_init(lq.lq_comm_unique_id(), 0, 1)
    sv = lq.ShardedState(10, comm=c)
    sv.init_random(3).apply(W.config5(10, 1, 50).gates).qft()
    assert abs(sv.norm2() - 1.0) <= 1e-12
    assert lq.lq_sv_exchange_stats(sv.h) == (0, 0)
    sv.free()
    lq.lq_comm_free(c)


@pytest.mark.parametrize("n,G", [(12, 2), (15, 4), (18, 8)])
def test_group_staged_exchange_is_the_nccl_data_path(lq, oracle, n, G):
    """LQ_OPT_GROUP_STAGED: group-mode exchanges through the NCCL path's
    pack / unpack kernels and peer map (device copies in place of the
    grouped send / receive): the config-5 generator + QFT + a Pauli sum
    against the oracle, and bit-identical to the in-place swap kernel."""
    m = G.bit_length() - 1
    w = W.config5(n, m, 300)
    terms = W.xyz_terms(n)
    ref = oracle.init_random(n, w.seed)
    oracle.apply_circuit(ref, w.gates)
    oracle.qft(ref)
    eo = oracle.expval(ref, terms)
    out = []
    for staged in (1, 0):
        lq.lq_set_option(lq.LQ_OPT_GROUP_STAGED, staged)
        try:
            sv = lq.ShardedState(n, group_world=G)
            sv.init_random(w.seed).apply(w.gates).qft()
            amps = sv.read()
            e = sv.expval(terms)
            assert lq.lq_sv_exchange_stats(sv.h)[0] > 0
            sv.free()
        finally:
            lq.lq_set_option(lq.LQ_OPT_GROUP_STAGED, 0)
        assert np.abs(amps - ref).max() <= AMP_TOL
        assert abs(e - eo) <= 1e-10 * max(1.0, abs(eo))
        out.append((amps, e))
    np.testing.assert_array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]


def test_sharded_schedule_cache_rebinds_theta(lq, oracle):
    """A cached sharded schedule (same gates, same layout) is reused with a
    different theta: the angles are bound per call (k_build_mats), not
    baked into the schedule."""
    n, G = 14, 4
    gates = W.hea_ansatz(n, 2, "ring")
    rng = np.random.default_rng(314)
    for _ in range(3):
        theta = rng.uniform(0, 2 * np.pi, 4 * n)
        sv = lq.ShardedState(n, group_world=G)
        sv.init_random(9).apply(gates, theta)
        ref = oracle.init_random(n, 9)
        oracle.apply_circuit(ref, gates, theta)
        assert np.abs(sv.read() - ref).max() <= AMP_TOL
        sv.free()


@pytest.mark.parametrize("n,G", [(11, 2), (14, 8)])
def test_sharded_write_checkpoint_restore(lq, oracle, n, G):
    """lq_sv_write on a sharded handle (checkpoint restore): read the whole
    state after a circuit, overwrite it with a basis state, write the
    checkpoint back -- once in the identity layout and once while the layout
    is permuted by exchanges and relabels -- then continue the circuit; equal
    to the oracle's uninterrupted run."""
    m = G.bit_length() - 1
    w = W.config5(n, m, 240)
    first, second = w.gates[:120], w.gates[120:]
    ref = oracle.init_random(n, w.seed)
    oracle.apply_circuit(ref, first)
    mid = ref.copy()
    oracle.apply_circuit(ref, second)
    sv = lq.ShardedState(n, group_world=G)
    sv.init_random(w.seed).apply(first)
    ckpt = sv.read()
    assert np.abs(ckpt - mid).max() <= AMP_TOL
    sv.init_basis(0)                                   # identity layout
    lq.lq_sv_write(sv.h, ckpt)
    assert np.abs(sv.read() - mid).max() <= AMP_TOL
    sv.apply(second)
    assert np.abs(sv.read() - ref).max() <= AMP_TOL
    # restore into a permuted layout: the logical amplitudes land where the layout says
    sv.init_random(1).apply(first)
    assert sv.shard_info()[3] != 0 or sv.qubit_map() != list(range(n - 1, -1, -1))
    lq.lq_sv_write(sv.h, ckpt)
    assert np.abs(sv.read() - mid).max() <= AMP_TOL
    sv.apply(second)
    assert np.abs(sv.read() - ref).max() <= AMP_TOL
    sv.free()
