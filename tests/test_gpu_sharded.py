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
