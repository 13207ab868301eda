"""GPU parity of the JIT-specialised tile passes (LQ_OPT_JIT=2, jit.cpp):
the same cases as the interpreter tests, forced through NVRTC-compiled
pass programs, against the CPU oracle -- and the JIT program is checked to
be bit-identical to the interpreter (both run the same exec_op templates in
the same order)."""
import numpy as np
import pytest

import workloads as W
from test_gpu_parity import AMP_TOL, grad_close, rich_circuit, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lq():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_23183_b200 import lq as _lq
    return _lq


@pytest.fixture(autouse=True)
def _jit(lq):
    lq.lq_set_option(lq.LQ_OPT_JIT, 2)
    yield
    lq.lq_set_option(lq.LQ_OPT_JIT, 1)
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, 0)
    lq.lq_set_option(lq.LQ_OPT_REG_BITS, 4)


@pytest.mark.parametrize("n,K,rb", [(14, 11, 4), (17, 12, 4), (20, 10, 4), (15, 9, 3)])
def test_jit_rich_random_circuit(lq, oracle, n, K, rb):
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, K)
    lq.lq_set_option(lq.LQ_OPT_REG_BITS, rb)
    rng = np.random.default_rng(7000 + n)
    gates = rich_circuit(n, 120, rng)
    ref = run_oracle(oracle, n, 99 + n, gates)
    got = run_gpu(lq, n, 99 + n, gates)
    assert np.abs(got - ref).max() <= AMP_TOL
    lq.lq_set_option(lq.LQ_OPT_JIT, 0)
    interp = run_gpu(lq, n, 99 + n, gates)
    np.testing.assert_array_equal(got, interp)


@pytest.mark.parametrize("n", [13, 18])
def test_jit_qft_roundtrip(lq, oracle, n):
    got = run_gpu(lq, n, 5 + n, [], qft="forward")
    ref = run_oracle(oracle, n, 5 + n, [], qft="forward")
    assert np.abs(got - ref).max() <= AMP_TOL
    sv = lq.StateVector(n)
    sv.init_random(5 + n).qft().qft(inverse=True)
    assert np.abs(sv.read() - oracle.init_random(n, 5 + n)).max() <= AMP_TOL
    sv.free()


def test_jit_config5_twin_with_qft(lq, oracle):
    """Config-5 generator (30 % of gates on the top qubit) at n = 16, then QFT."""
    w = W.config5(16, 1, 300)
    ref = run_oracle(oracle, 16, w.seed, w.gates, qft="forward")
    got = run_gpu(lq, 16, w.seed, w.gates, qft="forward")
    assert np.abs(got - ref).max() <= AMP_TOL


def test_jit_expval(lq, oracle):
    n = 14
    rng = np.random.default_rng(31)
    terms = W.random_pauli_sum(n, 40, rng)
    gates = rich_circuit(n, 60, rng)
    psi = run_oracle(oracle, n, 3, gates)
    eo = oracle.expval(psi, terms)
    sv = lq.StateVector(n)
    sv.init_random(3).apply(gates)
    e = sv.expval(terms)
    sv.free()
    assert abs(e - eo) <= 1e-10 * max(abs(eo), 1.0)


def test_jit_psr_config3_and_ring(lq, oracle):
    c3 = W.config3()
    g, e = lq.lq_param_shift_grad(c3.n, c3.gates, c3.theta, c3.terms)
    grad_close(g, oracle.param_shift_grad(c3.n, c3.gates, c3.theta, c3.terms))
    n = 12
    gates = W.hea_ansatz(n, 2, "ring")
    theta = np.random.default_rng(4).uniform(0, 2 * np.pi, size=4 * n)
    terms = W.xyz_terms(n)
    g, e = lq.lq_param_shift_grad(n, gates, theta, terms)
    which = [0, 5, 13, 30, 47]
    go = oracle.param_shift_grad(n, gates, theta, terms, which=which)
    grad_close(g[which], go)


@pytest.mark.parametrize("jit", [0, 2])
def test_qft_on_permuted_layout(lq, oracle, jit):
    """SWAP gates leave a permuted qubit map; the QFT then runs as generic
    Alg. 3 stage ops with a physical->logical map (no canonicalisation)."""
    lq.lq_set_option(lq.LQ_OPT_JIT, jit)
    n = 15
    rng = np.random.default_rng(5)
    perm = [("SWAP", int(a), int(b), -1, 0.0) for a, b in (rng.choice(n, 2, replace=False) for _ in range(9))]
    gates = perm + [("H", 3, -1, -1, 0.0), ("CNOT", 3, 11, -1, 0.0)]
    for inverse in (False, True):
        sv = lq.StateVector(n)
        sv.init_random(8).apply(gates).qft(inverse=inverse)
        ref = oracle.init_random(n, 8)
        oracle.apply_circuit(ref, gates)
        oracle.qft(ref, inverse=inverse)
        assert np.abs(sv.read() - ref).max() <= AMP_TOL
        sv.free()


def test_jit_constant_tables_two_streams(lq, oracle):
    """JIT passes read their op tables from a per-module constant bank that
    is refilled before each launch; modules are private to a stream, so the
    same circuit with different angles on two concurrent streams must not
    interfere."""
    import torch
    n = 14
    gates = W.hea_ansatz(n, 2, "ring")
    rng = np.random.default_rng(77)
    th = [rng.uniform(0, 2 * np.pi, 4 * n) for _ in range(2)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    svs = [lq.StateVector(n, stream=s) for s in streams]
    for rep in range(3):
        for sv, t in zip(svs, th):
            sv.init_random(5).apply(gates, t)
        torch.cuda.synchronize()
        for sv, t in zip(svs, th):
            ref = oracle.init_random(n, 5)
            oracle.apply_circuit(ref, gates, t)
            assert np.abs(sv.read() - ref).max() <= AMP_TOL
    for sv in svs:
        sv.free()
