"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Tolerances (BASELINE.json north_star; reading A16): amplitudes max-abs
<= 1e-10; expectations |E - E_o| <= 1e-10 max(|E_o|, 1); gradients
|g_i - g_o,i| <= 1e-10 max(|g_o,i|, ||g_o||_inf).
"""
import math

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

AMP_TOL = 1e-10


@pytest.fixture(scope="module")
def lq():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_23183_b200 import lq as _lq
    assert _lq.lq_device_count() >= 1
    return _lq


@pytest.fixture(autouse=True)
def _restore_options(lq):
    yield
    lq.lq_set_option(lq.LQ_OPT_FUSION, 1)
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, 0)
    lq.lq_set_option(lq.LQ_OPT_COALESCE_BITS, 3)
    lq.lq_set_option(lq.LQ_OPT_REG_BITS, 4)
    lq.lq_set_option(lq.LQ_OPT_JIT, 1)
    lq.lq_set_option(lq.LQ_OPT_FIRST_PASS_FREE, 1)
    lq.lq_set_option(lq.LQ_OPT_POISON_ALLOC, 0)
    lq.lq_set_option(lq.LQ_OPT_RELABEL_STORES, 0)
    lq.lq_set_option(lq.LQ_OPT_GRAPHS, 1)


def grad_close(g, go):
    scale = max(float(np.abs(go).max()), 1e-300)
    tol = 1e-10 * np.maximum(np.abs(go), scale)
    assert np.all(np.abs(g - go) <= tol), f"max grad err {np.abs(g - go).max():.3e} (scale {scale:.3e})"


ALL_KINDS = ("H", "X", "Y", "Z", "S", "SDG", "T", "TDG", "RX", "RY", "RZ", "CNOT", "CZ", "CP",
             "SWAP", "CRY", "RXX", "RYY", "RZZ", "U1", "U2", "CCX")


def rich_circuit(n, n_gates, rng):
    """Every gate kind the ABI accepts, on uniformly random qubits."""
    kinds = [k for k in ALL_KINDS if (k != "CCX" or n >= 3) and (k not in
             ("CNOT", "CZ", "CP", "SWAP", "CRY", "RXX", "RYY", "RZZ", "U2") or n >= 2)]
    gates = []
    for _ in range(n_gates):
        k = kinds[int(rng.integers(len(kinds)))]
        qs = [int(q) for q in rng.choice(n, size=3 if n >= 3 else n, replace=False)]
        ang = float(rng.uniform(0, 2 * np.pi)) if k in W.PARAMETRIC else 0.0
        if k in ("RX", "RY", "RZ", "H", "X", "Y", "Z", "S", "SDG", "T", "TDG"):
            gates.append((k, qs[0], -1, -1, ang))
        elif k == "U1":
            A = rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))
            Q, _ = np.linalg.qr(A)
            gates.append(("U1", qs[0], -1, -1, 0.0, Q))
        elif k == "U2":
            A = rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4))
            Q, _ = np.linalg.qr(A)
            gates.append(("U2", qs[0], qs[1], -1, 0.0, Q))
        elif k == "CCX":
            gates.append(("CCX", qs[0], qs[1], -1, 0.0, None, qs[2]))
        else:
            gates.append((k, qs[0], qs[1], -1, ang))
    return gates


def run_gpu(lq, n, seed, gates, theta=None, qft=None):
    sv = lq.StateVector(n)
    sv.init_random(seed)
    if gates:
        sv.apply(gates, theta)
    if qft is not None:
        sv.qft(inverse=qft == "inverse")
    out = sv.read()
    sv.free()
    return out


def run_oracle(oracle, n, seed, gates, theta=None, qft=None):
    psi = oracle.init_random(n, seed)
    if gates:
        oracle.apply_circuit(psi, gates, theta)
    if qft is not None:
        oracle.qft(psi, inverse=qft == "inverse")
    return psi


# ---------------------------------------------------------------- init / io

def test_init_random_matches_oracle(lq, oracle):
    for n in (1, 3, 10, 17):
        got = run_gpu(lq, n, 1234 + n, [])
        np.testing.assert_allclose(got, oracle.init_random(n, 1234 + n), rtol=0, atol=1e-13)


def test_init_random_relative_accuracy_at_small_amplitudes(lq, oracle):
    """|a_i|^2 = -2 ln u0 -> 0 as u0 -> 1: the device's log must stay
    relatively exact there, not only to 1e-13 absolute (a table-driven log
    that added -ln2 to log c ~ ln2 lost ~1e-10 relative on the smallest
    amplitudes of n = 22).  On the 64 smallest unnormalised amplitudes of the
    oracle's formula (c.1) and 4096 seeded others, state_i / a_i is one real
    constant 1/sqrt(S) to 1e-13 relative."""
    n, seed = 22, 4242
    raw = oracle.random_gaussian_at(seed, np.arange(1 << n, dtype=np.uint64))
    small = np.argsort(np.abs(raw))[:64]
    other = np.random.default_rng(5).choice(1 << n, 4096, replace=False)
    idx = np.unique(np.concatenate([small, other])).astype(np.uint64)
    sv = lq.StateVector(n)
    sv.init_random(seed)
    ratio = sv.gather(idx) / raw[idx.astype(np.int64)]
    sv.free()
    c = float(np.median(ratio.real))
    assert np.abs(ratio - c).max() <= 1e-13 * c, np.abs(ratio - c).max() / c


def test_init_basis_norm_gather_write(lq):
    n = 12
    sv = lq.StateVector(n)
    sv.init_basis(3000)
    a = sv.read()
    assert a[3000] == 1 and np.count_nonzero(a) == 1
    assert sv.norm2() == 1.0
    amps = (np.arange(1 << n) + 1j * np.arange(1 << n)[::-1]).astype(np.complex128)
    lq.lq_sv_write(sv.h, amps)
    idx = [0, 5, 4095, 77, 1234]
    np.testing.assert_array_equal(sv.gather(idx), amps[idx])
    np.testing.assert_array_equal(sv.read(100, 50), amps[100:150])
    sv.free()


# ---------------------------------------------------------------- circuits

@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 10, 12, 13, 14, 17, 20])
def test_rich_random_circuit(lq, oracle, n):
    rng = np.random.default_rng(1000 + n)
    gates = rich_circuit(n, 160, rng)
    ref = run_oracle(oracle, n, 55 + n, gates)
    got = run_gpu(lq, n, 55 + n, gates)
    assert np.abs(got - ref).max() <= AMP_TOL


@pytest.mark.parametrize("rb", [3, 4])
@pytest.mark.parametrize("K", [2, 3, 5, 8, 12])
@pytest.mark.parametrize("n", [9, 15])
def test_tile_sizes_and_multi_tile(lq, oracle, n, K, rb):
    """Small tiles force many tiles / ragged register sets at small n;
    both register-block sizes (8 or 16 amplitudes per thread)."""
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, K)
    lq.lq_set_option(lq.LQ_OPT_REG_BITS, rb)
    rng = np.random.default_rng(2000 + n * 16 + K)
    gates = rich_circuit(n, 120, rng)
    ref = run_oracle(oracle, n, 7, gates)
    got = run_gpu(lq, n, 7, gates)
    assert np.abs(got - ref).max() <= AMP_TOL


@pytest.mark.parametrize("coalesce", [0, 1, 3])
def test_coalesce_bits(lq, oracle, coalesce):
    lq.lq_set_option(lq.LQ_OPT_COALESCE_BITS, coalesce)
    n = 16
    rng = np.random.default_rng(31 + coalesce)
    gates = rich_circuit(n, 150, rng)
    ref = run_oracle(oracle, n, 9, gates)
    assert np.abs(run_gpu(lq, n, 9, gates) - ref).max() <= AMP_TOL


@pytest.mark.parametrize("n", [3, 11, 16])
def test_unfused_pair_and_diag_kernels(lq, oracle, n):
    """LQ_OPT_FUSION=0: one pair (a4) or diagonal (a3) pass per gate."""
    lq.lq_set_option(lq.LQ_OPT_FUSION, 0)
    rng = np.random.default_rng(3000 + n)
    gates = rich_circuit(n, 100, rng)
    ref = run_oracle(oracle, n, 11, gates)
    assert np.abs(run_gpu(lq, n, 11, gates) - ref).max() <= AMP_TOL


def test_diagonal_runs(lq, oracle):
    """Runs of diagonal gates on many qubits (diag pass path)."""
    n = 18
    rng = np.random.default_rng(4)
    gates = []
    for _ in range(200):
        k = ["Z", "S", "T", "SDG", "TDG", "RZ", "CZ", "CP", "RZZ"][int(rng.integers(9))]
        a, b = (int(q) for q in rng.choice(n, 2, replace=False))
        ang = float(rng.uniform(0, 2 * np.pi)) if k in W.PARAMETRIC else 0.0
        gates.append((k, a, -1 if k in ("Z", "S", "T", "SDG", "TDG", "RZ") else b, -1, ang))
    ref = run_oracle(oracle, n, 3, gates)
    assert np.abs(run_gpu(lq, n, 3, gates) - ref).max() <= AMP_TOL


def test_parameterised_gates_with_theta(lq, oracle):
    n = 12
    gates = W.hea_ansatz(n, 3, "ring")
    theta = np.random.default_rng(8).uniform(0, 2 * np.pi, 6 * n)
    ref = run_oracle(oracle, n, 21, gates, theta)
    assert np.abs(run_gpu(lq, n, 21, gates, theta) - ref).max() <= AMP_TOL


def test_app_a_cnot_on_gpu(lq):
    """PAPER.md App. A on the GPU."""
    r2 = 1 / math.sqrt(2)
    sv = lq.StateVector(2)
    lq.lq_sv_write(sv.h, np.array([r2, 0, 0, r2], np.complex128))
    sv.apply([("CNOT", 0, 1, -1, 0.0)])
    np.testing.assert_allclose(sv.read(), [r2, 0, r2, 0], atol=1e-16)


def test_app_b_toffoli_on_gpu(lq):
    """PAPER.md App. B on the GPU."""
    r2 = 1 / math.sqrt(2)
    sv = lq.StateVector(3)
    lq.lq_sv_write(sv.h, np.array([0, 0, 0, 0, 0, r2, r2, 0], np.complex128))
    sv.apply([("CCX", 0, 1, -1, 0.0, None, 2)])
    np.testing.assert_allclose(sv.read(), [0, 0, 0, 0, 0, r2, 0, r2], atol=1e-16)


# ---------------------------------------------------------------- config 1

def test_config1_exact(lq, oracle):
    """BASELINE configs[0]: n=10 seeded state, 200 random gates, full QFT."""
    w = W.config1()
    ref = run_oracle(oracle, w.n, w.seed, w.gates, qft="forward")
    got = run_gpu(lq, w.n, w.seed, w.gates, qft="forward")
    assert np.abs(got - ref).max() <= AMP_TOL
    assert abs(np.vdot(got, got).real - 1) < 1e-12


# ---------------------------------------------------------------- QFT

@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8, 11, 12, 13, 16, 19])
def test_qft_random_state(lq, oracle, n):
    ref = run_oracle(oracle, n, 40 + n, [], qft="forward")
    got = run_gpu(lq, n, 40 + n, [], qft="forward")
    assert np.abs(got - ref).max() <= AMP_TOL


@pytest.mark.parametrize("n", [3, 10, 15])
def test_qft_inverse_and_roundtrip(lq, oracle, n):
    ref = run_oracle(oracle, n, 60 + n, [], qft="inverse")
    assert np.abs(run_gpu(lq, n, 60 + n, [], qft="inverse") - ref).max() <= AMP_TOL
    sv = lq.StateVector(n).init_random(60 + n)
    sv.qft().qft(inverse=True)
    assert np.abs(sv.read() - oracle.init_random(n, 60 + n)).max() <= AMP_TOL
    # inverse first, then forward (layout reversed <-> identity both ways)
    sv.init_random(60 + n).qft(inverse=True).qft()
    assert np.abs(sv.read() - oracle.init_random(n, 60 + n)).max() <= AMP_TOL
    sv.free()


@pytest.mark.parametrize("rb", [3, 4])
@pytest.mark.parametrize("K", [3, 6, 12])
def test_qft_small_tiles(lq, oracle, K, rb):
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, K)
    lq.lq_set_option(lq.LQ_OPT_REG_BITS, rb)
    n = 14
    ref = run_oracle(oracle, n, 5, [], qft="forward")
    assert np.abs(run_gpu(lq, n, 5, [], qft="forward") - ref).max() <= AMP_TOL


@pytest.mark.parametrize("jit", [0, 2])
@pytest.mark.parametrize("n", [13, 15, 20])
def test_qft_relabel_store_chains(lq, oracle, n, jit):
    """plan_qft's last pass stores without a store exchange and relabels the
    qubits (PF_RELABEL): the forward QFT ends in a layout that is neither
    natural nor reversed, so a following QFT / inverse QFT takes the
    permuted-layout path.  Every link vs the oracle, interpreter and JIT."""
    lq.lq_set_option(lq.LQ_OPT_JIT, jit)
    psi = oracle.init_random(n, 40 + n)
    sv = lq.StateVector(n).init_random(40 + n)
    oracle.qft(psi)
    sv.qft()
    qm = sv.qubit_map()
    assert sorted(qm) == list(range(n))
    assert qm != list(range(n)) and qm != [n - 1 - q for q in range(n)]
    assert np.abs(sv.read() - psi).max() <= AMP_TOL
    oracle.qft(psi)
    sv.qft()
    assert np.abs(sv.read() - psi).max() <= AMP_TOL
    oracle.qft(psi, inverse=True)
    oracle.qft(psi, inverse=True)
    sv.qft(inverse=True).qft(inverse=True)
    assert np.abs(sv.read() - psi).max() <= AMP_TOL
    np.testing.assert_allclose(sv.read(), oracle.init_random(n, 40 + n), rtol=0, atol=AMP_TOL)
    sv.free()


def test_qft_then_gates_then_canonicalize(lq, oracle):
    """Gates after a QFT act through the qubit map; canonicalize
    materialises natural order."""
    n = 13
    rng = np.random.default_rng(17)
    gates = rich_circuit(n, 80, rng)
    psi = oracle.init_random(n, 2)
    oracle.qft(psi)
    oracle.apply_circuit(psi, gates)
    oracle.qft(psi)
    sv = lq.StateVector(n).init_random(2).qft().apply(gates).qft()
    assert np.abs(sv.read() - psi).max() <= AMP_TOL
    sv.canonicalize()
    assert sv.qubit_map() == [n - 1 - q for q in range(n)]
    import torch
    torch.cuda.synchronize()
    raw = sv.tensor.cpu().numpy()
    assert np.abs(raw - psi).max() <= AMP_TOL
    sv.free()


def test_config2_qft_n20_closed_form(lq, oracle):
    """BASELINE configs[1]: QFT(20) on 16 seeded basis states against the
    closed form N^-1/2 e^{2 pi i j k / N}, every amplitude, and
    on the seeded random state against the oracle's independent numpy ifft
    route (numpy.fft.ifft * sqrt(N))."""
    w = W.config2()
    n, N = w.n, 1 << w.n
    j = np.arange(N, dtype=np.int64)
    sv = lq.StateVector(n)
    for k in w.basis:
        sv.init_basis(k).qft()
        expect = np.exp(2j * np.pi * ((j * k) % N) / N) / math.sqrt(N)
        assert np.abs(sv.read() - expect).max() <= AMP_TOL
    sv.init_random(w.seed).qft()
    ref = np.fft.ifft(oracle.init_random(n, w.seed)) * math.sqrt(N)
    assert np.abs(sv.read() - ref).max() <= AMP_TOL
    sv.free()


# ---------------------------------------------------------------- expectation

@pytest.mark.parametrize("n", [1, 2, 4, 9, 14])
def test_expval_random_pauli_sums(lq, oracle, n):
    rng = np.random.default_rng(70 + n)
    terms = W.random_pauli_sum(n, min(40, 4 ** n), rng)
    psi = oracle.init_random(n, 70 + n)
    eo = oracle.expval(psi, terms)
    sv = lq.StateVector(n).init_random(70 + n)
    e = sv.expval(terms)
    assert abs(e - eo) <= 1e-10 * max(abs(eo), 1.0)
    sv.free()


def test_expval_wide_x_masks_direct_path(lq, oracle):
    """x masks wider than a tile take the direct pair kernel."""
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, 5)
    n = 13
    full = (1 << n) - 1
    terms = [(0.7, full, 0), (-0.3, full, full), (0.2, full & 0x5555, full & 0x0F0F), (1.1, 0, full)]
    psi = oracle.init_random(n, 3)
    eo = oracle.expval(psi, terms)
    sv = lq.StateVector(n).init_random(3)
    assert abs(sv.expval(terms) - eo) <= 1e-10 * max(abs(eo), 1.0)
    sv.free()


def test_expval_after_qft_uses_qubit_map(lq, oracle):
    n = 12
    rng = np.random.default_rng(12)
    terms = W.random_pauli_sum(n, 30, rng)
    psi = oracle.init_random(n, 4)
    oracle.qft(psi)
    sv = lq.StateVector(n).init_random(4).qft()
    assert sv.qubit_map() != [n - 1 - q for q in range(n)]
    eo = oracle.expval(psi, terms)
    assert abs(sv.expval(terms) - eo) <= 1e-10 * max(abs(eo), 1.0)
    sv.free()


# ---------------------------------------------------------------- parameter shift

def test_psr_single_ry_closed_form(lq):
    for t in [0.0, 0.3, math.pi / 2, 2.0]:
        g, e = lq.lq_param_shift_grad(1, [("RY", 0, -1, 0, 0.0)], [t], [(1.0, 0, 1)])
        assert abs(e - math.cos(t)) <= 1e-15 and abs(g[0] + math.sin(t)) <= 1e-15


def test_psr_app_e_table(lq, oracle):
    """PAPER.md App. E circuit (CRY included) on the GPU vs the oracle."""
    gates = W.edge_case_circuit()
    for th in ([0.5, 0.3, 0.2, 0.1], [10.0, 5.0, 3.0, 2.0], [1e-8, 1e-7, 1e-6, 1e-5],
               [math.pi / 2] * 4, [math.pi] * 4):
        g, _ = lq.lq_param_shift_grad(2, gates, th, [(1.0, 0, 1)])
        go = oracle.param_shift_grad(2, gates, np.array(th), [(1.0, 0, 1)])
        assert np.all(np.isfinite(g))
        # theta_3 (CRY) takes the four-term rule on both sides (reading A8)
        np.testing.assert_allclose(g, go, rtol=0, atol=1e-14)


def test_psr_cry_four_term_closed_form_and_oracle(lq, oracle):
    """Reading A8 (f3): H(0), CRY(t; 0 -> 1): <X_0> = cos(t/2), dE/dt =
    -sin(t/2)/2 exactly (the two-term rule would be off by a factor sqrt2);
    then a 10-qubit circuit mixing CRY and RX/RY/RZ parameters vs the
    oracle's four-term rule."""
    for t in [0.0, 0.4, 1.3, 2.9, 5.1]:
        g, e = lq.lq_param_shift_grad(2, [("H", 0, -1, -1, 0.0), ("CRY", 0, 1, 0, 0.0)], [t], [(1.0, 1, 0)])
        assert abs(e - math.cos(t / 2)) <= 1e-15 and abs(g[0] + math.sin(t / 2) / 2) <= 1e-15
    n = 10
    rng = np.random.default_rng(123)
    gates, p = [], 0
    for layer in range(3):
        for q in range(n):
            gates.append((["RY", "RX", "RZ"][(q + layer) % 3], q, -1, p, 0.0)); p += 1
        for q in range(layer % 2, n - 1, 2):
            gates.append(("CRY", q, q + 1, p, 0.0)); p += 1
            gates.append(("CNOT", q + 1, q, -1, 0.0))
    theta = rng.uniform(0, 2 * np.pi, p)
    terms = W.random_pauli_sum(n, 20, rng)
    g, e = lq.lq_param_shift_grad(n, gates, theta, terms)
    go = oracle.param_shift_grad(n, gates, theta, terms, threads=8)
    grad_close(g, go)
    assert abs(e - oracle.energy(n, gates, theta, terms)) <= 1e-10 * max(1.0, abs(e))


def test_config3_gradient(lq, oracle):
    """BASELINE configs[2]: n=4 HEA, 48 params, 15-term H, 96 shifted circuits."""
    w = W.config3()
    g, e = lq.lq_param_shift_grad(w.n, w.gates, w.theta, w.terms)
    go = oracle.param_shift_grad(w.n, w.gates, w.theta, w.terms)
    eo = oracle.energy(w.n, w.gates, w.theta, w.terms)
    grad_close(g, go)
    assert abs(e - eo) <= 1e-10 * max(abs(eo), 1)


PARAM_KINDS = ("RX", "RY", "RZ", "CP", "CRY", "RXX", "RYY", "RZZ")


@pytest.mark.parametrize("n", [1, 2, 3, 6, 9, 12])
def test_psr_every_kind(lq, oracle, n):
    """Parameter-shift gradients of circuits with every gate kind, one
    parameter per rotation (reading A7) plus two no gate uses
    (CRY four-term rule, reading A8), and Pauli sums with
    X / Y / Z factors, vs the oracle."""
    rng = np.random.default_rng(4200 + n)
    gates, n_par = [], 0
    for g in rich_circuit(n, 60, rng):
        if g[0] in PARAM_KINDS:
            g = (g[0], g[1], g[2], n_par, 0.0)
            n_par += 1
        gates.append(g)
    n_par += 2                                   # two parameters no gate uses: g = 0
    theta = rng.uniform(0, 2 * np.pi, n_par)
    terms = W.random_pauli_sum(n, min(12, 4 ** n), rng)
    g, e = lq.lq_param_shift_grad(n, gates, theta, terms)
    go = oracle.param_shift_grad(n, gates, theta, terms, threads=8)
    grad_close(g, go)
    assert g[-1] == 0.0 and g[-2] == 0.0
    eo = oracle.energy(n, gates, theta, terms)
    assert abs(e - eo) <= 1e-10 * max(abs(eo), 1)


@pytest.mark.parametrize("world", [2, 3])
def test_psr_shards_partition_components(lq, oracle, world):
    w = W.config3()
    full, e0 = lq.lq_param_shift_grad(w.n, w.gates, w.theta, w.terms)
    acc = np.zeros_like(full)
    for r in range(world):
        c = lq.lq_comm_init_local(r, world)
        assert lq.lq_comm_info(c) == (r, world, False)
        g, e = lq.lq_param_shift_grad(w.n, w.gates, w.theta, w.terms, comm=c)
        lq.lq_comm_free(c)
        owned = np.arange(full.size) % world == r
        assert np.all(g[~owned] == 0.0)
        acc += g
        assert e == (e0 if r == 0 else 0.0)
    np.testing.assert_array_equal(acc, full)   # bit-identical


def test_psr_nccl_world1_allreduce_path(lq, oracle):
    """lq_param_shift_grad / lq_psr_run with an NCCL communicator (world 1
    on this GPU): the combine writes this rank's share into the reduction
    buffer, one ncclAllReduce over n_params + 1 doubles, copies out -- the
    same gradient and E as the 1-GPU call, bit for bit."""
    w = W.config3()
    g0, e0 = lq.lq_param_shift_grad(w.n, w.gates, w.theta, w.terms)
    c = lq.lq_comm_init(lq.lq_comm_unique_id(), 0, 1)
    assert lq.lq_comm_info(c) == (0, 1, True)
    g1, e1 = lq.lq_param_shift_grad(w.n, w.gates, w.theta, w.terms, comm=c)
    lq.lq_psr_cache_clear()
    lq.lq_comm_free(c)
    np.testing.assert_array_equal(g1, g0)
    assert e1 == e0


@pytest.mark.parametrize("rb", [3, 4])
@pytest.mark.parametrize("n", [10, 16])
def test_xyz_ring_gradient_small(lq, oracle, n, rb):
    """Config-4 structure at n where the oracle runs every component."""
    lq.lq_set_option(lq.LQ_OPT_REG_BITS, rb)
    gates = W.hea_ansatz(n, 2, "ring")
    theta = np.random.default_rng(n).uniform(0, 2 * np.pi, 4 * n)
    terms = W.xyz_terms(n)
    g, e = lq.lq_param_shift_grad(n, gates, theta, terms)
    go = oracle.param_shift_grad(n, gates, theta, terms, threads=8)
    grad_close(g, go)
    eo = oracle.energy(n, gates, theta, terms)
    assert abs(e - eo) <= 1e-10 * max(abs(eo), 1)


@pytest.mark.parametrize("first_free", [0, 1])
def test_psr_zero_first_support_restriction(lq, oracle, first_free, monkeypatch):
    """A PSR plan's first pass synthesises |0...0>; while the union U of the
    tiles run so far misses some qubits, a pass loads only the indices inside
    U (the state is zero elsewhere; HBM holds garbage there) and runs only the
    tiles whose free bits lie in U.  The restricted run must equal the
    unrestricted one bit for bit (same arithmetic on the nonzero tiles) and
    the oracle; lq_psr_pass_bytes must show the restricted passes (n = 20 >
    2K - 3: the first two 11-bit tiles cannot cover every qubit)."""
    import torch
    n = 20
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, 11)
    lq.lq_set_option(lq.LQ_OPT_FIRST_PASS_FREE, first_free)
    gates = W.hea_ansatz(n, 3, "ring")
    npar = 6 * n
    theta = np.random.default_rng(20).uniform(0, 2 * np.pi, npar)
    terms = W.xyz_terms(n)
    st = torch.cuda.current_stream()
    th = torch.tensor(theta, device="cuda")

    def run():
        lq.lq_psr_cache_clear()
        P = lq.lq_psr_create(n, gates, npar, terms, stream=st)
        g = torch.zeros(npar, dtype=torch.float64, device="cuda")
        e = torch.zeros(1, dtype=torch.float64, device="cuda")
        lq.lq_psr_run(P, th.data_ptr(), g.data_ptr(), e.data_ptr())
        torch.cuda.synchronize()
        pb = lq.lq_psr_pass_bytes(P)
        lq.lq_psr_free(P)
        return g.cpu().numpy(), e.item(), pb

    g1, e1, pb1 = run()
    for _ in range(3):   # shared-memory races in the zero-slot synthesis would show as run-to-run noise
        g2, e2, _ = run()
        assert np.array_equal(g2, g1) and e2 == e1
    monkeypatch.setenv("LQ_NO_SUPPORT", "1")
    g0, e0, pb0 = run()
    monkeypatch.delenv("LQ_NO_SUPPORT")
    N = 1 << n
    # the zero-first pass writes only (every tile without support tracking,
    # tile 0 alone with it: HBM holds the state only inside the support)
    assert pb0[0] == (0, 16 * N) and pb1[0] == (0, 16 << 11)
    assert all(b in (16 * N, 32 * N) for k, b in pb0[1:] if k == 0)
    assert [k for k, _ in pb1] == [k for k, _ in pb0]
    restricted = [(b1, b0) for (k, b1), (_, b0) in zip(pb1, pb0) if k == 0 and b1 < b0]
    assert restricted and all(b1 % (16 << 11) == 0 for b1, _ in restricted)
    assert np.array_equal(g1, g0) and e1 == e0
    which = [0, n, 2 * n + 5, npar - 1]
    go = oracle.param_shift_grad(n, gates, theta, terms, which=which, threads=8)
    scale = float(np.abs(g1).max())
    for p, v in zip(which, go):
        assert abs(g1[p] - v) <= 1e-10 * max(abs(v), scale), (p, g1[p], v)
    assert abs(e1 - oracle.energy(n, gates, theta, terms)) <= 1e-10 * max(abs(e1), 1)


@pytest.mark.parametrize("relabel", [0, 3, 4, 5])
def test_psr_relabel_stores(lq, oracle, relabel):
    """Relabelling out-of-place stores (LQ_OPT_RELABEL_STORES):
    each tile pass writes the state into the other buffer of a ping-pong pair,
    in the frame where the next pass's tile is the contiguous low bits, under
    support tracking and with poisoned (NaN) work buffers.  Energy and sampled
    gradient components equal the oracle's; every mode agrees with the
    in-place plan to rounding; repeated runs are bit-identical."""
    import torch
    n = 18
    lq.lq_set_option(lq.LQ_OPT_POISON_ALLOC, 1)
    lq.lq_set_option(lq.LQ_OPT_RELABEL_STORES, relabel)
    gates = W.hea_ansatz(n, 4, "ring")
    npar = 8 * n
    theta = np.random.default_rng(180 + relabel).uniform(0, 2 * np.pi, npar)
    terms = W.xyz_terms(n) + [(0.3, 0b101 << 4, 1 << 17), (-0.2, 0, (1 << 17) | 1)]
    st = torch.cuda.current_stream()
    th = torch.tensor(theta, device="cuda")

    def run():
        lq.lq_psr_cache_clear()
        P = lq.lq_psr_create(n, gates, npar, terms, stream=st)
        g = torch.zeros(npar, dtype=torch.float64, device="cuda")
        e = torch.zeros(1, dtype=torch.float64, device="cuda")
        lq.lq_psr_run(P, th.data_ptr(), g.data_ptr(), e.data_ptr())
        torch.cuda.synchronize()
        lq.lq_psr_free(P)
        return g.cpu().numpy(), e.item()

    g1, e1 = run()
    g2, e2 = run()
    assert np.array_equal(g1, g2) and e1 == e2
    lq.lq_set_option(lq.LQ_OPT_RELABEL_STORES, 0)
    g0, e0 = run()
    scale = float(np.abs(g0).max())
    assert np.abs(g1 - g0).max() <= 1e-12 * max(scale, 1.0) and abs(e1 - e0) <= 1e-12 * max(abs(e0), 1)
    which = [0, 5, n + 3, 3 * n + 7, npar - 1]
    go = oracle.param_shift_grad(n, gates, theta, terms, which=which, threads=8)
    for p, v in zip(which, go):
        assert abs(g1[p] - v) <= 1e-10 * max(abs(v), scale), (p, g1[p], v)
    assert abs(e1 - oracle.energy(n, gates, theta, terms)) <= 1e-10 * max(abs(e1), 1)


@pytest.mark.parametrize("wide", [False, True])
def test_psr_support_tracking_untouched_qubits(lq, oracle, wide, monkeypatch):
    """Support tracking when the ansatz never touches qubits 15..19: the
    union of tiles may never cover every bit, the Pauli-group passes then read
    through the support mask, and a group whose x mask is wider than a tile
    (read by the direct kernel from HBM) must switch the tracking off.  Bit
    for bit equal to the untracked run, and equal to the oracle."""
    import torch
    n = 20
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, 11)
    gates = W.hea_ansatz(15, 2, "ring")
    npar = 60
    theta = np.random.default_rng(15).uniform(0, 2 * np.pi, npar)
    terms = W.xyz_terms(n) + [(0.5, (1 << 19) | 1, 0), (0.25, 0, (1 << 19) | (1 << 3))]
    if wide:
        terms.append((0.125, (1 << 12) - 1, 0b101))   # x over 12 bits: a direct group
    st = torch.cuda.current_stream()
    th = torch.tensor(theta, device="cuda")

    def run():
        P = lq.lq_psr_create(n, gates, npar, terms, stream=st)
        g = torch.zeros(npar, dtype=torch.float64, device="cuda")
        e = torch.zeros(1, dtype=torch.float64, device="cuda")
        lq.lq_psr_run(P, th.data_ptr(), g.data_ptr(), e.data_ptr())
        torch.cuda.synchronize()
        pb = lq.lq_psr_pass_bytes(P)
        lq.lq_psr_free(P)
        return g.cpu().numpy(), e.item(), pb

    g1, e1, pb1 = run()
    monkeypatch.setenv("LQ_NO_SUPPORT", "1")
    g0, e0, pb0 = run()
    monkeypatch.delenv("LQ_NO_SUPPORT")
    assert np.array_equal(g1, g0) and e1 == e0
    # (with the wide group the tracking stays on only if the tiles end up
    # covering every bit; either way the results must agree)
    if not wide:
        assert sum(b for _, b in pb1) < sum(b for _, b in pb0)
    go = oracle.param_shift_grad(n, gates, theta, terms, threads=8)
    grad_close(g1, go)
    eo = oracle.energy(n, gates, theta, terms)
    assert abs(e1 - eo) <= 1e-10 * max(abs(eo), 1)


@pytest.mark.parametrize("first_free", [0, 1])
@pytest.mark.parametrize("nq_ansatz,layers", [(4, 3), (8, 3)])
def test_psr_support_tracking_read_only_passes(lq, oracle, first_free, nq_ansatz, layers):
    """A read-only pass (only Pauli groups, PF_NO_STORE) writes nothing, so
    it must not widen the support: the next pass may load only what a storing
    pass wrote.  An ansatz on the first 4 or 8 of 20 qubits leaves the Pauli
    groups of the idle qubits to read-only passes (with FIRST_PASS_FREE = 0
    the plan is [gates, RO, RO, RO]).  Every fresh work buffer is filled
    with NaN bytes (LQ_OPT_POISON_ALLOC), so a load of memory no pass wrote
    shows up in E and g; both must equal the oracle."""
    n = 20
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, 11)
    lq.lq_set_option(lq.LQ_OPT_FIRST_PASS_FREE, first_free)
    lq.lq_set_option(lq.LQ_OPT_POISON_ALLOC, 1)
    lq.lq_psr_cache_clear()
    gates = W.hea_ansatz(nq_ansatz, layers, "ring")
    npar = 2 * nq_ansatz * layers
    theta = np.random.default_rng(nq_ansatz).uniform(0, 2 * np.pi, npar)
    terms = W.xyz_terms(n)
    g, e = lq.lq_param_shift_grad(n, gates, theta, terms)
    lq.lq_psr_cache_clear()
    assert np.all(np.isfinite(g)) and math.isfinite(e)
    go = oracle.param_shift_grad(n, gates, theta, terms, threads=8)
    grad_close(g, go)
    eo = oracle.energy(n, gates, theta, terms)
    assert abs(e - eo) <= 1e-10 * max(abs(eo), 1)


def test_psr_compile_time_circuit_index(lq, monkeypatch):
    """Launches of B <= 4 circuits compile one tile-body copy per circuit
    (the op-table offset as a constant).  B = 3 over 241 circuits (last batch:
    one circuit), B = 4, and the runtime-index build must agree bit for bit
    (each circuit's arithmetic and its fixed-order sums do not depend on B)."""
    n = 20
    lq.lq_set_option(lq.LQ_OPT_TILE_BITS, 11)
    gates = W.hea_ansatz(n, 3, "ring")
    npar = 6 * n
    theta = np.random.default_rng(7).uniform(0, 2 * np.pi, npar)
    terms = W.xyz_terms(n)
    out = []
    for env in ({"LQ_PSR_BATCH": "3"}, {"LQ_PSR_BATCH": "4"}, {"LQ_PSR_BATCH": "3", "LQ_JIT_RUNTIME_CIRC": "1"},
                {}):
        for k in ("LQ_PSR_BATCH", "LQ_JIT_RUNTIME_CIRC"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        lq.lq_psr_cache_clear()
        out.append(lq.lq_param_shift_grad(n, gates, theta, terms))
    for k in ("LQ_PSR_BATCH", "LQ_JIT_RUNTIME_CIRC"):
        monkeypatch.delenv(k, raising=False)
    lq.lq_psr_cache_clear()
    g0, e0 = out[0]
    for g, e in out[1:]:
        assert np.array_equal(g, g0) and e == e0


def test_config4_full_size_closed_forms(lq):
    """n=24 (configs[3] size): theta = 0 gives E = 0.4*23 + 0.3*24 = 16.4
    exactly; the product ansatz has a closed-form energy and gradient."""
    from closed_forms import product_energy_and_grad
    n = 24
    w = W.config4()
    g, e = lq.lq_param_shift_grad(n, w.gates[:3 * n], np.zeros(2 * n), w.terms)
    assert abs(e - 16.4) <= 1e-10 * 16.4
    gates, theta = W.product_ansatz(n, np.random.default_rng(24))
    g, e = lq.lq_param_shift_grad(n, gates, theta, W.xyz_terms(n))
    E, gref = product_energy_and_grad(n, theta)
    assert abs(e - E) <= 1e-10 * max(abs(E), 1)
    grad_close(g, gref)


# (configs[3] in full against the oracle: tests/test_gpu_fullsize.py)


# ---------------------------------------------------------------- boundary errors

def test_boundary_rejections_leave_state_untouched(lq):
    n = 6
    sv = lq.StateVector(n).init_random(5)
    before = sv.read()
    bad = [
        [("H", 6, -1, -1, 0.0)],                 # qubit out of range
        [("CNOT", 2, 2, -1, 0.0)],               # duplicate qubits
        [("H", 0, -1, -1, 0.3)],                 # angle on a fixed gate
        [("RX", 0, -1, 3, 0.0)],                 # param_idx without theta
    ]
    for gates in bad:
        with pytest.raises(lq.LQError) as ei:
            sv.apply(gates)
        assert ei.value.status == lq.LQ_ERR_ARG
    with pytest.raises(lq.LQError) as ei:
        sv.apply([("RX", 0, -1, -1, float("nan"))])
    assert ei.value.status == lq.LQ_ERR_NONFINITE
    with pytest.raises(lq.LQError) as ei:
        sv.apply([("RX", 0, -1, 0, 0.0)], [float("inf")])
    assert ei.value.status == lq.LQ_ERR_NONFINITE
    np.testing.assert_array_equal(sv.read(), before)
    with pytest.raises(lq.LQError):
        lq.lq_param_shift_grad(2, [("RX", 0, -1, 0, 0.0), ("RY", 1, -1, 0, 0.0)], [0.1], [(1.0, 0, 1)])
    with pytest.raises(lq.LQError):
        sv.expval([(1.0, 1 << 6, 0)])
    sv.free()


# ---------------------------------------------------------------- VQE outer loop (f2)

def test_vqe_adam_config3_trajectory_vs_oracle(lq, oracle):
    """lq_vqe_adam (batched PSR + device Adam) follows the oracle's Adam
    trajectory on config 3 for 30 iterations (gradients agree to ~1e-15, so
    the iterates may drift only by rounding)."""
    w = W.config3()
    th, tr, T = lq.lq_vqe_adam(w.n, w.gates, w.theta, w.terms, max_iter=30)
    tho, tro, To = oracle.vqe_adam(w.n, w.gates, w.theta, w.terms, max_iter=30, threads=8)
    assert T == To == 30 and tr.size == 31
    np.testing.assert_allclose(tr, tro, rtol=0, atol=1e-11)
    np.testing.assert_allclose(th, tho, rtol=0, atol=1e-10)


def test_vqe_adam_single_qubit_and_zero_hamiltonian(lq):
    th, tr, T = lq.lq_vqe_adam(1, [("RY", 0, -1, 0, 0.0)], [0.1], [(1.0, 0, 1)], lr=0.05, tol=1e-12,
                               max_iter=3000)
    assert abs(tr[-1] + 1.0) < 1e-6 and abs(math.cos(th[0]) - tr[-1]) < 1e-15
    w = W.config3()
    th, tr, T = lq.lq_vqe_adam(w.n, w.gates, w.theta, [], max_iter=10)
    assert T == 1 and np.all(tr == 0.0)
    np.testing.assert_array_equal(th, w.theta)
    with pytest.raises(lq.LQError):
        lq.lq_vqe_adam(1, [("RY", 0, -1, 0, 0.0)], [float("nan")], [(1.0, 0, 1)])


def test_cuda_graph_replay_is_bit_identical(lq):
    """LQ_OPT_GRAPHS: a launch-bound PSR plan is captured as a CUDA graph on
    its second run with the same pointers and replayed after; the replays
    give the stream path's bits, count their kernels, and follow theta
    changes written into the same device buffer.  The device-resident VQE
    loop (stopping rule + Adam in the graph) reproduces the host loop's
    trajectory bit for bit, including an early stop."""
    import torch
    w = W.config3()
    npar = len(w.theta)
    st = torch.cuda.current_stream()
    th0 = torch.tensor(w.theta, device="cuda")
    th1 = th0 + 0.25
    th = th0.clone()
    P = lq.lq_psr_create(w.n, w.gates, npar, w.terms, stream=st)
    g = torch.zeros(npar, dtype=torch.float64, device="cuda")
    e = torch.zeros(1, dtype=torch.float64, device="cuda")

    def run():
        lq.lq_psr_run(P, th.data_ptr(), g.data_ptr(), e.data_ptr())
        torch.cuda.synchronize()
        return g.cpu().numpy().copy(), e.item()
    lq.lq_set_option(lq.LQ_OPT_GRAPHS, 0)
    ref = [run()]
    th.copy_(th1)
    ref.append(run())
    th.copy_(th0)
    lq.lq_set_option(lq.LQ_OPT_GRAPHS, 1)
    got = []
    for k in range(4):      # direct, capture + replay, replay, replay (theta changed)
        if k == 3:
            th.copy_(th1)
        c0 = lq.lq_launch_count()
        got.append(run())
        assert lq.lq_launch_count() > c0
    lq.lq_psr_free(P)
    for k in range(3):
        assert np.array_equal(got[k][0], ref[0][0]) and got[k][1] == ref[0][1]
    assert np.array_equal(got[3][0], ref[1][0]) and got[3][1] == ref[1][1]
    for tol, it in ((1e-7, 40), (1e-3, 200)):   # full run / early stop
        lq.lq_set_option(lq.LQ_OPT_GRAPHS, 0)
        a = lq.lq_vqe_adam(w.n, w.gates, w.theta, w.terms, max_iter=it, tol=tol)
        lq.lq_set_option(lq.LQ_OPT_GRAPHS, 1)
        b = lq.lq_vqe_adam(w.n, w.gates, w.theta, w.terms, max_iter=it, tol=tol)
        assert a[2] == b[2] and np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        if tol == 1e-3:
            assert b[2] < it


def test_cuda_graph_single_state_replay(lq):
    """Cached single-state plans (a circuit without parameters, the QFT) are
    captured as CUDA graphs on their second run on the same state buffers
    and replayed after: bit-identical to the stream path, across a state that
    is re-initialised between runs and a second state (new buffers)."""
    rng = np.random.default_rng(77)
    n = 14
    gates = rich_circuit(n, 60, rng)
    outs = {}
    for graphs in (0, 1):
        lq.lq_set_option(lq.LQ_OPT_GRAPHS, graphs)
        res = []
        for k in range(2):
            sv = lq.StateVector(n)
            for r in range(4):     # direct, capture + replay, replay, replay
                sv.init_random(100 + r).apply(gates).qft()
                res.append(sv.read())
            sv.free()
        outs[graphs] = res
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)


# ---------------------------------------------------------------- Trotter XYZ (f1)

def test_trotter_xyz_vs_oracle(lq, oracle):
    """lq_trotter_xyz (macro-steps of up to 8 Trotter steps per fused plan,
    RXX/RYY as register-pair rotations, op K_GG) vs the oracle's native
    4x4-matrix steps:
    energies and final amplitudes, n = 11, from |1...1> and from a random
    state, record cadences 1 and 5."""
    n = 11
    for init, rec, steps in (("ones", 1, 12), ("random", 5, 23)):
        sv = lq.StateVector(n)
        ref = oracle.init_basis(n, (1 << n) - 1) if init == "ones" else oracle.init_random(n, 17)
        if init == "ones":
            sv.init_basis((1 << n) - 1)
        else:
            sv.init_random(17)
        E = sv.trotter_xyz(1.0, 0.7, 0.4, 2.0, 1.0, 0.1, 0.05, steps, rec)
        Eo = oracle.trotter_xyz(ref, 1.0, 0.7, 0.4, 2.0, 1.0, 0.1, 0.05, steps, rec)
        assert E.size == Eo.size == 1 + steps // rec
        np.testing.assert_allclose(E, Eo, rtol=0, atol=1e-10 * max(1.0, np.abs(Eo).max()))
        assert np.abs(sv.read() - ref).max() <= AMP_TOL
        sv.free()


def test_trotter_diagonal_chain_closed_form_n20(lq):
    """Jx = Jy = 0 from |1...1>: E(t) = -Jz (n-1) + n A sin(w t) exactly."""
    n = 20
    sv = lq.StateVector(n).init_basis((1 << n) - 1)
    E = sv.trotter_xyz(0.0, 0.0, 1.0, 2.0, 1.0, 0.0, 0.02, 50, 10)
    t = 0.02 * 10 * np.arange(E.size)
    np.testing.assert_allclose(E, -(n - 1) + n * 2.0 * np.sin(t), rtol=0, atol=1e-12)
    assert abs(sv.norm2() - 1) < 1e-12
    with pytest.raises(lq.LQError):
        sv.trotter_xyz(1.0, 1.0, 1.0, 0.0, 1.0, 0.0, -0.1, 3)
    sv.free()


def test_max_size_n33_monomial_qft_closed_form(lq):
    """Largest single-GPU state (n = 33, 128 GiB): a 400-gate monomial
    circuit from a basis state, then the full QFT (4 tile passes of 12 bits,
    bit reversal as a relabel); 2^18 sampled amplitudes against the closed
    form e^{i phi} N^-1/2 e^{2 pi i j k' / N} (SURVEY c.4 (i)); norm."""
    import torch
    from closed_forms import monomial_forward, qft_of_basis
    n = 33
    torch.cuda.empty_cache()
    rng = np.random.default_rng(3333)
    gates = W.monomial_circuit(n, 400, rng)
    k = int(rng.integers(0, 1 << n))
    kp, ph = monomial_forward(n, gates, k)
    sv = lq.StateVector(n)
    sv.init_basis(k).apply(gates).qft()
    idx = np.unique(rng.integers(0, 1 << n, size=1 << 18, dtype=np.uint64))
    assert np.abs(sv.gather(idx) - ph * qft_of_basis(n, kp, idx)).max() <= 1e-12
    assert abs(sv.norm2() - 1.0) <= 1e-11
    sv.free()
    del sv
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n", [25, 28, 29, 31])
def test_qft_balanced_stage_packing_closed_form(lq, n):
    """plan_qft's balanced packing (planner.cpp): the strided passes share
    n - K stages evenly and their spare tile bits lengthen the coalescing run
    (n = 28: 8+8+12 stages with 256-byte runs, n = 31: 7+6+6+12 with 512-byte
    runs).  QFT of a basis state against the closed form on sampled
    amplitudes, then QFT^-1 back to the basis state."""
    import torch
    from closed_forms import qft_of_basis
    torch.cuda.empty_cache()
    rng = np.random.default_rng(2800 + n)
    k = int(rng.integers(0, 1 << n))
    sv = lq.StateVector(n).init_basis(k).qft()
    idx = np.unique(np.concatenate([rng.integers(0, 1 << n, size=1 << 16, dtype=np.uint64),
                                    np.array([0, 1, (1 << n) - 1, k], dtype=np.uint64)]))
    assert np.abs(sv.gather(idx) - qft_of_basis(n, k, idx)).max() <= 1e-12
    assert abs(sv.norm2() - 1.0) <= 1e-11
    sv.qft(inverse=True)
    got = sv.gather(idx)
    want = (idx == np.uint64(k)).astype(np.complex128)
    assert np.abs(got - want).max() <= 1e-12
    assert abs(sv.norm2() - 1.0) <= 1e-11
    sv.free()
    del sv
    torch.cuda.empty_cache()


# ---------------------------------------------------------------- degenerate cases

@pytest.mark.parametrize("jit", [0, 2])
def test_degenerate_sizes_and_empty_inputs(lq, oracle, jit):
    """n = 1 and n = 2 states through every 1q gate, QFT and expectation;
    empty gate lists and Pauli sums; a PSR ansatz with no gates (its only
    pass synthesises |0...0> and reads it, PF_LOAD_ZERO + read-only); an
    unused parameter (gradient exactly 0) -- interpreter and JIT."""
    lq.lq_set_option(lq.LQ_OPT_JIT, jit)
    try:
        oneq = [("H", 0, -1, -1, 0.0), ("RX", 0, -1, -1, 0.7), ("RY", 0, -1, -1, 1.1), ("RZ", 0, -1, -1, 2.3),
                ("S", 0, -1, -1, 0.0), ("T", 0, -1, -1, 0.0), ("X", 0, -1, -1, 0.0), ("Y", 0, -1, -1, 0.0),
                ("Z", 0, -1, -1, 0.0), ("SDG", 0, -1, -1, 0.0), ("TDG", 0, -1, -1, 0.0)]
        for n in (1, 2):
            gates = oneq + ([("CNOT", 0, 1, -1, 0.0), ("RYY", 1, 0, -1, 0.4), ("CRY", 1, 0, -1, 0.9)] if n == 2 else [])
            sv = lq.StateVector(n).init_random(40 + n)
            ref = oracle.init_random(n, 40 + n)
            sv.apply(gates).qft()
            oracle.apply_circuit(ref, gates)
            oracle.qft(ref)
            assert np.abs(sv.read() - ref).max() <= AMP_TOL
            terms = [(0.5, 1, 0), (-0.3, 1, 1), (0.8, 0, 1)] + ([(0.2, 3, 3)] if n == 2 else [])
            assert abs(sv.expval(terms) - oracle.expval(ref, terms)) <= 1e-12
            before = sv.read()
            sv.apply([])
            np.testing.assert_array_equal(sv.read(), before)
            assert sv.expval([]) == 0.0
            sv.free()
        n = 6
        terms = W.random_pauli_sum(n, 12, np.random.default_rng(3))
        g, e = lq.lq_param_shift_grad(n, [], [], terms)
        psi0 = oracle.init_basis(n, 0)
        assert g.size == 0 and abs(e - oracle.expval(psi0, terms)) <= 1e-12
        gates = [("RY", 0, -1, 0, 0.0), ("RX", 3, -1, 2, 0.0), ("CNOT", 0, 5, -1, 0.0)]   # param 1 unused
        th = np.array([0.3, 1.7, -0.4])
        terms = [(0.7, 0, 1 << 0), (0.4, 0, 1 << 3), (0.3, 1 << 0, 1 << 5), (-0.2, 1 << 3, 0)]
        g, e = lq.lq_param_shift_grad(n, gates, th, terms)
        assert g[1] == 0.0
        go = oracle.param_shift_grad(n, gates, th, terms)
        grad_close(g, go)
    finally:
        lq.lq_set_option(lq.LQ_OPT_JIT, 1)


@pytest.mark.parametrize("mask", [0xff0007, 0x8003ff, 0xfff, 0x3fe00007 >> 8])
def test_tile_sweep_touches_every_amplitude_once(lq, mask):
    """lq_tile_sweep (the access-pattern ceiling of bench.py's roofline)
    swaps re and im of every amplitude once per sweep: after the warm-up plus
    one timed sweep the buffer is unchanged, after the warm-up plus two it is
    swapped everywhere -- every tile is visited exactly once."""
    import torch
    nb = 24
    x = torch.randn(1 << nb, dtype=torch.complex128, device="cuda")
    x0 = x.clone()
    ms = lq.lq_tile_sweep(x.data_ptr(), x.numel() * 16, nb, mask, 1)
    assert ms > 0 and torch.equal(x, x0)
    lq.lq_tile_sweep(x.data_ptr(), x.numel() * 16, nb, mask, 2)
    assert torch.equal(torch.view_as_real(x)[:, 0], torch.view_as_real(x0)[:, 1])
    assert torch.equal(torch.view_as_real(x)[:, 1], torch.view_as_real(x0)[:, 0])
