"""Pins for the CPU oracle (runs without a GPU).

Each test checks the oracle against something other than itself: values the
paper prints (tests/golden/, with citations), closed forms, the independent
matrix-based route (oracle/fullmatrix.py, n <= 6), a library routine
(numpy.fft) or invariants.  Chosen so that a dropped term, a wrong sign or
index, or a transposed operand in oracle.c fails at least one of them.
"""
import math
import os

import numpy as np
import pytest

import workloads as W
from closed_forms import product_energy_and_grad
from oracle import fullmatrix as FM

GOLD = os.path.join(os.path.dirname(__file__), "golden")
R2 = 1.0 / math.sqrt(2.0)

ONEQ = ["H", "X", "Y", "Z", "S", "SDG", "T", "TDG", "RX", "RY", "RZ"]
TWOQ = ["CNOT", "CZ", "CP", "SWAP", "CRY", "RXX", "RYY", "RZZ"]


def rand_state(n, rng):
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return (v / np.linalg.norm(v)).astype(np.complex128)


def _read_state_golden(name):
    rows, gate = [], None
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        if line.startswith("gate"):
            gate = line.split()[1:]
            continue
        f = line.split()
        val = lambda s: R2 if s == "r2" else float(s)
        rows.append((int(f[0]), val(f[1]) + 1j * val(f[2]), val(f[3]) + 1j * val(f[4])))
    N = len(rows)
    psi_in = np.zeros(N, np.complex128)
    psi_out = np.zeros(N, np.complex128)
    for i, a, b in rows:
        psi_in[i], psi_out[i] = a, b
    return gate, psi_in, psi_out


# ---------------------------------------------------------------- printed values

def test_app_a_cnot(oracle):
    gate, psi, expect = _read_state_golden("app_a_cnot.txt")
    oracle.apply_gate(psi, gate[0], int(gate[1]), int(gate[2]))
    np.testing.assert_array_equal(psi, expect)


def test_app_b_toffoli(oracle):
    gate, psi, expect = _read_state_golden("app_b_toffoli.txt")
    oracle.apply_gate(psi, gate[0], int(gate[1]), int(gate[2]), q2=int(gate[3]))
    np.testing.assert_array_equal(psi, expect)


def _app_e_rows():
    rows = []
    for line in open(os.path.join(GOLD, "app_e_gradients.txt")):
        if line.startswith("#") or not line.strip():
            continue
        name, th, g, tol = [s.strip() for s in line.split("|")]
        ev = lambda s: {"pi": math.pi, "pi/2": math.pi / 2}.get(s, None) or float(s)
        rows.append((name, [ev(s) for s in th.split()], [float(s) for s in g.split()], float(tol)))
    return rows


@pytest.mark.parametrize("row", _app_e_rows(), ids=lambda r: r[0])
def test_app_e_psr_table(oracle, row):
    name, theta, expect, tol = row
    gates = W.edge_case_circuit()
    g = oracle.param_shift_grad(2, gates, np.array(theta), [(1.0, 0, 1)])
    assert np.all(np.isfinite(g))
    np.testing.assert_allclose(g, expect, rtol=0, atol=tol)


# ---------------------------------------------------------------- matrix route

@pytest.mark.parametrize("n", [1, 2, 3, 5, 6])
def test_every_1q_gate_vs_full_matrix(oracle, n):
    rng = np.random.default_rng(100 + n)
    for name in ONEQ:
        for q in range(n):
            ang = float(rng.uniform(0, 2 * np.pi))
            psi = rand_state(n, rng)
            ref = FM.gate_unitary(n, (name, q, -1, -1, ang)) @ psi
            oracle.apply_gate(psi, name, q, -1, ang)
            np.testing.assert_allclose(psi, ref, rtol=0, atol=1e-14, err_msg=f"{name} q{q}")


@pytest.mark.parametrize("n", [2, 3, 4, 6])
def test_every_2q_gate_vs_full_matrix(oracle, n):
    rng = np.random.default_rng(200 + n)
    for name in TWOQ:
        for a in range(n):
            for b in range(n):
                if a == b:
                    continue
                ang = float(rng.uniform(0, 2 * np.pi))
                psi = rand_state(n, rng)
                ref = FM.gate_unitary(n, (name, a, b, -1, ang)) @ psi
                oracle.apply_gate(psi, name, a, b, ang)
                np.testing.assert_allclose(psi, ref, rtol=0, atol=1e-14,
                                           err_msg=f"{name} ({a},{b})")


@pytest.mark.parametrize("n", [2, 4, 6])
def test_u1_u2_matrices_vs_full_matrix(oracle, n):
    rng = np.random.default_rng(300 + n)
    for _ in range(6):
        A = rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))
        B = rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4))
        q = int(rng.integers(n))
        a, b = rng.choice(n, 2, replace=False)
        psi = rand_state(n, rng)
        ref = FM.gate_unitary(n, ("U1", q, -1, -1, 0.0, A)) @ psi
        oracle.apply_gate(psi, "U1", q, mat=A)
        np.testing.assert_allclose(psi, ref, atol=1e-13)
        psi = rand_state(n, rng)
        ref = FM.gate_unitary(n, ("U2", int(a), int(b), -1, 0.0, B)) @ psi
        oracle.apply_gate(psi, "U2", int(a), int(b), mat=B)
        np.testing.assert_allclose(psi, ref, atol=1e-13)


def test_toffoli_all_positions_vs_full_matrix(oracle):
    n = 4
    rng = np.random.default_rng(7)
    for a in range(n):
        for b in range(n):
            for c in range(n):
                if len({a, b, c}) < 3:
                    continue
                psi = rand_state(n, rng)
                ref = FM.gate_unitary(n, ("CCX", a, b, -1, 0.0, None, c)) @ psi
                oracle.apply_gate(psi, "CCX", a, b, q2=c)
                np.testing.assert_allclose(psi, ref, atol=1e-14)


@pytest.mark.parametrize("n", [3, 5, 6])
def test_random_circuit_vs_full_matrix(oracle, n):
    rng = np.random.default_rng(400 + n)
    gates = W.random_circuit(n, 120, rng, rng)
    psi0 = oracle.init_random(n, 1234 + n)
    ref = FM.circuit_unitary(n, gates) @ psi0
    out = oracle.apply_circuit(psi0.copy(), gates)
    np.testing.assert_allclose(out, ref, atol=1e-13)


# ---------------------------------------------------------------- invariants

def test_involutions_and_compositions(oracle):
    n = 5
    rng = np.random.default_rng(11)
    psi0 = rand_state(n, rng)
    for name in ["H", "X", "Y", "Z"]:
        psi = psi0.copy()
        oracle.apply_gate(psi, name, 2)
        oracle.apply_gate(psi, name, 2)
        np.testing.assert_allclose(psi, psi0, atol=1e-14)
    for name in ["CNOT", "SWAP", "CZ"]:
        psi = psi0.copy()
        oracle.apply_gate(psi, name, 1, 3)
        oracle.apply_gate(psi, name, 1, 3)
        np.testing.assert_allclose(psi, psi0, atol=1e-14)
    for a, b in [("S", "SDG"), ("T", "TDG")]:
        psi = psi0.copy()
        oracle.apply_gate(psi, a, 4)
        oracle.apply_gate(psi, b, 4)
        np.testing.assert_allclose(psi, psi0, atol=1e-14)
    # S^2 = Z, T^2 = S, HXH = Z, Y = i X Z
    for seq, single in [(["S", "S"], "Z"), (["T", "T"], "S"), (["H", "X", "H"], "Z")]:
        p1, p2 = psi0.copy(), psi0.copy()
        for g in seq:
            oracle.apply_gate(p1, g, 0)
        oracle.apply_gate(p2, single, 0)
        np.testing.assert_allclose(p1, p2, atol=1e-14)
    p1, p2 = psi0.copy(), psi0.copy()
    oracle.apply_gate(p1, "Z", 3)
    oracle.apply_gate(p1, "X", 3)
    oracle.apply_gate(p2, "Y", 3)
    np.testing.assert_allclose(1j * p1, p2, atol=1e-14)
    # RZ(a) RZ(b) = RZ(a+b); same for RX, RY
    for r in ["RX", "RY", "RZ"]:
        p1, p2 = psi0.copy(), psi0.copy()
        oracle.apply_gate(p1, r, 1, angle=0.7)
        oracle.apply_gate(p1, r, 1, angle=1.9)
        oracle.apply_gate(p2, r, 1, angle=2.6)
        np.testing.assert_allclose(p1, p2, atol=1e-14)
    # RX(pi) = -iX, RY(pi) = -iY, RZ(pi) = -iZ
    for r, g in [("RX", "X"), ("RY", "Y"), ("RZ", "Z")]:
        p1, p2 = psi0.copy(), psi0.copy()
        oracle.apply_gate(p1, r, 2, angle=math.pi)
        oracle.apply_gate(p2, g, 2)
        np.testing.assert_allclose(p1, -1j * p2, atol=1e-15)


def test_norm_preserved_by_random_circuit(oracle):
    n = 12
    rng = np.random.default_rng(3)
    psi = oracle.init_random(n, 99)
    oracle.apply_circuit(psi, W.random_circuit(n, 300, rng, rng))
    assert abs(oracle.norm2(psi) - 1.0) < 1e-12


def test_rotation_sign_closed_forms(oracle):
    """Reading A3: RX(t)|0> has <Y> = -sin t; RY(t)|0> has <X> = +sin t;
    RZ(t)|+> has <X> = cos t, <Y> = sin t.  (Direct consequence of
    e^{-i t G/2}.)"""
    for t in [0.0, 0.3, 1.1, math.pi / 2, 2.0, 4.5]:
        psi = oracle.zeros(1)
        oracle.apply_gate(psi, "RX", 0, angle=t)
        assert oracle.expval(psi, [(1.0, 1, 1)]) == pytest.approx(-math.sin(t), abs=1e-15)
        assert oracle.expval(psi, [(1.0, 0, 1)]) == pytest.approx(math.cos(t), abs=1e-15)
        psi = oracle.zeros(1)
        oracle.apply_gate(psi, "RY", 0, angle=t)
        assert oracle.expval(psi, [(1.0, 1, 0)]) == pytest.approx(math.sin(t), abs=1e-15)
        psi = oracle.zeros(1)
        oracle.apply_gate(psi, "H", 0)
        oracle.apply_gate(psi, "RZ", 0, angle=t)
        assert oracle.expval(psi, [(1.0, 1, 0)]) == pytest.approx(math.cos(t), abs=1e-15)
        assert oracle.expval(psi, [(1.0, 1, 1)]) == pytest.approx(math.sin(t), abs=1e-15)


# ---------------------------------------------------------------- init

def test_init_basis(oracle):
    psi = oracle.init_basis(3, 6)
    expect = np.zeros(8, np.complex128)
    expect[6] = 1
    np.testing.assert_array_equal(psi, expect)


def test_init_random_gaussian_and_normalised(oracle):
    n = 16
    a = oracle.init_random(n, 2024)
    b = oracle.init_random(n, 2024)
    c = oracle.init_random(n, 2025)
    np.testing.assert_array_equal(a, b)
    assert np.abs(a - c).max() > 1e-3
    assert abs(oracle.norm2(a) - 1.0) < 1e-13
    N = 1 << n
    z = a * math.sqrt(N)             # components ~ N(0, 1/2) each
    assert abs(z.real.mean()) < 5 * math.sqrt(0.5 / N)
    assert abs(z.imag.mean()) < 5 * math.sqrt(0.5 / N)
    assert abs(z.real.var() - 0.5) < 0.02 and abs(z.imag.var() - 0.5) < 0.02
    assert abs(np.mean(z.real * z.imag)) < 0.01
    # |z|^2 ~ Exp(1): P(|z|^2 < 1) = 1 - 1/e
    assert abs(np.mean(np.abs(z) ** 2 < 1.0) - (1 - math.exp(-1))) < 0.01
    # Gaussian kurtosis of each component is 3
    k = np.mean(z.real ** 4) / np.mean(z.real ** 2) ** 2
    assert abs(k - 3.0) < 0.1


# ---------------------------------------------------------------- QFT

def alg3_gates(n):
    g = []
    for i in range(n):
        g.append(("H", i, -1, -1, 0.0))
        for j in range(i + 1, n):
            g.append(("CP", i, j, -1, math.pi / 2 ** (j - i)))
    for i in range(n // 2):
        g.append(("SWAP", i, n - 1 - i, -1, 0.0))
    return g


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6])
def test_alg3_equals_qft_definition_matrix(n):
    """Reading A5: Alg. 3 under MSB-first equals the closed form of P:601
    (numerically via the independent matrix route)."""
    assert len(alg3_gates(n)) == W.qft_gate_count(n)
    np.testing.assert_allclose(FM.circuit_unitary(n, alg3_gates(n)), FM.qft_matrix(n), atol=1e-14)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 10])
def test_qft_basis_states_closed_form(oracle, n):
    N = 1 << n
    j = np.arange(N, dtype=np.int64)
    for k in sorted({0, 1, N - 1, N // 3, (5 * N) // 7} & set(range(N))):
        psi = oracle.init_basis(n, k)
        oracle.qft(psi)
        expect = np.exp(2j * np.pi * ((j * k) % N) / N) / math.sqrt(N)
        np.testing.assert_allclose(psi, expect, atol=1e-13)


@pytest.mark.parametrize("n", [4, 9, 12])
def test_qft_random_state_vs_numpy_ifft(oracle, n):
    psi = oracle.init_random(n, 77 + n)
    ref = np.fft.ifft(psi) * math.sqrt(1 << n)
    oracle.qft(psi)
    np.testing.assert_allclose(psi, ref, atol=1e-13)


def test_qft_vs_dft_matrix_and_roundtrip(oracle):
    n = 7
    psi0 = oracle.init_random(n, 5)
    psi = psi0.copy()
    oracle.qft(psi)
    np.testing.assert_allclose(psi, FM.qft_matrix(n) @ psi0, atol=1e-13)
    oracle.qft(psi, inverse=True)
    np.testing.assert_allclose(psi, psi0, atol=1e-13)


# ---------------------------------------------------------------- expectation

def test_expectation_small_closed_forms(oracle):
    psi = oracle.zeros(1)
    assert oracle.expval(psi, [(1.0, 0, 1)]) == 1.0          # <Z> on |0>
    bell = np.array([R2, 0, 0, R2], np.complex128)
    assert oracle.expval(bell, [(1.0, 3, 0)]) == pytest.approx(1.0, abs=1e-15)   # XX
    assert oracle.expval(bell, [(1.0, 3, 3)]) == pytest.approx(-1.0, abs=1e-15)  # YY
    assert oracle.expval(bell, [(1.0, 0, 3)]) == pytest.approx(1.0, abs=1e-15)   # ZZ
    assert oracle.expval(bell, [(1.0, 1, 0)]) == pytest.approx(0.0, abs=1e-15)   # X on q0


@pytest.mark.parametrize("n", [2, 4, 6])
def test_expectation_vs_hamiltonian_matrix(oracle, n):
    rng = np.random.default_rng(500 + n)
    terms = W.random_pauli_sum(n, min(15, 4 ** n - 1), rng)
    psi = rand_state(n, rng)
    Hm = FM.hamiltonian_matrix(n, terms)
    ref = float(np.real(np.vdot(psi, Hm @ psi)))
    assert oracle.expval(psi, terms) == pytest.approx(ref, abs=1e-13)


@pytest.mark.parametrize("n", [6, 8, 10])
def test_xyz_energy_at_theta_zero(oracle, n):
    """SURVEY c.4: ring ansatz at theta = 0 leaves |0...0> (CNOTs act on
    controls = 0), so E = Jz (n-1) + hz n exactly."""
    gates = W.hea_ansatz(n, 2, "ring")
    e = oracle.energy(n, gates, np.zeros(4 * n), W.xyz_terms(n))
    assert e == pytest.approx(0.4 * (n - 1) + 0.3 * n, abs=1e-13)


# ---------------------------------------------------------------- PSR

def test_psr_single_ry_closed_form(oracle):
    """North star: <Z> after RY(t)|0> is cos t; its PSR derivative is -sin t."""
    gates = [("RY", 0, -1, 0, 0.0)]
    for t in [0.0, 0.3, math.pi / 2, 2.0, 5.5]:
        assert oracle.energy(1, gates, [t], [(1.0, 0, 1)]) == pytest.approx(math.cos(t), abs=1e-15)
        g = oracle.param_shift_grad(1, gates, np.array([t]), [(1.0, 0, 1)])
        assert g[0] == pytest.approx(-math.sin(t), abs=1e-15)


@pytest.mark.parametrize("n", [3, 6, 8])
def test_psr_product_ansatz_closed_form(oracle, n):
    rng = np.random.default_rng(600 + n)
    gates, theta = W.product_ansatz(n, rng)
    terms = W.xyz_terms(n)
    E, g = product_energy_and_grad(n, theta)
    assert oracle.energy(n, gates, theta, terms) == pytest.approx(E, abs=1e-13)
    np.testing.assert_allclose(oracle.param_shift_grad(n, gates, theta, terms, threads=4), g,
                               atol=1e-13)


def test_psr_matches_central_difference_cfg3(oracle):
    """PSR vs central finite difference on config 3."""
    w = W.config3()
    g = oracle.param_shift_grad(w.n, w.gates, w.theta, w.terms)
    h = 1e-5
    fd = np.zeros_like(g)
    for p in range(w.theta.size):
        tp, tm = w.theta.copy(), w.theta.copy()
        tp[p] += h
        tm[p] -= h
        fd[p] = (oracle.energy(w.n, w.gates, tp, w.terms) - oracle.energy(w.n, w.gates, tm, w.terms)) / (2 * h)
    np.testing.assert_allclose(g, fd, atol=1e-8)


def test_psr_vs_matrix_route_gradient(oracle):
    """Exact derivative through the matrix route: d/dt <0|U(t)^+ H U(t)|0>
    with dU from the generator, n = 3 ring ansatz."""
    n = 3
    rng = np.random.default_rng(9)
    gates = W.hea_ansatz(n, 2, "ring")
    theta = rng.uniform(0, 2 * np.pi, 4 * n)
    terms = W.random_pauli_sum(n, 10, rng)
    Hm = FM.hamiltonian_matrix(n, terms)
    gens = {"RX": FM.X, "RY": FM.Y, "RZ": FM.Z}
    psi0 = np.zeros(1 << n, np.complex128)
    psi0[0] = 1
    exact = np.zeros(theta.size)
    for k, (name, a, b, p, _) in enumerate(gates):
        if p < 0:
            continue
        pre = FM.circuit_unitary(n, gates[:k + 1], theta)
        post = FM.circuit_unitary(n, gates[k + 1:], theta)
        G = FM.embed(n, {a: gens[name]})
        dpsi = post @ (-0.5j * G) @ pre @ psi0
        psi = post @ pre @ psi0
        exact[p] = 2 * np.real(np.vdot(psi, Hm @ dpsi))
    g = oracle.param_shift_grad(n, gates, theta, terms)
    np.testing.assert_allclose(g, exact, atol=1e-13)


def test_psr_cry_closed_form_four_term(oracle):
    """Reading A8 (f3): after H(0), CRY(t; 0 -> 1) the state is
    (|00> + cos(t/2)|10> + sin(t/2)|11>)/sqrt2, so <X_0> = cos(t/2) and
    dE/dt = -sin(t/2)/2 exactly.  The paper's two-term rule would give
    -(sqrt2/2) sin(t/2) here (E carries frequency 1/2); the four-term rule
    must reproduce the exact derivative."""
    gates = [("H", 0, -1, -1, 0.0), ("CRY", 0, 1, 0, 0.0)]
    for t in [0.0, 0.4, 1.3, math.pi / 2, 2.9, 5.1]:
        assert oracle.energy(2, gates, [t], [(1.0, 1, 0)]) == pytest.approx(math.cos(t / 2), abs=1e-15)
        g = oracle.param_shift_grad(2, gates, np.array([t]), [(1.0, 1, 0)])
        assert g[0] == pytest.approx(-math.sin(t / 2) / 2, abs=1e-15)
        if abs(math.sin(t / 2)) > 0.1:   # the two-term value is really different
            assert abs(g[0] - (-math.sqrt(2) / 2 * math.sin(t / 2))) > 1e-2


def test_psr_cry_vs_matrix_route_gradient(oracle):
    """Exact derivative through the matrix route for a circuit mixing RX/RY/RZ
    and CRY parameters: CRY(t) = exp(-i t G / 2), G = |1><1|_c (x) Y_t."""
    n = 3
    rng = np.random.default_rng(77)
    gates = [("RY", 0, -1, 0, 0.0), ("RX", 1, -1, 1, 0.0), ("H", 2, -1, -1, 0.0),
             ("CRY", 0, 1, 2, 0.0), ("CNOT", 1, 2, -1, 0.0), ("CRY", 2, 0, 3, 0.0),
             ("RZ", 1, -1, 4, 0.0), ("CRY", 1, 2, 5, 0.0), ("RY", 2, -1, 6, 0.0)]
    theta = rng.uniform(0, 2 * np.pi, 7)
    terms = W.random_pauli_sum(n, 12, rng)
    Hm = FM.hamiltonian_matrix(n, terms)
    psi0 = np.zeros(1 << n, np.complex128)
    psi0[0] = 1
    exact = np.zeros(theta.size)
    for k, (name, a, b, p, _) in enumerate(gates):
        if p < 0:
            continue
        pre = FM.circuit_unitary(n, gates[:k + 1], theta)
        post = FM.circuit_unitary(n, gates[k + 1:], theta)
        G = FM.embed(n, {a: FM.P1, b: FM.Y}) if name == "CRY" else FM.embed(n, {a: {"RX": FM.X, "RY": FM.Y, "RZ": FM.Z}[name]})
        dpsi = post @ (-0.5j * G) @ pre @ psi0
        exact[p] = 2 * np.real(np.vdot(post @ pre @ psi0, Hm @ dpsi))
    g = oracle.param_shift_grad(n, gates, theta, terms)
    np.testing.assert_allclose(g, exact, atol=1e-13)


def test_expval_rejects_non_hermitian_imag(oracle):
    """a non-real <P> is an error, never silent.  A Pauli
    product is Hermitian, so <psi|P|psi> is real for every finite psi: the
    check fires only on a corrupted state buffer (NaN / Inf), which must be
    rejected rather than summed."""
    psi = np.array([1, 1j], np.complex128) / math.sqrt(2)
    # <Y> on (|0> + i|1>)/sqrt2 = 1 (real) -- must pass
    assert oracle.expval(psi, [(1.0, 1, 1)]) == pytest.approx(1.0)
    for bad in (complex(np.nan, 0.0), complex(0.0, np.inf), complex(np.inf, np.nan)):
        psi2 = psi.copy()
        psi2[1] = bad
        for term in ((1.0, 1, 1), (1.0, 1, 0), (1.0, 0, 1)):
            with pytest.raises(oracle.OracleError):
                oracle.expval(psi2, [term])


def test_splitmix64_published_vector(oracle):
    """The counter hash of init_random is Vigna's
    SplitMix64 output function: seeded with 1234567 the generator's first
    five outputs (state advanced by the golden gamma 0x9E3779B97F4A7C15 each
    step, i.e. splitmix64(seed + k*gamma)) are the published test vector."""
    gamma = 0x9E3779B97F4A7C15
    want = [6457827717110365317, 3203168211198807973, 9817491932198370423,
            4593380528125082431, 16408922859458223821]
    got = [oracle.splitmix64((1234567 + k * gamma) % 2**64) for k in range(5)]
    assert got == want


def test_uniform_deviate_endpoints(oracle):
    """u = ((x >> 11) + 0.5) 2^-53 (c.1 step 2) at the ends of its range: the
    cell midpoints 2^-54 and 1 - 2^-54 (u is never 0, so ln u0 is finite),
    and 1/2 + 2^-54 at x = 2^63."""
    assert oracle.u53(0) == 2.0 ** -54
    assert oracle.u53(2**64 - 1) == 1.0 - 2.0 ** -54
    assert oracle.u53(2**63) == 0.5 + 2.0 ** -54
    assert oracle.u53(2**11 - 1) == 2.0 ** -54     # the low 11 bits are dropped


def test_init_random_hand_computed_amplitudes(oracle):
    """init_random(n, seed)[i] = a_i / sqrt(sum_j |a_j|^2) with
    a_i = sqrt(-2 ln u0) e^{2 pi i u1}, u = ((x >> 11) + 0.5) 2^-53,
    x0 = splitmix64(seed ^ 2i), x1 = splitmix64(seed ^ (2i+1)) (c.1 step 2),
    computed here by hand from the pinned hash for n = 3 (all 8 amplitudes,
    so the normalisation is explicit too).  Catches a seed-convention slip
    such as seed ^ i, a swapped u0/u1 or a dropped +0.5."""
    n, seed = 3, 0xDEADBEEF12345678
    a = []
    for i in range(1 << n):
        x0, x1 = oracle.splitmix64(seed ^ (2 * i)), oracle.splitmix64(seed ^ (2 * i + 1))
        u0, u1 = ((x0 >> 11) + 0.5) * 2.0 ** -53, ((x1 >> 11) + 0.5) * 2.0 ** -53
        r = math.sqrt(-2.0 * math.log(u0))
        a.append(complex(r * math.cos(2 * math.pi * u1), r * math.sin(2 * math.pi * u1)))
    a = np.array(a)
    want = a / math.sqrt(float(np.sum(np.abs(a) ** 2)))
    got = oracle.init_random(n, seed)
    assert np.abs(got - want).max() <= 1e-15
    # the per-index route used for states too large for the host
    idx = np.array([5, 0, 7], np.uint64)
    np.testing.assert_allclose(oracle.random_gaussian_at(seed, idx), a[[5, 0, 7]], rtol=0, atol=1e-15)
    big = oracle.init_random(12, 77)
    raw = oracle.random_gaussian_at(77, np.arange(1 << 12, dtype=np.uint64))
    assert np.abs(big - raw / math.sqrt(float(np.sum(np.abs(raw) ** 2)))).max() <= 1e-15


# ---------------------------------------------------------------- VQE outer loop (f2)

def test_vqe_first_adam_step_closed_form(oracle):
    """At t = 1 the bias-corrected moments are m_hat = g, v_hat = g^2, so the
    first update is theta_1 = theta_0 - lr g / (|g| + eps) componentwise
    (sign descent of size lr) -- a property of Adam, not a retyping of it."""
    w = W.config3()
    th1, trace, T = oracle.vqe_adam(w.n, w.gates, w.theta, w.terms, max_iter=1)
    g0 = oracle.param_shift_grad(w.n, w.gates, w.theta, w.terms)
    assert T == 1 and trace.size == 2
    np.testing.assert_allclose(th1, w.theta - 1e-2 * g0 / (np.abs(g0) + 1e-8), rtol=0, atol=1e-15)
    assert trace[0] == pytest.approx(oracle.energy(w.n, w.gates, w.theta, w.terms), abs=0)
    assert trace[1] == pytest.approx(oracle.energy(w.n, w.gates, th1, w.terms), abs=0)


def test_vqe_single_qubit_converges_to_ground_state(oracle):
    """H = Z, ansatz RY(theta), theta_0 = 0.1: E = cos theta has
    its minimum -1 at theta = pi (ground state |1>)."""
    th, trace, T = oracle.vqe_adam(1, [("RY", 0, -1, 0, 0.0)], [0.1], [(1.0, 0, 1)], lr=0.05, tol=1e-12,
                                   max_iter=3000)
    assert trace[-1] == pytest.approx(-1.0, abs=1e-6)
    assert abs(math.cos(th[0]) - trace[-1]) < 1e-15
    assert trace[0] == pytest.approx(math.cos(0.1), abs=1e-15)


def test_vqe_zero_hamiltonian_converges_at_once(oracle):
    """a zero-term Hamiltonian gives E = 0 and g = 0, so Adam's
    moments stay 0, theta is unchanged and |E_1 - E_0| = 0 < tol stops the loop."""
    w = W.config3()
    th, trace, T = oracle.vqe_adam(w.n, w.gates, w.theta, [], max_iter=10)
    assert T == 1 and np.all(trace == 0.0)
    np.testing.assert_array_equal(th, w.theta)


def test_vqe_config3_energy_decreases(oracle):
    """Descent: with lr = 1e-2 the config-3 energy trace falls over 25 steps."""
    w = W.config3()
    th, trace, T = oracle.vqe_adam(w.n, w.gates, w.theta, w.terms, max_iter=25)
    assert T == 25 and trace[-1] < trace[0] - 0.05


# ---------------------------------------------------------------- Trotter XYZ (f1)

def test_trotter_diagonal_chain_closed_form(oracle):
    """with Jx = Jy = 0 the Hamiltonian is diagonal and |1...1>
    stays an eigenstate: <Z_i Z_{i+1}> = 1, <Z_i> = -1, so
    E(t) = -Jz (n-1) + n h(t) exactly at every recorded time."""
    n, jz, A, w = 6, 1.0, 2.0, 1.0
    psi = oracle.init_basis(n, (1 << n) - 1)
    E = oracle.trotter_xyz(psi, 0.0, 0.0, jz, A, w, 0.0, 0.05, 40, record_every=4)
    t = 0.05 * 4 * np.arange(E.size)
    np.testing.assert_allclose(E, -jz * (n - 1) + n * A * np.sin(w * t), rtol=0, atol=1e-13)
    assert abs(oracle.norm2(psi) - 1) < 1e-13


def _expm_reference(oracle, n, jx, jy, jz, A, w, t0, dt, steps):
    """Piecewise-constant exact propagator: prod_j exp(-i H(t_j) dt) through
    dense matrices (fullmatrix route + scipy expm), from |1...1>."""
    from scipy.linalg import expm
    psi = np.zeros(1 << n, np.complex128)
    psi[-1] = 1.0
    for j in range(steps):
        Hm = FM.hamiltonian_matrix(n, oracle.xyz_hamiltonian(n, jx, jy, jz, A * math.sin(w * (t0 + j * dt))))
        psi = expm(-1j * dt * Hm) @ psi
    return psi


def test_trotter_first_order_error_ratio(oracle):
    """halving dt halves the first-order Trotter error against
    the exact piecewise-constant propagator (ratio in [1.7, 2.3]), N = 4."""
    n, T = 4, 1.0
    errs = []
    for steps in (50, 100):
        dt = T / steps
        psi = oracle.init_basis(n, (1 << n) - 1)
        oracle.trotter_xyz(psi, 1.0, 0.7, 0.4, 2.0, 1.0, 0.0, dt, steps, record_every=steps)
        ref = _expm_reference(oracle, n, 1.0, 0.7, 0.4, 2.0, 1.0, 0.0, dt, steps)
        errs.append(np.abs(psi - ref).max())
    assert 1.7 <= errs[0] / errs[1] <= 2.3, errs
    assert errs[1] < 1e-2


def test_trotter_small_step_and_static_drift(oracle):
    """One step with dt -> 0 is the identity to O(dt); with A = 0 the energy
    drift over a fixed time shrinks with dt."""
    n = 5
    psi = oracle.init_random(n, 3)
    ref = psi.copy()
    oracle.trotter_xyz(psi, 1.0, 0.7, 0.4, 2.0, 1.0, 0.3, 1e-6, 1)
    assert 0 < np.abs(psi - ref).max() < 1e-5
    drift = []
    for steps in (20, 80):
        psi = oracle.init_random(n, 4)
        E = oracle.trotter_xyz(psi, 1.0, 0.7, 0.4, 0.0, 1.0, 0.0, 1.0 / steps, steps, record_every=steps)
        drift.append(abs(E[-1] - E[0]))
    assert drift[1] < drift[0]


def test_monomial_closed_forms_match_oracle(oracle):
    """The monomial trackers used by the full-scale sharded GPU tests (c.4 (i),
    (vi)) agree with the oracle at n = 8 (forward map + QFT closed form,
    inverse circuit, backward walk after a 1q layer)."""
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from closed_forms import monomial_backward, monomial_forward, monomial_inverse, qft_of_basis
    n = 8
    rng = np.random.default_rng(1)
    g = W.monomial_circuit(n, 200, rng, global_qubits=1, p_global=0.3)
    k = 77
    kp, ph = monomial_forward(n, g, k)
    psi = oracle.init_basis(n, k)
    oracle.apply_circuit(psi, g)
    assert abs(psi[kp] - ph) < 1e-14 and abs(np.abs(psi).sum() - 1) < 1e-14
    oracle.qft(psi)
    assert np.abs(psi - ph * qft_of_basis(n, kp, np.arange(1 << n))).max() < 1e-14
    oracle.qft(psi, inverse=True)
    oracle.apply_circuit(psi, monomial_inverse(g))
    assert abs(psi[k] - 1) < 1e-13
    layer, col = [], []
    for q in range(n):
        kind, t = ["H", "RX", "RY"][q % 3], 0.3 + q
        layer.append((kind, q, -1, -1, t if kind != "H" else 0.0))
        c, s = np.cos(t / 2), np.sin(t / 2)
        col.append({"H": (1 / np.sqrt(2), 1 / np.sqrt(2)), "RX": (c, -1j * s), "RY": (c, s)}[kind])
    psi = oracle.init_basis(n, 0)
    oracle.apply_circuit(psi, layer + g)
    for j in range(1 << n):
        kk, ph = monomial_backward(n, g, j)
        a = ph
        for q in range(n):
            a *= col[q][(kk >> (n - 1 - q)) & 1]
        assert abs(psi[j] - a) < 1e-14


def test_circuit_inverse_helper_is_identity(oracle):
    """The test helper used by the full-size round trips: C^-1 C = I on the
    config-5 alphabet (oracle at n = 8)."""
    from closed_forms import circuit_inverse
    import workloads as W
    w = W.config5(n=8, m=2, n_gates=300)
    psi = oracle.init_random(8, w.seed)
    ref = psi.copy()
    oracle.apply_circuit(psi, w.gates)
    assert np.abs(psi - ref).max() > 1e-3
    oracle.apply_circuit(psi, circuit_inverse(w.gates))
    assert np.abs(psi - ref).max() <= 1e-13
