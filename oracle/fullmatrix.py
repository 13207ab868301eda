"""Matrix-based route (explicit 2^n x 2^n unitaries).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  An independent second
implementation used to pin the bitwise C oracle for n <= 6: every gate becomes
a full 2^n x 2^n matrix built from Kronecker products of single-qubit
operators, qubit 0 being the leftmost (most significant) factor (MSB-first,
PAPER.md:579).  Controlled gates are built from projectors
|0><0| (x) I + |1><1| (x) U; two-qubit matrices are expanded as
sum_{rk} U[r,k] |r_a><k_a| (x) |r_b><k_b| with q0 the high sub-index bit
(reading A2).  Nothing here shares code with oracle.c.
"""
from __future__ import annotations

import numpy as np

I2 = np.eye(2, dtype=np.complex128)
X = np.array([[0, 1], [1, 0]], np.complex128)
Y = np.array([[0, -1j], [1j, 0]], np.complex128)
Z = np.array([[1, 0], [0, -1]], np.complex128)
H = np.array([[1, 1], [1, -1]], np.complex128) / np.sqrt(2.0)
S = np.diag([1, 1j]).astype(np.complex128)
T = np.diag([1, np.exp(1j * np.pi / 4)]).astype(np.complex128)
P0 = np.diag([1, 0]).astype(np.complex128)
P1 = np.diag([0, 1]).astype(np.complex128)


def _expm_pauli(G: np.ndarray, theta: float) -> np.ndarray:
    """exp(-i theta G / 2) for an involutory G, via its eigendecomposition
    (numpy.linalg.eigh) rather than the cos/sin closed form."""
    w, v = np.linalg.eigh(G)
    return (v * np.exp(-0.5j * theta * w)) @ v.conj().T


def one_qubit_matrix(name: str, angle: float = 0.0) -> np.ndarray:
    table = {"H": H, "X": X, "Y": Y, "Z": Z, "S": S, "SDG": S.conj().T,
             "T": T, "TDG": T.conj().T}
    if name in table:
        return table[name]
    if name in ("RX", "RY", "RZ"):
        return _expm_pauli({"RX": X, "RY": Y, "RZ": Z}[name], angle)
    raise KeyError(name)


def embed(n: int, ops: dict) -> np.ndarray:
    """kron over qubits 0..n-1 (qubit 0 leftmost) of ops.get(q, I)."""
    M = np.array([[1.0 + 0j]])
    for q in range(n):
        M = np.kron(M, ops.get(q, I2))
    return M


def controlled(n: int, c: int, t: int, U: np.ndarray) -> np.ndarray:
    return embed(n, {c: P0}) + embed(n, {c: P1, t: U})


def two_qubit_full(n: int, a: int, b: int, U4: np.ndarray) -> np.ndarray:
    M = np.zeros((1 << n, 1 << n), np.complex128)
    for r in range(4):
        for k in range(4):
            if U4[r, k] == 0:
                continue
            Ea = np.zeros((2, 2), np.complex128)
            Eb = np.zeros((2, 2), np.complex128)
            Ea[r >> 1, k >> 1] = 1
            Eb[r & 1, k & 1] = 1
            M += U4[r, k] * embed(n, {a: Ea, b: Eb})
    return M


def gate_unitary(n: int, gate: tuple, theta=None) -> np.ndarray:
    name, a, b, p, ang = gate[:5]
    angle = theta[p] if p is not None and p >= 0 else ang
    if name in ("H", "X", "Y", "Z", "S", "SDG", "T", "TDG", "RX", "RY", "RZ"):
        return embed(n, {a: one_qubit_matrix(name, angle)})
    if name == "U1":
        return embed(n, {a: np.asarray(gate[5], np.complex128).reshape(2, 2)})
    if name == "CNOT":
        return controlled(n, a, b, X)
    if name == "CZ":
        return controlled(n, a, b, Z)
    if name == "CP":
        return controlled(n, a, b, np.diag([1, np.exp(1j * angle)]))
    if name == "CRY":
        return controlled(n, a, b, one_qubit_matrix("RY", angle))
    if name == "SWAP":
        return sum(embed(n, {a: A, b: B}) for A, B in
                   [(I2, I2), (X, X), (Y, Y), (Z, Z)]) / 2.0
    if name == "U2":
        return two_qubit_full(n, a, b, np.asarray(gate[5], np.complex128).reshape(4, 4))
    if name in ("RXX", "RYY", "RZZ"):
        P = {"RXX": X, "RYY": Y, "RZZ": Z}[name]
        return _expm_pauli(embed(n, {a: P, b: P}), angle)
    if name == "CCX":
        c2 = gate[6]
        return (np.eye(1 << n) - embed(n, {a: P1, b: P1})
                + embed(n, {a: P1, b: P1, c2: X}))
    raise KeyError(name)


def circuit_unitary(n: int, gates, theta=None) -> np.ndarray:
    U = np.eye(1 << n, dtype=np.complex128)
    for g in gates:
        U = gate_unitary(n, g, theta) @ U
    return U


def qft_matrix(n: int) -> np.ndarray:
    """F[k, x] = N^-1/2 e^{2 pi i x k / N}, with the phase
    reduced exactly as (x k mod N) before exponentiation."""
    N = 1 << n
    x = np.arange(N, dtype=np.int64)
    return np.exp(2j * np.pi * ((np.outer(x, x) % N) / N)) / np.sqrt(N)


def pauli_matrix(n: int, x_mask: int, z_mask: int) -> np.ndarray:
    ops = {}
    for q in range(n):
        xb, zb = (x_mask >> q) & 1, (z_mask >> q) & 1
        if xb or zb:
            ops[q] = Y if (xb and zb) else (X if xb else Z)
    return embed(n, ops)


def hamiltonian_matrix(n: int, terms) -> np.ndarray:
    return sum(c * pauli_matrix(n, x, z) for c, x, z in terms)
