"""Seeded synthetic inputs for the five BASELINE.json configs.

This module is the ONLY code shared by the oracle (``oracle/``) and the CUDA
path (``paper_2512_23183_b200``).  It holds no arithmetic of the method: it
only draws gate kinds, qubit indices, angles, Pauli strings, coefficients,
basis indices and seeds, and spells out the circuit *structure* the configs
name.  Gates are plain tuples ``(name, q0, q1, param_idx, angle)``; each side
maps names to its own codes and matrices.

Conventions:
  * qubit q <-> amplitude-index bit n-1-q (MSB-first, Alg. 1).
  * Pauli term = (coeff, x_mask, z_mask) with bit q of a mask = qubit q;
    Y on qubit q sets both bits (P = prod_q X^x Z^z up to i^{|x&z|}).
  * param_idx >= 0 means "angle = theta[param_idx]" (ansatz gates, D9/D10);
    param_idx = -1 means the literal ``angle`` is used (0.0 for fixed gates).

Seeds: base seed 251223183; per config
``numpy.random.SeedSequence(251223183 + cfg).spawn(5)`` gives independent
streams for (state, circuit kinds/qubits, angles/params, coefficients/strings,
basis indices), each through ``default_rng`` (PCG64).  ``init_random`` takes
the state stream's first uint64.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

BASE_SEED = 251223183

Gate = Tuple[str, int, int, int, float]   # (name, q0, q1, param_idx, angle)
Term = Tuple[float, int, int]             # (coeff, x_mask, z_mask)

ONE_QUBIT_FIXED = ("H", "X", "Y", "Z", "S", "SDG", "T", "TDG")
ROTATIONS = ("RX", "RY", "RZ")
TWO_QUBIT = ("CNOT", "CZ", "CP", "SWAP", "CRY")
# config 1 gate alphabet (BASELINE.json configs[0]); reading A12
CFG1_KINDS = ("H", "X", "Y", "Z", "S", "T", "RX", "RY", "RZ", "CNOT", "CZ")
# config 5 alphabet: the 1q/2q kinds of config 1 (reading A13)
CFG5_KINDS = CFG1_KINDS
PARAMETRIC = ("RX", "RY", "RZ", "CP", "CRY", "RXX", "RYY", "RZZ")


def streams(cfg: int):
    """The five independent PCG64 streams of config ``cfg`` (1-based)."""
    ss = np.random.SeedSequence(BASE_SEED + cfg).spawn(5)
    return [np.random.default_rng(s) for s in ss]


def state_seed(cfg: int) -> int:
    return int(streams(cfg)[0].integers(0, 2**64, dtype=np.uint64))


@dataclass
class Workload:
    name: str
    n: int
    gates: List[Gate] = field(default_factory=list)
    theta: Optional[np.ndarray] = None
    terms: List[Term] = field(default_factory=list)
    seed: Optional[int] = None          # init_random seed (None = |0...0>)
    basis: List[int] = field(default_factory=list)
    qft: bool = False                   # full QFT appended after `gates`
    meta: dict = field(default_factory=dict)


def pauli_word_to_masks(word: str) -> Tuple[int, int]:
    """MSB-first word over IXYZ: char i acts on qubit i."""
    x = z = 0
    for q, ch in enumerate(word):
        if ch in "XY":
            x |= 1 << q
        if ch in "ZY":
            z |= 1 << q
        if ch not in "IXYZ":
            raise ValueError(f"bad Pauli letter {ch!r}")
    return x, z


def masks_to_pauli_word(n: int, x: int, z: int) -> str:
    out = []
    for q in range(n):
        xb, zb = (x >> q) & 1, (z >> q) & 1
        out.append("IXZY"[xb + 2 * zb])
    return "".join(out)


def random_circuit(n: int, n_gates: int, rng_kind, rng_angle, kinds=CFG1_KINDS,
                   global_qubits: int = 0, p_global: float = 0.0) -> List[Gate]:
    """Reading A12/A13: kind uniform over ``kinds``; 1q qubit uniform; 2q an
    ordered pair of distinct qubits; theta ~ U[0, 2pi) for RX/RY/RZ.
    With ``global_qubits`` = m > 0, each gate with prob ``p_global`` draws its
    (first) qubit from {0..m-1} and a 2q partner uniformly from the other n-1
    qubits (random control/target order); otherwise all qubits come from
    {m..n-1}."""
    gates: List[Gate] = []
    m = global_qubits
    for _ in range(n_gates):
        kind = kinds[int(rng_kind.integers(0, len(kinds)))]
        two = kind in TWO_QUBIT
        if m > 0:
            on_global = bool(rng_kind.random() < p_global)
            if on_global:
                a = int(rng_kind.integers(0, m))
                if two:
                    b = int(rng_kind.integers(0, n - 1))
                    b = b + 1 if b >= a else b
                    if rng_kind.random() < 0.5:
                        a, b = b, a
                else:
                    b = -1
            else:
                a = int(rng_kind.integers(m, n))
                if two:
                    b = int(rng_kind.integers(m, n - 1))
                    b = b + 1 if b >= a else b
                else:
                    b = -1
        else:
            a = int(rng_kind.integers(0, n))
            if two:
                b = int(rng_kind.integers(0, n - 1))
                b = b + 1 if b >= a else b
            else:
                b = -1
        angle = float(rng_angle.uniform(0.0, 2.0 * math.pi)) if kind in ROTATIONS else 0.0
        gates.append((kind, a, b, -1, angle))
    return gates


def hea_ansatz(n: int, layers: int, entangler: str = "ladder") -> List[Gate]:
    """Reading A14: per layer RY(q) q=0..n-1, then RZ(q), then CNOT(q,q+1)
    for q=0..n-2 (ladder) or CNOT(q,(q+1) mod n) for q=0..n-1 (ring).
    theta index = layer*2n + q (RY), layer*2n + n + q (RZ).  P:739-750."""
    gates: List[Gate] = []
    for l in range(layers):
        for q in range(n):
            gates.append(("RY", q, -1, l * 2 * n + q, 0.0))
        for q in range(n):
            gates.append(("RZ", q, -1, l * 2 * n + n + q, 0.0))
        if entangler == "ladder":
            pairs = [(q, q + 1) for q in range(n - 1)]
        elif entangler == "ring":
            pairs = [(q, (q + 1) % n) for q in range(n)] if n > 2 else [(0, 1)]
        else:
            raise ValueError(entangler)
        for a, b in pairs:
            gates.append(("CNOT", a, b, -1, 0.0))
    return gates


def xyz_terms(n: int, jx=1.0, jy=0.7, jz=0.4, hz=0.3) -> List[Term]:
    """Reading A9/A10: open chain H = sum_{i<n-1} (Jx XX + Jy YY + Jz ZZ)_{i,i+1}
    + hz sum_i Z_i; 3(n-1) + n terms (93 at n=24).  Term order: all XX, all YY,
    all ZZ, all Z."""
    terms: List[Term] = []
    for i in range(n - 1):
        m = (1 << i) | (1 << (i + 1))
        terms.append((jx, m, 0))
    for i in range(n - 1):
        m = (1 << i) | (1 << (i + 1))
        terms.append((jy, m, m))
    for i in range(n - 1):
        m = (1 << i) | (1 << (i + 1))
        terms.append((jz, 0, m))
    for i in range(n):
        terms.append((hz, 0, 1 << i))
    return terms


def random_pauli_sum(n: int, n_terms: int, rng, sigma: float = 0.5) -> List[Term]:
    """Reading A11: ``n_terms`` DISTINCT strings uniform over {I,X,Y,Z}^n
    (identity allowed), coefficients ~ N(0, sigma)."""
    seen = set()
    words = []
    while len(words) < n_terms:
        w = "".join("IXYZ"[int(i)] for i in rng.integers(0, 4, size=n))
        if w not in seen:
            seen.add(w)
            words.append(w)
    coeffs = rng.normal(0.0, sigma, size=n_terms)
    out = []
    for c, w in zip(coeffs, words):
        x, z = pauli_word_to_masks(w)
        out.append((float(c), x, z))
    return out


def qft_gate_count(n: int) -> int:
    """Alg. 3 gate count n + n(n-1)/2 + floor(n/2), used for the
    updates/s metric."""
    return n + n * (n - 1) // 2 + n // 2


# --------------------------------------------------------------------------
# The five configs
# --------------------------------------------------------------------------

def config1(n: int = 10, n_gates: int = 200) -> Workload:
    s_state, s_circ, s_ang, _, _ = streams(1)
    seed = int(s_state.integers(0, 2**64, dtype=np.uint64))
    gates = random_circuit(n, n_gates, s_circ, s_ang)
    return Workload("cfg1_random_n10_qft", n, gates=gates, seed=seed, qft=True)


def config2(n: int = 20, n_basis: int = 16) -> Workload:
    s_state, _, _, _, s_basis = streams(2)
    seed = int(s_state.integers(0, 2**64, dtype=np.uint64))
    basis: List[int] = []
    while len(basis) < n_basis:
        k = int(s_basis.integers(0, 2**n))
        if k not in basis:
            basis.append(k)
    return Workload("cfg2_qft_n20", n, seed=seed, basis=basis, qft=True)


def config3(n: int = 4, layers: int = 6, n_terms: int = 15) -> Workload:
    _, _, s_par, s_coef, _ = streams(3)
    gates = hea_ansatz(n, layers, "ladder")
    theta = s_par.uniform(0.0, 2.0 * math.pi, size=layers * 2 * n)
    terms = random_pauli_sum(n, n_terms, s_coef, 0.5)
    return Workload("cfg3_vqe_n4", n, gates=gates, theta=theta, terms=terms)


def config4(n: int = 24, layers: int = 10) -> Workload:
    _, _, s_par, _, s_idx = streams(4)
    gates = hea_ansatz(n, layers, "ring")
    theta = s_par.uniform(0.0, 2.0 * math.pi, size=layers * 2 * n)
    terms = xyz_terms(n)
    # seeded subset of gradient components the oracle checks
    sample = sorted(int(i) for i in s_idx.choice(layers * 2 * n, size=8, replace=False))
    return Workload("cfg4_xyz_psr_n24", n, gates=gates, theta=theta, terms=terms,
                    meta={"oracle_params": sample})


def config5(n: int = 34, m: int = 1, n_gates: int = 1000) -> Workload:
    """n=34 @ G=2 (m=1), n=36 @ G=8 (m=3); reduced twins reuse m (A13)."""
    s_state, s_circ, s_ang, _, _ = streams(5)
    seed = int(s_state.integers(0, 2**64, dtype=np.uint64))
    gates = random_circuit(n, n_gates, s_circ, s_ang, kinds=CFG5_KINDS,
                           global_qubits=m, p_global=0.3)
    return Workload(f"cfg5_sharded_n{n}_m{m}", n, gates=gates, seed=seed, qft=True,
                    meta={"m": m})


def product_ansatz(n: int, rng) -> Tuple[List[Gate], np.ndarray]:
    """Closed-form family: one layer RY(theta_q) then
    RZ(phi_q) on every qubit, no entanglers.  theta index q (RY), n+q (RZ)."""
    gates: List[Gate] = [("RY", q, -1, q, 0.0) for q in range(n)]
    gates += [("RZ", q, -1, n + q, 0.0) for q in range(n)]
    theta = rng.uniform(0.0, 2.0 * math.pi, size=2 * n)
    return gates, theta


def monomial_circuit(n: int, n_gates: int, rng, global_qubits: int = 0,
                     p_global: float = 0.0) -> List[Gate]:
    """Closed-form family (c.4 (i)): only X, Y, Z, S, T, RZ, CNOT, CZ."""
    kinds = ("X", "Y", "Z", "S", "T", "RZ", "CNOT", "CZ")
    return random_circuit(n, n_gates, rng, rng, kinds=kinds,
                          global_qubits=global_qubits, p_global=p_global)


def edge_case_circuit() -> List[Gate]:
    """PAPER.md App. E test circuit (wiring S:449-457):
    RX(t0) q0, RY(t1) q1, RZ(t2) q0, CNOT(0->1), CRY(t3; control 1 -> target 0);
    observable <Z_0>."""
    return [("RX", 0, -1, 0, 0.0), ("RY", 1, -1, 1, 0.0), ("RZ", 0, -1, 2, 0.0),
            ("CNOT", 0, 1, -1, 0.0), ("CRY", 1, 0, 3, 0.0)]


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}
