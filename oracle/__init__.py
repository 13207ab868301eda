"""Plain CPU oracle for the LogosQ dense state-vector hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` leg / ``--impl reference`` arm may import this
package.  The product (``paper_2512_23183_b200``) never imports it and shares
no code with it; both read their inputs from ``workloads`` only.

``oracle.c`` holds the arithmetic (each function cites the PAPER.md passage it
follows); this module only marshals numpy arrays through ctypes and runs
independent circuits on several host threads (ctypes releases the GIL), which
is parallelism *across* circuits only, never inside one.

``fullmatrix.py`` is the second, independent route (explicit 2^n x 2^n
Kronecker-product unitaries, "matrix-based") used to pin the C
oracle at n <= 6.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from typing import Iterable, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# Oracle-private codes; must match the enum in oracle.c.
KINDS = {name: i for i, name in enumerate(
    ["H", "X", "Y", "Z", "S", "SDG", "T", "TDG", "RX", "RY", "RZ",
     "CNOT", "CZ", "CP", "SWAP", "U1", "U2", "CRY", "CCX", "RXX", "RYY", "RZZ"])}


def build(force: bool = False) -> str:
    """Compile oracle.c with plain gcc -O2 (no fast-math, no vector intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared",
                               "-fno-fast-math", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i32, u64, dbl = ctypes.c_int, ctypes.c_uint64, ctypes.c_double
        _lib.or_init_basis.argtypes = [P, i32, u64]
        _lib.or_init_random.argtypes = [P, i32, u64]
        _lib.or_apply_gate.argtypes = [P, i32, i32, i32, i32, i32, dbl, P]
        _lib.or_apply_circuit.argtypes = [P, i32, i32, P, P, P, P, P, P, P, P]
        _lib.or_qft.argtypes = [P, i32, i32]
        _lib.or_expval.argtypes = [P, i32, i32, P, P, P, P]
        _lib.or_energy.argtypes = [i32, i32, P, P, P, P, P, P, P, P, i32, P, P, P, P]
        _lib.or_param_shift.argtypes = [i32, i32, P, P, P, P, P, P, P, P, i32, i32,
                                        P, P, P, P, i32, P]
        _lib.or_splitmix64.argtypes = [u64]
        _lib.or_splitmix64.restype = u64
        _lib.or_random_gaussian_at.argtypes = [u64, P, u64, P]
        _lib.or_u53.argtypes = [u64]
        _lib.or_u53.restype = dbl
        _lib.or_norm2.argtypes = [P, i32]
        _lib.or_norm2.restype = dbl
    return _lib


class OracleError(RuntimeError):
    pass


def _check(rc: int):
    if rc != 0:
        raise OracleError({-1: "bad argument", -2: "non-real expectation",
                           -3: "out of memory"}.get(rc, f"error {rc}"))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _state(psi: np.ndarray) -> np.ndarray:
    if psi.dtype != np.complex128 or not psi.flags.c_contiguous:
        raise TypeError("oracle states are C-contiguous complex128 arrays")
    return psi


class _Circuit:
    """Gate list marshalled to parallel arrays.  Gate tuples are
    (name, q0, q1, param_idx, angle[, mat][, q2])."""

    def __init__(self, gates: Sequence[tuple]):
        g = len(gates)
        self.n_gates = g
        self.kinds = np.zeros(max(g, 1), np.int32)
        self.q0 = np.full(max(g, 1), -1, np.int32)
        self.q1 = np.full(max(g, 1), -1, np.int32)
        self.q2 = np.full(max(g, 1), -1, np.int32)
        self.pidx = np.full(max(g, 1), -1, np.int32)
        self.angles = np.zeros(max(g, 1), np.float64)
        self.mats = np.zeros((max(g, 1), 32), np.float64)
        for i, gate in enumerate(gates):
            name, a, b, p, ang = gate[:5]
            self.kinds[i] = KINDS[name]
            self.q0[i], self.q1[i], self.pidx[i], self.angles[i] = a, b, p, ang
            if len(gate) > 5 and gate[5] is not None:
                m = np.asarray(gate[5], np.complex128).reshape(-1)
                self.mats[i, : 2 * m.size] = np.stack([m.real, m.imag], -1).reshape(-1)
            if len(gate) > 6:
                self.q2[i] = gate[6]

    def args(self):
        return (self.n_gates, _ptr(self.kinds), _ptr(self.q0), _ptr(self.q1),
                _ptr(self.q2), _ptr(self.pidx), _ptr(self.angles), _ptr(self.mats))


class _Terms:
    def __init__(self, terms: Sequence[tuple]):
        self.n = len(terms)
        self.c = np.array([t[0] for t in terms] or [0.0], np.float64)
        self.x = np.array([t[1] for t in terms] or [0], np.uint64)
        self.z = np.array([t[2] for t in terms] or [0], np.uint64)

    def args(self):
        return (self.n, _ptr(self.c), _ptr(self.x), _ptr(self.z))


def zeros(n: int) -> np.ndarray:
    return init_basis(n, 0)


def init_basis(n: int, k: int) -> np.ndarray:
    psi = np.empty(1 << n, np.complex128)
    lib().or_init_basis(_ptr(psi), n, k)
    return psi


def init_random(n: int, seed: int) -> np.ndarray:
    psi = np.empty(1 << n, np.complex128)
    lib().or_init_random(_ptr(psi), n, int(seed) & (2**64 - 1))
    return psi


def splitmix64(x: int) -> int:
    return int(lib().or_splitmix64(int(x) & (2**64 - 1)))


def u53(x: int) -> float:
    """init_random's uniform deviate ((x >> 11) + 0.5) 2^-53 (c.1 step 2)."""
    return float(lib().or_u53(int(x) & (2**64 - 1)))


def random_gaussian_at(seed: int, idx) -> np.ndarray:
    """Unnormalised init_random amplitudes a_i at the given indices
    (init_random(n, seed) = a / sqrt(sum_i |a_i|^2) over all 2^n indices)."""
    idx = np.ascontiguousarray(idx, np.uint64)
    out = np.empty(idx.size, np.complex128)
    lib().or_random_gaussian_at(int(seed) & (2**64 - 1), _ptr(idx), idx.size, _ptr(out))
    return out


def apply_gate(psi: np.ndarray, name: str, q0: int, q1: int = -1, angle: float = 0.0,
               mat=None, q2: int = -1) -> np.ndarray:
    psi = _state(psi)
    n = psi.size.bit_length() - 1
    m = None
    if mat is not None:
        c = np.asarray(mat, np.complex128).reshape(-1)
        m = np.zeros(32, np.float64)
        m[: 2 * c.size] = np.stack([c.real, c.imag], -1).reshape(-1)
    _check(lib().or_apply_gate(_ptr(psi), n, KINDS[name], q0, q1, q2, float(angle),
                               _ptr(m) if m is not None else None))
    return psi


def apply_circuit(psi: np.ndarray, gates: Sequence[tuple], theta=None) -> np.ndarray:
    psi = _state(psi)
    n = psi.size.bit_length() - 1
    c = _Circuit(gates)
    th = np.ascontiguousarray(theta if theta is not None else [0.0], np.float64)
    _check(lib().or_apply_circuit(_ptr(psi), n, *c.args(), _ptr(th)))
    return psi


def qft(psi: np.ndarray, inverse: bool = False) -> np.ndarray:
    psi = _state(psi)
    lib().or_qft(_ptr(psi), psi.size.bit_length() - 1, int(bool(inverse)))
    return psi


def expval(psi: np.ndarray, terms: Sequence[tuple]) -> float:
    psi = _state(psi)
    t = _Terms(terms)
    out = ctypes.c_double()
    _check(lib().or_expval(_ptr(psi), psi.size.bit_length() - 1, *t.args(), ctypes.byref(out)))
    return out.value


def norm2(psi: np.ndarray) -> float:
    psi = _state(psi)
    return lib().or_norm2(_ptr(psi), psi.size.bit_length() - 1)


def energy(n: int, gates, theta, terms) -> float:
    c, t = _Circuit(gates), _Terms(terms)
    th = np.ascontiguousarray(theta, np.float64)
    out = ctypes.c_double()
    _check(lib().or_energy(n, *c.args(), _ptr(th), *t.args(), ctypes.byref(out)))
    return out.value


def param_shift_grad(n: int, gates, theta, terms, which: Optional[Iterable[int]] = None,
                     threads: int = 1) -> np.ndarray:
    """g_p for p in ``which`` (default: all parameters)."""
    theta = np.ascontiguousarray(theta, np.float64)
    which = list(range(theta.size)) if which is None else [int(w) for w in which]
    c, t = _Circuit(gates), _Terms(terms)

    def one(p):
        out = np.zeros(1, np.float64)
        w = np.array([p], np.int32)
        _check(lib().or_param_shift(n, *c.args(), _ptr(theta), theta.size, *t.args(),
                                    _ptr(w), 1, _ptr(out)))
        return out[0]

    if threads <= 1 or len(which) <= 1:
        return np.array([one(p) for p in which])
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return np.array(list(ex.map(one, which)))


def vqe_adam(n: int, gates, theta0, terms, lr: float = 1e-2, beta1: float = 0.9, beta2: float = 0.999,
             eps: float = 1e-8, tol: float = 1e-7, max_iter: int = 350, threads: int = 1):
    """VQE outer loop: theta^{t+1} = theta^t - lr Adam(g^t)
     with Adam's bias-corrected moments (the paper cites Kingma
    & Ba; beta/eps defaults), gradients by the parameter-shift
    rule above.  Stops when |E_t - E_{t-1}| < tol (t >= 1) or t == max_iter
    (SPEC.md:478).  Returns (theta_T, [E_0 .. E_T], T)."""
    theta = np.array(theta0, np.float64, copy=True)
    m = np.zeros_like(theta)
    v = np.zeros_like(theta)
    trace = []
    t = 0
    while True:
        e = energy(n, gates, theta, terms)
        trace.append(e)
        if (t >= 1 and abs(e - trace[-2]) < tol) or t == max_iter:
            return theta, np.array(trace), t
        g = param_shift_grad(n, gates, theta, terms, threads=threads)
        m = beta1 * m + (1.0 - beta1) * g
        v = beta2 * v + (1.0 - beta2) * (g * g)
        m_hat = m / (1.0 - beta1 ** (t + 1))
        v_hat = v / (1.0 - beta2 ** (t + 1))
        theta = theta - (lr * m_hat) / (np.sqrt(v_hat) + eps)
        t += 1


def xyz_hamiltonian(n: int, jx: float, jy: float, jz: float, h: float):
    """Eq. (9): H = -sum_{i<n-1} (Jx X_i X_{i+1} + Jy Y_i Y_{i+1}
    + Jz Z_i Z_{i+1}) - h sum_i Z_i (open chain, reading A10) as Pauli terms
    (coeff, x_mask, z_mask) with bit q = qubit q."""
    terms = []
    for i in range(n - 1):
        m = (1 << i) | (1 << (i + 1))
        terms += [(-jx, m, 0), (-jy, m, m), (-jz, 0, m)]
    terms += [(-h, 0, 1 << i) for i in range(n)]
    return terms


def trotter_xyz(psi: np.ndarray, jx: float, jy: float, jz: float, amp: float, omega: float, t0: float,
                dt: float, n_steps: int, record_every: int = 1) -> np.ndarray:
    """First-order Trotter evolution (Eq. 12) of psi in place:
    step j applies exp(-i H_k(t_j) dt) for the groups of P:825-831 in the
    order RXX(-2 Jx dt) on (i, i+1) for i ascending, RYY(-2 Jy dt), RZZ(-2 Jz
    dt), RZ(-2 h(t_j) dt) on each qubit, h(t) = amp sin(omega t)
    (signs of Eq. 9, reading A20; order SPEC.md:541), each gate as its
    native matrix.  Returns E(t) = <psi|H(t)|psi> (Eq. 13) at t0 and after
    every record_every steps."""
    n = psi.size.bit_length() - 1
    h = lambda t: amp * math.sin(omega * t)
    out = [expval(psi, xyz_hamiltonian(n, jx, jy, jz, h(t0)))]
    for j in range(n_steps):
        tj = t0 + j * dt
        gates = []
        for name, J in (("RXX", jx), ("RYY", jy), ("RZZ", jz)):
            gates += [(name, i, i + 1, -1, -2.0 * J * dt) for i in range(n - 1)]
        gates += [("RZ", i, -1, -1, -2.0 * h(tj) * dt) for i in range(n)]
        apply_circuit(psi, gates)
        if (j + 1) % record_every == 0:
            out.append(expval(psi, xyz_hamiltonian(n, jx, jy, jz, h(t0 + (j + 1) * dt))))
    return np.array(out)
