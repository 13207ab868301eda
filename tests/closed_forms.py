"""Closed forms used as pins by several test files (no oracle code)."""
import numpy as np


def product_energy_and_grad(n, theta, terms_j=(1.0, 0.7, 0.4), hz=0.3):
    """Closed form for the product ansatz RY(t_q) then RZ(p_q): Bloch vector
    b_q = (sin t cos p, sin t sin p, cos t); E = sum_i sum_a J_a b^a_i b^a_{i+1}
    + hz sum_q b^z_q; gradient by the product rule (SURVEY c.4)."""
    t, p = theta[:n], theta[n:]
    b = np.stack([np.sin(t) * np.cos(p), np.sin(t) * np.sin(p), np.cos(t)], 1)
    db_dt = np.stack([np.cos(t) * np.cos(p), np.cos(t) * np.sin(p), -np.sin(t)], 1)
    db_dp = np.stack([-np.sin(t) * np.sin(p), np.sin(t) * np.cos(p), 0 * t], 1)
    J = np.array(terms_j)
    E = sum(float(np.sum(J * b[i] * b[i + 1])) for i in range(n - 1)) + hz * float(b[:, 2].sum())
    gt, gp = np.zeros(n), np.zeros(n)
    for q in range(n):
        for nb in (q - 1, q + 1):
            if 0 <= nb < n:
                gt[q] += np.sum(J * db_dt[q] * b[nb])
                gp[q] += np.sum(J * db_dp[q] * b[nb])
        gt[q] += hz * db_dt[q, 2]
    return E, np.concatenate([gt, gp])


# ---- monomial circuits (SURVEY c.4 (i), (vi)): X, Y, Z, S, T, RZ, CNOT, CZ
# map basis states to phased basis states; qubit q <-> index bit n-1-q.
_DIAG1 = {"Z": lambda a: -1.0, "S": lambda a: 1j, "T": lambda a: np.exp(1j * np.pi / 4)}


def _bit(k, n, q):
    return (k >> (n - 1 - q)) & 1


def monomial_forward(n, gates, k):
    """|k> -> phase |k'> through the circuit (closed form, O(#gates))."""
    ph = 1.0 + 0j
    for name, a, b, _, ang in gates:
        if name == "X":
            k ^= 1 << (n - 1 - a)
        elif name == "Y":              # Y|0> = i|1>, Y|1> = -i|0>
            ph *= -1j if _bit(k, n, a) else 1j
            k ^= 1 << (n - 1 - a)
        elif name in _DIAG1:
            if _bit(k, n, a):
                ph *= _DIAG1[name](ang)
        elif name == "RZ":             # diag(e^{-i t/2}, e^{i t/2})
            ph *= np.exp(0.5j * ang) if _bit(k, n, a) else np.exp(-0.5j * ang)
        elif name == "CNOT":
            if _bit(k, n, a):
                k ^= 1 << (n - 1 - b)
        elif name == "CZ":
            if _bit(k, n, a) and _bit(k, n, b):
                ph = -ph
        else:
            raise ValueError(name)
    return k, ph


def monomial_backward(n, gates, j):
    """Output basis index j -> (input index k, phase) with <j|C|k> = phase."""
    ph = 1.0 + 0j
    for name, a, b, _, ang in reversed(gates):
        if name == "X":
            j ^= 1 << (n - 1 - a)
        elif name == "Y":              # out bit 1 came from |0> with i, out 0 from |1> with -i
            ph *= 1j if _bit(j, n, a) else -1j
            j ^= 1 << (n - 1 - a)
        elif name in _DIAG1:
            if _bit(j, n, a):
                ph *= _DIAG1[name](ang)
        elif name == "RZ":
            ph *= np.exp(0.5j * ang) if _bit(j, n, a) else np.exp(-0.5j * ang)
        elif name == "CNOT":
            if _bit(j, n, a):
                j ^= 1 << (n - 1 - b)
        elif name == "CZ":
            if _bit(j, n, a) and _bit(j, n, b):
                ph = -ph
        else:
            raise ValueError(name)
    return j, ph


def monomial_inverse(gates):
    inv = {"S": "SDG", "T": "TDG"}
    return [(inv.get(g[0], g[0]), g[1], g[2], g[3], -g[4] if g[0] == "RZ" else g[4]) for g in reversed(gates)]


def qft_of_basis(n, k, idx):
    """QFT|k> at indices idx: N^-1/2 e^{2 pi i ((j k) mod N) / N}."""
    N = 1 << n
    jk = (np.asarray(idx, dtype=object) * int(k)) % N
    return np.exp(2j * np.pi * np.array([float(x) for x in jk]) / N) / np.sqrt(N)


def circuit_inverse(gates):
    """C^-1 for the config-1/5 alphabet and the monomial kinds: reversed
    order, S <-> S^dagger, T <-> T^dagger, rotation angles negated
    (R(t)^-1 = R(-t)); H, X, Y, Z, CNOT, CZ, SWAP are
    involutions."""
    inv = {"S": "SDG", "SDG": "S", "T": "TDG", "TDG": "T"}
    out = []
    for g in reversed(gates):
        name = g[0]
        if name in ("RX", "RY", "RZ", "CP", "CRY", "RXX", "RYY", "RZZ"):
            assert g[3] == -1, "parameterised gates need theta"
            out.append((name, g[1], g[2], g[3], -g[4]))
        elif name in inv or name in ("H", "X", "Y", "Z", "CNOT", "CZ", "SWAP"):
            out.append((inv.get(name, name), g[1], g[2], g[3], g[4]))
        else:
            raise ValueError(name)
    return out
