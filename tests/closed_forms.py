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
