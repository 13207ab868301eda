import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W, oracle
from paper_2512_23183_b200 import lq
oracle.build()
for n in (13, 16):
    psi = oracle.init_random(n, 3)
    sv = lq.StateVector(n).init_random(3)
    for name, terms in [("Z0", [(1.0, 0, 1)]), ("Zlast", [(1.0, 0, 1 << (n-1))]), ("ZZ01", [(1.0, 0, 3)]),
                        ("XX01", [(1.0, 3, 0)]), ("YY01", [(1.0, 3, 3)]), ("XXmid", [(1.0, 3 << 6, 0)]),
                        ("X0", [(1.0, 1, 0)]), ("Y0", [(1.0, 1, 1)]), ("xyz", W.xyz_terms(n))]:
        e = sv.expval(terms); eo = oracle.expval(psi, terms)
        print(n, name, e, eo, "OK" if abs(e-eo) < 1e-10 else "BAD")
for n in (4, 10, 14):
    gates = W.hea_ansatz(n, 2, "ring")
    theta = np.random.default_rng(n).uniform(0, 2*np.pi, 4*n)
    for terms_name, terms in [("Z0", [(1.0, 0, 1)]), ("xyz", W.xyz_terms(n))]:
        g, e = lq.lq_param_shift_grad(n, gates, theta, terms)
        eo = oracle.energy(n, gates, theta, terms)
        print("psr", n, terms_name, e, eo, "OK" if abs(e-eo) < 1e-10 else "BAD")
