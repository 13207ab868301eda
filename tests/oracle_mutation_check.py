# Mutation check for the oracle pins: applies plausible bugs to the oracle
# (oracle/oracle.c and oracle/__init__.py) one at a time and confirms
# tests/test_oracle_pins.py catches each.  Run manually:
#   python tests/oracle_mutation_check.py
import shutil, subprocess, sys

FILES = {"c": "oracle/oracle.c", "py": "oracle/__init__.py"}
for f in FILES.values():
    shutil.copy(f, "/tmp/" + f.replace("/", "_") + ".bak")
orig = {k: open(f).read() for k, f in FILES.items()}
muts = [
 ("c", "case OR_RY:  U[0][0] = c; U[0][1] = -s; U[1][0] = s;", "case OR_RY:  U[0][0] = c; U[0][1] = s; U[1][0] = -s;"),
 ("c", "int t_bit = n - 1 - t;", "int t_bit = t;"),
 ("c", "OR_PI / ldexp(1.0, j - i), NULL);\n        }\n        for (int i = 0; i < n / 2", "-OR_PI / ldexp(1.0, j - i), NULL);\n        }\n        for (int i = 0; i < n / 2"),
 ("c", "if (xb && zb)\n                or_apply_gate(phi, n, OR_Y", "if (xb && zb)\n                or_apply_gate(phi, n, OR_X"),
 ("c", "grad[w] = (e_plus - e_minus) / 2.0;", "grad[w] = (e_plus - e_minus);"),
 ("c", "psi[j] = U[1][0] * a + U[1][1] * b;\n    }\n}\n\n/* 2q", "psi[j] = U[1][1] * a + U[1][0] * b;\n    }\n}\n\n/* 2q"),
 ("c", "uint64_t idx[4] = { i, i | mb, i | ma, i | ma | mb };", "uint64_t idx[4] = { i, i | ma, i | mb, i | ma | mb };"),
 ("c", "case OR_S:   U[0][0] = 1; U[0][1] = 0; U[1][0] = 0; U[1][1] = I;", "case OR_S:   U[0][0] = 1; U[0][1] = 0; U[1][0] = 0; U[1][1] = -I;"),
 ("c", "psi[i] *= s;", "psi[i] *= 1.0;"),
 ("c", "case OR_RX:  U[0][0] = c; U[0][1] = -I * s; U[1][0] = -I * s;", "case OR_RX:  U[0][0] = c; U[0][1] = I * s; U[1][0] = I * s;"),
 # f3: the paper's two-term rule applied to CRY, and a wrong four-term sign
 ("c", "grad[w] = c1 * (e[0] - e[1]) - c2 * (e[2] - e[3]);", "grad[w] = (e[0] - e[1]) / 2.0;"),
 ("c", "grad[w] = c1 * (e[0] - e[1]) - c2 * (e[2] - e[3]);", "grad[w] = c1 * (e[0] - e[1]) + c2 * (e[2] - e[3]);"),
 ("c", "U[r][k] = (r == k ? c : 0.0) - I * s * K[r][k];", "U[r][k] = (r == k ? c : 0.0) + I * s * K[r][k];"),
 # f2: Adam without bias correction, and beta1 / beta2 swapped
 ("py", "m_hat = m / (1.0 - beta1 ** (t + 1))", "m_hat = m"),
 ("py", "v = beta2 * v + (1.0 - beta2) * (g * g)", "v = beta1 * v + (1.0 - beta1) * (g * g)"),
 # f1: Trotter signs / field time / term order
 ("py", 'gates += [(name, i, i + 1, -1, -2.0 * J * dt) for i in range(n - 1)]', 'gates += [(name, i, i + 1, -1, 2.0 * J * dt) for i in range(n - 1)]'),
 ("py", 'gates += [("RZ", i, -1, -1, -2.0 * h(tj) * dt) for i in range(n)]', 'gates += [("RZ", i, -1, -1, -2.0 * h(tj + dt) * dt) for i in range(n)]'),
 ("py", "terms += [(-jx, m, 0), (-jy, m, m), (-jz, 0, m)]", "terms += [(-jx, m, 0), (-jy, m, 0), (-jz, 0, m)]"),
 # init_random (c.1 step 2): seed convention, u mapping, hash, and the |Im| / NaN rejection
 ("c", "uint64_t x0 = or_splitmix64(seed ^ (2 * i));", "uint64_t x0 = or_splitmix64(seed ^ i);"),
 ("c", "return ((double)(x >> 11) + 0.5) * 0x1.0p-53;", "return ((double)(x >> 11) + 0.0) * 0x1.0p-53;"),
 ("c", "double r = sqrt(-2.0 * log(u0));", "double r = sqrt(-2.0 * log(u1));"),
 ("c", "double u1 = or_u53(x1);", "double u1 = or_u53(x0);"),
 ("c", "return z ^ (z >> 31);", "return z ^ (z >> 30);"),
 ("c", "if (!(fabs(cimag(v)) <= 1e-10) || !isfinite(creal(v))) {", "if (fabs(cimag(v)) > 1e-10) {"),
]
for which, a, b in muts:
    assert a in orig[which], a
    open(FILES[which], "w").write(orig[which].replace(a, b, 1))
    subprocess.run([sys.executable, "-c", "import oracle; oracle.build()"], capture_output=True)
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-q", "-x", "-p", "no:cacheprovider"],
                       capture_output=True, text=True)
    last = r.stdout.strip().splitlines()[-1]
    print(("CAUGHT " if r.returncode else "MISSED ") + which + ": " + a[:60].replace("\n", " "), "|", last, flush=True)
    open(FILES[which], "w").write(orig[which])
subprocess.run([sys.executable, "-c", "import oracle; oracle.build()"], capture_output=True)
