# Mutation check for the oracle pins: applies plausible bugs to oracle/oracle.c one at a time
# and confirms tests/test_oracle_pins.py catches each.  Run manually: python tests/oracle_mutation_check.py
import shutil; shutil.copy("oracle/oracle.c", "/tmp/oracle.c.bak")
import subprocess, shutil, sys
src = open('/tmp/oracle.c.bak').read()
muts = [
 ("case OR_RY:  U[0][0] = c; U[0][1] = -s; U[1][0] = s;", "case OR_RY:  U[0][0] = c; U[0][1] = s; U[1][0] = -s;"),
 ("int t_bit = n - 1 - t;", "int t_bit = t;"),
 ("OR_PI / ldexp(1.0, j - i), NULL);\n        }\n        for (int i = 0; i < n / 2", "-OR_PI / ldexp(1.0, j - i), NULL);\n        }\n        for (int i = 0; i < n / 2"),
 ("if (xb && zb)\n                or_apply_gate(phi, n, OR_Y", "if (xb && zb)\n                or_apply_gate(phi, n, OR_X"),
 ("grad[w] = (e_plus - e_minus) / 2.0;", "grad[w] = (e_plus - e_minus);"),
 ("psi[j] = U[1][0] * a + U[1][1] * b;\n    }\n}\n\n/* 2q", "psi[j] = U[1][1] * a + U[1][0] * b;\n    }\n}\n\n/* 2q"),
 ("uint64_t idx[4] = { i, i | mb, i | ma, i | ma | mb };", "uint64_t idx[4] = { i, i | ma, i | mb, i | ma | mb };"),
 ("case OR_S:   U[0][0] = 1; U[0][1] = 0; U[1][0] = 0; U[1][1] = I;", "case OR_S:   U[0][0] = 1; U[0][1] = 0; U[1][0] = 0; U[1][1] = -I;"),
 ("psi[i] *= s;", "psi[i] *= 1.0;"),
 ("case OR_RX:  U[0][0] = c; U[0][1] = -I * s; U[1][0] = -I * s;", "case OR_RX:  U[0][0] = c; U[0][1] = I * s; U[1][0] = I * s;"),
]
for a, b in muts:
    assert a in src, a
    open('oracle/oracle.c','w').write(src.replace(a, b, 1))
    r = subprocess.run([sys.executable,'-m','pytest','tests/test_oracle_pins.py','-q','-x','-p','no:cacheprovider'],capture_output=True,text=True)
    last = r.stdout.strip().splitlines()[-1]
    print(('CAUGHT ' if r.returncode else 'MISSED ') + a[:50].replace('\n',' '), '|', last)
open('oracle/oracle.c','w').write(src)
