"""A few line-GaBP sweeps on poisson J (default 9) for an ncu capture of k_line_phase."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1904_04093_b200 as g
J = int(os.environ.get("LINE_J", "9"))
p = g.assemble("poisson", J)
D = g.LineGabpEngine(p.A, p.nx, p.nx)
lam, m = D.make_state()
x = np.zeros(p.A.n)
for _ in range(3):
    D.sweep(p.b, lam, m, x)
print("ok")
