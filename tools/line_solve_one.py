"""One device line-GaBP solve of 6 iterations at poisson J (default 11), for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_04093_b200 as g
J = int(os.environ.get("LINE_J", "11"))
p = g.assemble("poisson", J)
D = g.LineGabpEngine(p.A, p.nx, p.nx)
print(D.solve(p.b, g.RegionSolveOptions(tol=0.0, max_iter=6)).iterations)
