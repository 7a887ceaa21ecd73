"""GabpLine V(1,1) multigrid at poisson J (default 11): one warm solve of 2 cycles (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1904_04093_b200 as g
J = int(os.environ.get("LINE_J", "11"))
p = g.assemble("poisson", J)
H = g.Hierarchy("poisson", J, J - 1, smoother=g.MgSmoother.GabpLine)
spec = g.CycleSpec(1, 1, g.MgSmoother.GabpLine)
g.mg_solve(H, spec, p.b, g.MgSolveOptions(tol=0.0, max_cycles=1))
rep = g.mg_solve(H, spec, p.b, g.MgSolveOptions(tol=0.0, max_cycles=2))
print(rep.status, rep.iterations)
