"""GabpLine V(1,1) cycles at poisson J (default 11) for an ncu capture of k_line_mean_rows/_cols."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_04093_b200 as g
J = int(os.environ.get("LINE_J", "11"))
p = g.assemble("poisson", J)
H = g.Hierarchy("poisson", J, J - 1, smoother=g.MgSmoother.GabpLine)
rep = g.mg_solve(H, g.CycleSpec(1, 1, g.MgSmoother.GabpLine), p.b, g.MgSolveOptions(tol=0.0, max_cycles=2))
print(rep.status, rep.iterations)
