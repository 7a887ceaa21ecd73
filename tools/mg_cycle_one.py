"""Config-5 (sigma=1) red-black GaBP V(2,2): one warm solve of 3 cycles (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1904_04093_b200 as g
J = int(os.environ.get("MG_J", "12"))
levels = [g.config5_level(J, k, sigma=1.0) for k in range(J - 4)]
h = g.Hierarchy.from_levels([p.A for p in levels], [p.nx for p in levels], g.MgSmoother.GabpRedBlack)
b = torch.tensor(levels[0].b, device="cuda"); x = torch.zeros_like(b)
spec = g.CycleSpec(2, 2, g.MgSmoother.GabpRedBlack)
g.mg_solve_device(h, spec, b.data_ptr(), x.data_ptr(), g.MgSolveOptions(tol=0.0, max_cycles=1))
torch.cuda.synchronize()
rep = g.mg_solve_device(h, spec, b.data_ptr(), x.data_ptr(), g.MgSolveOptions(tol=0.0, max_cycles=3))
torch.cuda.synchronize()
print(rep.status, rep.iterations)
