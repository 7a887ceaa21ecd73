"""Device-resident line-GaBP solve: time per iteration (full sweeps: precisions and means)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1904_04093_b200 as g
for J in (9, 11):
    p = g.assemble("poisson", J)
    D = g.LineGabpEngine(p.A, p.nx, p.nx)
    opt = g.RegionSolveOptions(tol=0.0, max_iter=5)
    D.solve(p.b, opt)
    K = 40
    opt = g.RegionSolveOptions(tol=0.0, max_iter=K)
    t = time.perf_counter()
    rep = D.solve(p.b, opt)
    dt = (time.perf_counter() - t) / K
    print(f"J={J} n={p.A.n}: line solve {rep.iterations} iterations, {dt*1e3:.3f} ms/iteration")
