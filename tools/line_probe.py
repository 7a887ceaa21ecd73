"""Time line-GaBP sweeps (region GaBP over grid lines) and the GabpLine multigrid cycle on the device."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1904_04093_b200 as g
for J in (7, 9, 11):
    p = g.assemble("poisson", J)
    D = g.LineGabpEngine(p.A, p.nx, p.nx)
    lam, m = D.make_state()
    x = np.zeros(p.A.n)
    D.sweep(p.b, lam, m, x)
    K = 10
    t = time.perf_counter()
    for _ in range(K):
        D.sweep(p.b, lam, m, x)
    dt = (time.perf_counter() - t) / K
    print(f"J={J} n={p.A.n}: line sweep (incl. host state copies) {dt*1e3:.3f} ms")
    H = g.Hierarchy("poisson", J, J - 1, smoother=g.MgSmoother.GabpLine)
    spec = g.CycleSpec(1, 1, g.MgSmoother.GabpLine)
    rep = g.mg_solve(H, spec, p.b, g.MgSolveOptions(tol=1e-8 * np.abs(p.b).max()))
    t = time.perf_counter()
    rep = g.mg_solve(H, spec, p.b, g.MgSolveOptions(tol=1e-8 * np.abs(p.b).max()))
    dt = time.perf_counter() - t
    print(f"J={J}: mg GabpLine V(1,1) {rep.status.name} in {rep.iterations} cycles, {dt*1e3:.1f} ms "
          f"({dt / max(rep.iterations, 1) * 1e3:.2f} ms/cycle)")
