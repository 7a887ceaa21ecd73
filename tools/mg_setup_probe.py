"""Where the multigrid setup time goes at config-5 size (levels, engine builds, probes, recording)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1904_04093_b200 as g
J = int(os.environ.get("MG_J", "12"))
torch.zeros(1, device="cuda"); torch.cuda.synchronize()
t = time.perf_counter()
levels = [g.config5_level(J, k, sigma=1.0) for k in range(J - 4)]
print(f"levels generated: {time.perf_counter() - t:.3f} s")
t = time.perf_counter()
e = g.GabpEngine(levels[0].A); torch.cuda.synchronize()
print(f"one fine GabpEngine build: {time.perf_counter() - t:.3f} s")
del e
for sm in (g.MgSmoother.GabpRedBlack, g.MgSmoother.GsRedBlack):
    torch.cuda.synchronize(); t = time.perf_counter()
    h = g.Hierarchy.from_levels([p.A for p in levels], [p.nx for p in levels], sm)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    b = torch.tensor(levels[0].b, device="cuda"); x = torch.zeros_like(b)
    g.mg_solve_device(h, g.CycleSpec(2, 2, sm), b.data_ptr(), x.data_ptr(), g.MgSolveOptions(tol=0.0, max_cycles=1))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"{sm.name}: Hierarchy {t1 - t:.3f} s, first cycle (incl. recording) {t2 - t1:.3f} s")
    del h
