"""Setup-time breakdown of the config-5 hierarchy (BGABP_TIMING=1 prints per phase)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_1904_04093_b200 as g  # noqa: E402

levels = [g.config5_level(12, k, sigma=1.0) for k in range(8)]
b = levels[0].b
g.GabpEngine(g.poisson5(64, 64))
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    h = g.Hierarchy.from_levels([p.A for p in levels], [p.nx for p in levels], g.MgSmoother.GabpRedBlack)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = g.mg_solve(h, g.CycleSpec(2, 2, g.MgSmoother.GabpRedBlack), b,
                   g.MgSolveOptions(tol=1e-8 * float(np.abs(b).max()), max_cycles=100))
    t2 = time.perf_counter()
    print(f"setup {1e3 * (t1 - t0):.1f} ms, solve {1e3 * (t2 - t1):.1f} ms ({r.iterations} cycles, {r.status.name})",
          file=sys.stderr)
    del h
