"""Short driver for ncu: config-5-family V(2,2) red-black GaBP cycles.

    python tools/prof_mg.py [--J 11] [--sigma 1.0] [--cycles 2]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1904_04093_b200 as g  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--J", type=int, default=11)
ap.add_argument("--sigma", type=float, default=1.0)
ap.add_argument("--cycles", type=int, default=2)
ap.add_argument("--smoother", default="rb")
a = ap.parse_args()
levels = [g.config5_level(a.J, k, sigma=a.sigma) for k in range(a.J - 4)]
sm = {"rb": g.MgSmoother.GabpRedBlack, "gs": g.MgSmoother.GsRedBlack}[a.smoother]
h = g.Hierarchy.from_levels([p.A for p in levels], [p.nx for p in levels], sm)
b = torch.tensor(levels[0].b, device="cuda")
x = torch.zeros_like(b)
SW = int(os.environ.get("PROF_MG_SWEEPS", "2"))
rep = g.mg_solve_device(h, g.CycleSpec(SW, SW, sm), b.data_ptr(), x.data_ptr(),
                        g.MgSolveOptions(tol=1e-8 * float(np.abs(levels[0].b).max()), max_cycles=a.cycles))
torch.cuda.synchronize()
print(rep.status, rep.iterations)
if os.environ.get("PROF_MG_TIME"):
    import time
    tol_t = 1e-8 * float(np.abs(levels[0].b).max())
    for _ in range(2):
        x.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = g.mg_solve_device(h, g.CycleSpec(SW, SW, sm), b.data_ptr(), x.data_ptr(),
                                g.MgSolveOptions(tol=tol_t, max_cycles=int(os.environ["PROF_MG_TIME"])))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"timed: {rep.status} {rep.iterations} cycles, {dt:.4f} s, {1e3 * dt / max(rep.iterations, 1):.4f} ms/cycle")
