"""Short driver for ncu: config 2 (poisson5 2048^2) solve steps, or --config N.

    python tools/prof_step.py [--config 2] [--steps 8]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1904_04093_b200 as g  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--steps", type=int, default=8)
ap.add_argument("--sched", default="flood")
a = ap.parse_args()
P = g.config_problem(a.config)
eng = g.GabpEngine(P.A)
b = torch.tensor(P.b, device="cuda")
sched = g.Schedule.parallel_flood() if a.sched == "flood" else g.Schedule.red_black_grid(P.nx, P.nx)
eng.solve_device_begin(b.data_ptr(), sched, g.GabpOptions(tol=1e-8 * float(np.abs(P.b).max()), max_iter=20000))
eng.solve_device_steps(a.steps)
torch.cuda.synchronize()
print(eng.solve_device_end())
