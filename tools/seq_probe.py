"""Time sequential (lexicographic) GaBP solve steps on poisson5(N,N) on the device."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1904_04093_b200 as g
for N in (64, 512, 2048):
    P = g.config_problem(2, size=N)
    eng = g.GabpEngine(P.A)
    b = torch.tensor(P.b, device="cuda")
    for name, s in (("sequential", g.Schedule.sequential()), ("red-black", g.Schedule.red_black_grid(N, N))):
        K = 50 if N == 2048 else 200
        eng.solve_device_begin(b.data_ptr(), s, g.GabpOptions(tol=0.0, max_iter=K + 10))
        eng.solve_device_steps(3); torch.cuda.synchronize()
        t = time.perf_counter(); eng.solve_device_steps(K); torch.cuda.synchronize(); dt = time.perf_counter() - t
        eng.solve_device_end()
        print(f"N={N} {name}: {dt / K * 1e3:.3f} ms/iteration (sweep + residual + stop test)")
