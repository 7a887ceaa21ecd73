"""Red-black solve iterations on config 2 (for an ncu launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1904_04093_b200 as g
N = int(os.environ.get("RB_N", "2048"))
P = g.config_problem(2, size=N)
eng = g.GabpEngine(P.A)
b = torch.tensor(P.b, device="cuda")
eng.solve_device_begin(b.data_ptr(), g.Schedule.red_black_grid(N, N), g.GabpOptions(tol=0.0, max_iter=40))
eng.solve_device_steps(20); torch.cuda.synchronize()
print(eng.solve_device_end()[:2])
