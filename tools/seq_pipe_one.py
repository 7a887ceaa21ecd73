"""One pipelined sequential launch of SEQ_K sweeps on config-2 (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1904_04093_b200 as g
N = int(os.environ.get("SEQ_N", "2048")); K = int(os.environ.get("SEQ_K", "256"))
P = g.config_problem(2, size=N)
eng = g.GabpEngine(P.A)
b = torch.tensor(P.b, device="cuda")
eng.solve_device_begin(b.data_ptr(), g.Schedule.sequential(), g.GabpOptions(tol=0.0, max_iter=K + 10))
eng.solve_device_steps(K); torch.cuda.synchronize()
print(eng.solve_device_end()[:2])
