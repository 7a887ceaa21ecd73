"""A few sequential (lexicographic) solve iterations on poisson5(N,N) for an ncu capture of k_seq_grid5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1904_04093_b200 as g
N = int(os.environ.get("SEQ_N", "512"))
P = g.config_problem(2, size=N)
eng = g.GabpEngine(P.A)
b = torch.tensor(P.b, device="cuda")
eng.solve_device_begin(b.data_ptr(), g.Schedule.sequential(), g.GabpOptions(tol=0.0, max_iter=20))
eng.solve_device_steps(6)
torch.cuda.synchronize()
eng.solve_device_end()
print("ok")
