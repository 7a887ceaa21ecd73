"""Are lexicographic pipeline solves limited per pipeline (dependencies) or per GPU (resources)?
Runs one, then two independent pipelined solves concurrently (separate engines and streams)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1904_04093_b200 as g
N = int(os.environ.get("SEQ_N", "2048"))
K = int(os.environ.get("SEQ_K", "256"))
P = g.config_problem(2, size=N)
b = torch.tensor(P.b, device="cuda")
engs = [g.GabpEngine(P.A) for _ in range(3)]
for m in (1, 2, 3):
    for e in engs[:m]:
        e.solve_device_begin(b.data_ptr(), g.Schedule.sequential(), g.GabpOptions(tol=0.0, max_iter=K + 10))
    torch.cuda.synchronize()
    t = time.perf_counter()
    for e in engs[:m]:
        e.solve_device_steps(K)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    for e in engs[:m]:
        e.solve_device_end()
    print(f"{m} concurrent pipelines, N={N} K={K}: {dt / K * 1e3:.3f} ms per iteration of each")
