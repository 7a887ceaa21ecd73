"""Steady-state throughput of the pipelined lexicographic solve (sweep + residual + stop test)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1904_04093_b200 as g
N = int(os.environ.get("SEQ_N", "2048"))
P = g.config_problem(2, size=N)
eng = g.GabpEngine(P.A)
b = torch.tensor(P.b, device="cuda")
for K in (int(os.environ.get("SEQ_K", "0")) or 64, 512):
    eng.solve_device_begin(b.data_ptr(), g.Schedule.sequential(), g.GabpOptions(tol=0.0, max_iter=K + 10))
    torch.cuda.synchronize()
    t = time.perf_counter(); eng.solve_device_steps(K); torch.cuda.synchronize(); dt = time.perf_counter() - t
    st, its, _, _ = eng.solve_device_end()
    print(f"N={N} K={K}: {dt / K * 1e3:.3f} ms/iteration ({st.name}, {its} decided)")
