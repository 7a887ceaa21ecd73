"""Steady-state throughput of the pipelined lexicographic solve (sweep + residual + stop test):
one launch of K sweeps (device-resident b), and whole solves through GabpEngine.solve."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1904_04093_b200 as g
N = int(os.environ.get("SEQ_N", "2048"))
P = g.config_problem(2, size=N)
eng = g.GabpEngine(P.A)
b = torch.tensor(P.b, device="cuda")
for K in [int(k) for k in os.environ.get("SEQ_K", "64,512,2048").split(",")]:
    eng.solve_device_begin(b.data_ptr(), g.Schedule.sequential(), g.GabpOptions(tol=0.0, max_iter=K + 10))
    torch.cuda.synchronize()
    t = time.perf_counter(); eng.solve_device_steps(K); torch.cuda.synchronize(); dt = time.perf_counter() - t
    st, its, _, _ = eng.solve_device_end()
    print(f"N={N} K={K}: {dt / K * 1e3:.3f} ms/iteration in one launch ({st.name}, {its} decided)")
for it in [int(k) for k in os.environ.get("SEQ_SOLVE", "1000,5000").split(",") if k]:
    eng.solve(P.b, g.Schedule.sequential(), g.GabpOptions(tol=0.0, max_iter=10))
    t = time.perf_counter()
    rep = eng.solve(P.b, g.Schedule.sequential(), g.GabpOptions(tol=0.0, max_iter=it))
    dt = time.perf_counter() - t
    print(f"N={N} solve max_iter={it}: {dt:.3f} s, {dt / rep.iterations * 1e3:.3f} ms/iteration "
          f"({rep.status.name}, {rep.iterations}) host b / x")
