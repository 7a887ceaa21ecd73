import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np, torch
import paper_1904_04093_b200 as g
P = g.config_problem(2); eng = g.GabpEngine(P.A); n = P.A.n
b_pin = torch.from_numpy(P.b).pin_memory(); b_np = b_pin.numpy(); x_pin = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
tol = 1e-8*np.abs(P.b).max(); s = g.Schedule.parallel_flood()
for K in (2, 500, 500, 2000):
    torch.cuda.synchronize(); t=time.perf_counter(); r = eng.solve(b_np, s, g.GabpOptions(tol=tol, max_iter=K), x_out=x_pin); dt=time.perf_counter()-t
    print("solve K=%d %.2f ms  (%.3f ms/iter)" % (K, dt*1e3, dt*1e3/K), r.iterations)
bd = b_pin.cuda()
for K in (500, 2000):
    eng.solve_device_begin(bd.data_ptr(), s, g.GabpOptions(tol=tol, max_iter=K)); torch.cuda.synchronize()
    t=time.perf_counter(); eng.solve_device_steps(K+2); st=eng.solve_device_end(); dt=time.perf_counter()-t
    print("device K=%d %.2f ms (%.3f ms/iter)" % (K, dt*1e3, dt*1e3/K), st[:2])
xd = torch.empty(n, dtype=torch.float64, device='cuda')
torch.cuda.synchronize(); t=time.perf_counter(); xd.copy_(b_pin); torch.cuda.synchronize(); print("H2D %.2f ms" % ((time.perf_counter()-t)*1e3))
torch.cuda.synchronize(); t=time.perf_counter(); torch.from_numpy(x_pin).copy_(xd); torch.cuda.synchronize(); print("D2H %.2f ms" % ((time.perf_counter()-t)*1e3))
