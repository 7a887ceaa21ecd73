"""Step-time probe of the flood solve loop on config 2/3 (one-iteration vs two-iteration launches).

    BGABP_FLOOD2=0|1 BGABP_FLOOD2_H=64 BGABP_FLOOD2_ST=4 python tools/flood2_probe.py [config]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1904_04093_b200 as g  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
P = g.config_problem(cfg)
eng = g.GabpEngine(P.A)
dev = torch.device("cuda", 0)
stream = torch.cuda.ExternalStream(eng.stream(), device=dev)
b = torch.from_numpy(P.b).to(dev)
opt = g.GabpOptions(tol=0.0, max_iter=100000)
eng.solve_device_begin(b.data_ptr(), g.Schedule.parallel_flood(), opt)
eng.solve_device_steps(64)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 512
e0.record(stream)
eng.solve_device_steps(K)
e1.record(stream)
e1.synchronize()
ms = e0.elapsed_time(e1) / K
hot = eng.solve_device_steps_timed(64) / 64
st, its, _, _ = eng.solve_device_end()
print(f"config {cfg} FLOOD2={os.environ.get('BGABP_FLOOD2', '1')} H={os.environ.get('BGABP_FLOOD2_H', '64')} "
      f"ST={os.environ.get('BGABP_FLOOD2_ST', '4')}: {ms * 1e3:.1f} us/iteration (kernel {hot * 1e3:.1f} us/iteration), "
      f"{eng.num_edges / (ms / 1e3):.3e} edge-upd/s, status {int(st)} its {its}")
