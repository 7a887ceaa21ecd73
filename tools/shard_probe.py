"""Per-iteration time of the peer-memory sharded flood solve on one GPU (config 2 split into P row
blocks; P shards share the GPU, so this measures the sharding overhead, not multi-GPU scaling).

    python tools/shard_probe.py [P ...]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1904_04093_b200 as g  # noqa: E402
from paper_1904_04093_b200.shard import GpuShard, ShardLayout, dia_halo, local_matrix, sharded_solve_p2p  # noqa: E402

P2 = g.config_problem(2)
A, b = P2.A, P2.b
iters = 512
opt = g.GabpOptions(tol=0.0, max_iter=iters)
binf = float(np.abs(b).max())
eng = g.GabpEngine(A)
eng.solve(b, g.Schedule.parallel_flood(), g.GabpOptions(tol=0.0, max_iter=32))
torch.cuda.synchronize()
t0 = time.perf_counter()
rep = eng.solve(b, g.Schedule.parallel_flood(), opt)
single = (time.perf_counter() - t0) / iters
print(f"single engine: {single * 1e6:.1f} us/iteration")
del eng
for P in [int(a) for a in sys.argv[1:]] or [2, 4, 8]:
    layouts = ShardLayout.partition(A.n, dia_halo(A), P, align=2048)
    shards = {k: GpuShard(local_matrix(A, layouts[k]), layouts[k], b[layouts[k].glo:layouts[k].ghi]) for k in range(P)}
    sharded_solve_p2p(shards, layouts, binf, g.GabpOptions(tol=0.0, max_iter=64), graph=True)  # warm / capture
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st, its, det, xs, hist = sharded_solve_p2p(shards, layouts, binf, opt, graph=True)
    dt = (time.perf_counter() - t0) / iters
    x = np.concatenate([xs[k] for k in range(P)])
    same = np.array_equal(x, rep.solution) and np.array_equal(hist, rep.residual_history)
    print(f"{P} peer shards on one GPU: {dt * 1e6:.1f} us/iteration ({dt / single:.2f}x single), bit-identical: {same}")
    if not same:
        print("  status/its", st, its, int(rep.status), rep.iterations, "hist equal", np.array_equal(hist, rep.residual_history),
              "x maxdiff", float(np.max(np.abs(x - rep.solution))), "first bad", int(np.argmax(x != rep.solution)),
              "n bad", int(np.sum(x != rep.solution)))
        hb = np.nonzero(hist != rep.residual_history)[0]
        print("  hist lengths", len(hist), len(rep.residual_history), "bad idx", hb[:5], hist[hb[:3]], rep.residual_history[hb[:3]])
        st2, its2, _, xs2, hist2 = sharded_solve_p2p(shards, layouts, binf, opt, graph=False)
        x2 = np.concatenate([xs2[k] for k in range(P)])
        print("  event mode: x equal", np.array_equal(x2, rep.solution), "hist equal", np.array_equal(hist2, rep.residual_history),
              "n bad", int(np.sum(x2 != rep.solution)))
    del shards
