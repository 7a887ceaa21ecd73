"""Throughput of the engine's staged host->device upload (bgabp_create of the config-5 fine level,
84M entries) and of the pageable D2H of a solve's x; knobs BGABP_STAGE_MB / BGABP_STAGE_THREADS."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_1904_04093_b200 as g  # noqa: E402

P = g.config5_level(12, 0, sigma=1.0)
A = P.A
nbytes = A.nnz * 12 + (A.n + 1) * 4
g.GabpEngine(g.poisson5(64, 64))  # context + stager warm
torch.cuda.synchronize()
best = 1e9
for _ in range(3):
    t0 = time.perf_counter()
    e = g.GabpEngine(A)
    torch.cuda.synchronize()
    best = min(best, time.perf_counter() - t0)
    del e
print(f"STAGE_MB={os.environ.get('BGABP_STAGE_MB', '32')} THREADS={os.environ.get('BGABP_STAGE_THREADS', '16')}: "
      f"create {best * 1e3:.1f} ms for {nbytes / 1e9:.2f} GB CSR ({nbytes / best / 1e9:.1f} GB/s incl. validation + build)",
      f"nproc={os.cpu_count()}")
