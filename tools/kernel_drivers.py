#!/usr/bin/env python
"""Short drivers that exercise one kernel family each, for ncu captures (tools/profile_r02.sh).

    python tools/kernel_drivers.py <family> [--n N]

families (kernels):
  flood    config-2 solve steps              k_flood_solve_dia, k_solve_decide_lag2
  flood3   config-3 solve steps              k_flood_solve_dia<4, nonsymmetric>
  sweep    per-sweep API on config 2         k_flood_dia, k_aggregate_dia, k_state_gather/scatter
  sell     csr7 (config 4 on SELL) steps     k_flood_solve_sell_tma
  sellrand random DD graph on SELL steps     k_flood_solve_sell_tma / k_flood_solve_sell
  rb       red-black solve on config 2       k_rb_half, k_residual_dia
  seq      lexicographic solve on 2048^2     k_seq_pipe
  levels   greedy-coloured order, random DD  k_level_csr, k_residual_csr
  frozen   precompute_lambda + corrections   k_lambda_*, k_sigma_*, k_corr_*
  mg       config-5 V(2,2) red-black GaBP    k_restrict, k_prolong_add, k_residual_dia, k_rb_mean_half, k_gemv_rows
  mggs     config-5 V(2,2) red-black GS      k_gs_rb_half
  line     line-GaBP V(1,1) J = 11           k_line_mean_rows, k_line_mean_cols
  linesolve  line-GaBP solve J = 11          k_line_full_rows, k_line_full_cols
  build    engine setup on config 4          k_dia_fill, k_dia_facts
Each prints one line and exits 0; the shapes are the configs' (BASELINE.json) unless --n is given.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1904_04093_b200 as g  # noqa: E402


def steps(eng, b, sched, k, tol=0.0):
    bd = torch.tensor(b, device="cuda")
    eng.solve_device_begin(bd.data_ptr(), sched, g.GabpOptions(tol=tol, max_iter=k + 8))
    eng.solve_device_steps(k)
    torch.cuda.synchronize()
    return eng.solve_device_end()[:2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("family")
    ap.add_argument("--n", type=int, default=0)
    a = ap.parse_args()
    f = a.family.rstrip("0123456789") if a.family not in ("flood3",) else a.family  # mg2.. = mg (ncu passes)
    if f in ("flood", "flood3"):
        P = g.config_problem(2 if f == "flood" else 3, size=a.n)
        print(f, steps(g.GabpEngine(P.A), P.b, g.Schedule.parallel_flood(), 40))
    elif f == "sweep":
        P = g.config_problem(2, size=a.n)
        eng = g.GabpEngine(P.A)
        st = eng.make_state()
        x = np.zeros(P.A.n)
        for _ in range(3):
            eng.sweep(P.b, g.Schedule.parallel_flood(), st, x)
        print(f, "ok")
    elif f == "sell":
        P = g.config_problem(4, size=a.n)
        print(f, steps(g.GabpEngine(P.A, g.Layout.Csr), P.b, g.Schedule.parallel_flood(), 12))
    elif f == "sellrand":  # random diagonally dominant graph (bench --workload csr_random)
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from bench import random_dd
        n = a.n or (1 << 22)
        ro, ci, v, b = random_dd(n, 6, 7)
        print(f, steps(g.GabpEngine(g.SparseMatrix(n, ro, ci, v), g.Layout.Csr), b, g.Schedule.parallel_flood(), 12))
    elif f == "rb":
        N = a.n or 2048
        P = g.config_problem(2, size=N)
        print(f, steps(g.GabpEngine(P.A), P.b, g.Schedule.red_black_grid(N, N), 30))
    elif f == "seq":
        P = g.config_problem(2, size=a.n)
        print(f, steps(g.GabpEngine(P.A), P.b, g.Schedule.sequential(), 64))
    elif f == "levels":
        import scipy.sparse as sp
        n = a.n or (1 << 20)
        rng = np.random.default_rng(3)
        r = np.repeat(np.arange(n), 4)
        c = rng.integers(0, n, size=4 * n)
        keep = r != c
        M = sp.coo_matrix((-rng.random(keep.sum()), (r[keep], c[keep])), shape=(n, n))
        M = (M + M.T).tocsr()
        M = (M + sp.diags(1.0 + np.asarray(abs(M).sum(axis=1)).ravel())).tocsr()
        M.sort_indices()
        A = g.SparseMatrix(n, M.indptr.astype(np.int32), M.indices.astype(np.int32), M.data)
        b = rng.uniform(-1, 1, n)
        print(f, steps(g.GabpEngine(A, g.Layout.Csr), b, g.Schedule.red_black(A), 6))
    elif f == "frozen":
        P = g.config_problem(2, size=a.n)
        eng = g.GabpEngine(P.A)
        fz = eng.precompute_lambda(g.Schedule.parallel_flood(), 1e-10, 40)
        e = eng.correction_sweeps(P.b, g.Schedule.parallel_flood(), fz, 4)
        print(f, fz.iterations, float(np.abs(e).max()))
    elif f in ("mg", "mggs"):
        J = a.n or 12
        levels = [g.config5_level(J, k, sigma=1.0) for k in range(J - 4)]
        sm = g.MgSmoother.GabpRedBlack if f == "mg" else g.MgSmoother.GsRedBlack
        h = g.Hierarchy.from_levels([p.A for p in levels], [p.nx for p in levels], sm)
        b = torch.tensor(levels[0].b, device="cuda")
        x = torch.zeros_like(b)
        rep = g.mg_solve_device(h, g.CycleSpec(2, 2, sm), b.data_ptr(), x.data_ptr(),
                                g.MgSolveOptions(tol=0.0, max_cycles=3))
        torch.cuda.synchronize()
        print(f, rep.status, rep.iterations)
    elif f == "line":
        J = a.n or 11
        h = g.Hierarchy("poisson", J, J - 4, {}, g.MgSmoother.GabpLine)
        rep = g.mg_solve(h, g.CycleSpec(1, 1, g.MgSmoother.GabpLine), h.fine_rhs(), g.MgSolveOptions(tol=0.0,
                                                                                                     max_cycles=3))
        print(f, rep.status, rep.iterations)
    elif f == "linesolve":
        J = a.n or 11
        p = g.assemble("poisson", J)
        eng = g.LineGabpEngine(p.A, p.nx, p.nx)
        rep = eng.solve(p.b, g.RegionSolveOptions(tol=0.0, max_iter=4))
        print(f, rep.status, rep.iterations)
    elif f == "build":
        P = g.config_problem(4, size=a.n)
        for _ in range(2):
            eng = g.GabpEngine(P.A)
            del eng
        print(f, "ok")
    else:
        raise SystemExit(f"unknown family {f}")


if __name__ == "__main__":
    main()
