#!/usr/bin/env python
"""Config 5 (BASELINE.json): which coarse-grid rule lets the reference's V(2,2) cycle converge on
the sigma = 2 lognormal field?  Runs on the GPU through the product API (Hierarchy.from_levels +
mg_solve, the reference's own transfer operators and cycle, multigrid.cpp:111-318) and prints one
JSON document with the per-cycle residual factor of every (rule, smoother, sigma).

Rules for the coarse operators (the reference rediscretises each level, multigrid.cpp:79-83; for
a field it does not define the coarse K, so the rule is the builder's choice):
  fw_logK     full-weighted log K (weighted geometric mean) -- the generator's rule
  fw_K        full-weighted K (arithmetic)
  fw_invK     full-weighted 1/K (harmonic)
  inject      the coinciding fine vertex's K
  galerkin    A_c = R A_f P with the reference's restriction R and prolongation P (9-point coarse
              operators), smoothed with the four-colour orders
and a two-grid cycle with the exact coarse solve (fine 127^2, coarse 63^2 dense) for each
rediscretisation rule.  Galerkin hierarchies are built with the sweeps_expand probe on and off
(BGABP_MG_NO_PROBE=1).

    python tools/config5_coarse_rules.py [--J 10] [--cycles 40] > profiles/r02_config5_coarse_rules.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1904_04093_b200 as g  # noqa: E402

S = g.MgSmoother
RULES = {"fw_logK": 0, "fw_K": 1, "fw_invK": 2, "inject": 3}


def csr(A):
    return sp.csr_matrix((A.values, A.col_indices, A.row_offsets), shape=(A.n, A.n))


def restriction(mf):
    """mg_restrict (multigrid.cpp:111-130) as a matrix: coarse IX <-> fine 2IX+1, 1/16 [1 2 1; 2 4 2; 1 2 1]."""
    mc = (mf - 1) // 2
    rows, cols, vals = [], [], []
    w = {(-1, -1): 1, (0, -1): 2, (1, -1): 1, (-1, 0): 2, (0, 0): 4, (1, 0): 2, (-1, 1): 1, (0, 1): 2, (1, 1): 1}
    for IY in range(mc):
        for IX in range(mc):
            for (dx, dy), wt in w.items():
                x, y = 2 * IX + 1 + dx, 2 * IY + 1 + dy
                rows.append(IY * mc + IX)
                cols.append(y * mf + x)
                vals.append(wt / 16.0)
    return sp.csr_matrix((vals, (rows, cols)), shape=(mc * mc, mf * mf))


def to_sparse_matrix(M):
    M = M.tocsr()
    M.sum_duplicates()
    M.sort_indices()
    return g.SparseMatrix(M.shape[0], M.indptr.astype(np.int32), M.indices.astype(np.int32), M.data.astype(np.float64))


def factor(rep):
    h = np.asarray(rep.residual_history)
    k = len(h) - 1
    if k < 1 or not np.all(np.isfinite(h)) or h[0] == 0:
        return None, None
    overall = float((h[-1] / h[0]) ** (1.0 / k))
    tail = h[-6:] if len(h) >= 6 else h
    last = float((tail[-1] / tail[0]) ** (1.0 / (len(tail) - 1))) if len(tail) > 1 else overall
    return overall, last


def run(levels, nxs, b, sm, cycles, no_probe=False):
    if no_probe:
        os.environ["BGABP_MG_NO_PROBE"] = "1"
    try:
        t0 = time.perf_counter()
        h = g.Hierarchy.from_levels(levels, nxs, sm)
        setup = time.perf_counter() - t0
        tol = 1e-8 * float(np.abs(b).max())
        t0 = time.perf_counter()
        rep = g.mg_solve(h, g.CycleSpec(2, 2, sm), b, g.MgSolveOptions(tol=tol, max_cycles=cycles))
        dt = time.perf_counter() - t0
        f_all, f_last = factor(rep)
        return {"status": rep.status.name, "cycles": rep.iterations, "levels": h.num_levels(),
                "factor_per_cycle": f_all, "factor_last5": f_last, "detail": rep.detail,
                "final_rel_residual": float(rep.residual_history[-1] / np.abs(b).max()),
                "setup_s": setup, "solve_s": dt}
    except Exception as ex:  # e.g. a probe truncation leaving a coarse level too large for LU
        return {"status": "error", "detail": str(ex)}
    finally:
        os.environ.pop("BGABP_MG_NO_PROBE", None)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--J", type=int, default=10)
    ap.add_argument("--cycles", type=int, default=40)
    ap.add_argument("--sigmas", type=float, nargs="+", default=[2.0, 1.0])
    ap.add_argument("--rules", nargs="+", default=list(RULES) + ["galerkin"])
    ap.add_argument("--no-two-grid", action="store_true")
    args = ap.parse_args()
    J, nl = args.J, args.J - 4  # down to 31^2 as config 5
    out = {"J": J, "levels": nl, "cycle": "V(2,2)", "tol": "1e-8 ||b||_inf", "max_cycles": args.cycles,
           "multilevel": {}, "two_grid_exact": {}, "galerkin": {}}
    # the transfer operators as matrices must be the reference's (checked against the product's)
    rng = np.random.default_rng(0)
    u = rng.standard_normal(15 * 15)
    assert np.allclose(restriction(15) @ u, g.mg_restrict(u, 15), rtol=0, atol=1e-15)
    v = rng.standard_normal(7 * 7)
    assert np.allclose(4.0 * restriction(15).T @ v, g.mg_prolong(v, 7), rtol=0, atol=1e-15)
    for sigma in args.sigmas:
        for name, rule in RULES.items():
            if name not in args.rules:
                continue
            levels = [g.varcoef2d_rule_level(J, k, rule, sigma=sigma) for k in range(nl)]
            b = levels[0].b
            for smn, sm in (("gabp_red_black", S.GabpRedBlack), ("gs_red_black", S.GsRedBlack)):
                r = run([p.A for p in levels], [p.nx for p in levels], b, sm, args.cycles)
                out["multilevel"][f"sigma{sigma:g}/{name}/{smn}"] = r
                print(f"sigma {sigma} {name:8s} {smn:15s} {r}", file=sys.stderr, flush=True)
            # two-grid with the exact coarse solve (fine 127^2 -> coarse 63^2, dense)
            if args.no_two_grid:
                continue
            tg = [g.varcoef2d_rule_level(7, k, rule, sigma=sigma) for k in range(2)]
            for smn, sm in (("gabp_red_black", S.GabpRedBlack), ("gs_red_black", S.GsRedBlack)):
                r = run([p.A for p in tg], [p.nx for p in tg], tg[0].b, sm, args.cycles)
                out["two_grid_exact"][f"sigma{sigma:g}/{name}/{smn}"] = r
                print(f"sigma {sigma} two-grid {name:8s} {smn:15s} {r}", file=sys.stderr, flush=True)
        # Galerkin coarse operators from the fine level of the generator
        if "galerkin" not in args.rules:
            continue
        fine = g.varcoef2d_rule_level(J, 0, 0, sigma=sigma)
        mats, nxs = [csr(fine.A)], [fine.nx]
        while len(mats) < nl:
            R = restriction(nxs[-1])
            mats.append((R @ mats[-1] @ (4.0 * R.T)).tocsr())
            nxs.append((nxs[-1] - 1) // 2)
        levels = [to_sparse_matrix(M) for M in mats]
        for smn, sm in (("gabp_four_color", S.GabpFourColor), ("gabp_red_black", S.GabpRedBlack),
                        ("gs_four_color", S.GsFourColor)):
            for probe in (True, False):
                r = run(levels, nxs, fine.b, sm, args.cycles, no_probe=not probe)
                key = f"sigma{sigma:g}/galerkin/{smn}/probe_{'on' if probe else 'off'}"
                out["galerkin"][key] = r
                print(f"{key} {r}", file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
