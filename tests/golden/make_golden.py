"""Generate the golden vectors in tests/golden/ from the REFERENCE's own compiled code.

Run here (where /root/reference exists) after `make -C oracle ref`:

    python tests/golden/make_golden.py

Every output below comes from oracle/_ref/libbelief_ref.so, i.e. the reference's
sparse.cpp / gabp.cpp / schedule.cpp / problems.cpp / analysis.cpp compiled with its
Release flags (multigrid entries: the Eigen-free restatement over the reference engine).
Inputs come from the seeded generators restated from proj/tests/oracles.hpp; their
digests are stored too so a generator drift is caught separately from an engine drift.

Files: golden.npz (arrays) and golden.json (scalars + SHA-256 digests of arrays).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle.oracle import (Oracle, Schedule, MG_GABP_RB, MG_GABP_FC, MG_GABP_SEQ, MG_GS_RB,  # noqa: E402
                           MG_GABP_FLOOD)
from tests.cases import CASES, build_case  # noqa: E402


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    F = Oracle.reference()
    R = Oracle.restatement()
    if F is None:
        raise SystemExit("oracle/_ref/libbelief_ref.so missing: run `make -C oracle ref` first")
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"source": "oracle/_ref/libbelief_ref.so (reference sources, Release flags)", "cases": {}}

    # ---- per-sweep flood / ordered sweeps on every registered case -------------------------
    for name, spec in CASES.items():
        A, b, sched = build_case(R, name)
        e = F.engine(A)
        lam, m = e.make_state()
        x = np.zeros(A.n)
        rec = {"n": A.n, "nnz": A.nnz, "num_edges": e.num_edges, "input": digest(A.values) + digest(b),
               "sweeps": spec["sweeps"], "digests": [], "ok": []}
        for s in range(spec["sweeps"]):
            ok, err = e.sweep(b, sched, lam, m, x)
            beta = e.node_precisions(lam, m)
            r = F.residual_inf_norm(A, x, b)
            rec["digests"].append([digest(lam), digest(m), digest(x), digest(beta), float(r).hex()])
            rec["ok"].append([bool(ok), err])
            if s + 1 in spec.get("keep", ()):
                for k, v in (("lam", lam), ("m", m), ("x", x), ("beta", beta)):
                    arrays[f"{name}/{s + 1}/{k}"] = v.copy()
            if not ok:
                break
        meta["cases"][name] = rec

    # ---- solve() reports -------------------------------------------------------------------
    solves = {}
    for name, tol, max_iter, stop in [("poisson9_flood", 1e-10, 2000, 0), ("poisson9_rb", 1e-10, 2000, 0),
                                      ("dd25_nonsym_flood", 1e-12, 5000, 0), ("dd25_nonsym_seq", 1e-12, 5000, 0),
                                      ("dd20_sym_flood", 1e-12, 5000, 1), ("ex7x7_flood", 2e-4, 5000, 0),
                                      ("ex7x7_seq", 2e-4, 5000, 0), ("pivot2_seq", 2e-4, 50, 0),
                                      ("pivot2_flood", 2e-4, 50, 0), ("poisson64_flood", None, 300, 0)]:
        A, b, sched = build_case(R, name)
        if tol is None:
            tol = 1e-8 * np.abs(b).max()
        rep = F.engine(A).solve(b, sched, tol=tol, max_iter=max_iter, stop=stop)
        solves[name] = {"tol": tol, "max_iter": max_iter, "stop": stop, "status": rep.status,
                        "iterations": rep.iterations, "detail": rep.detail, "flops": rep.flop_estimate,
                        "history": [float(v).hex() for v in rep.residual_history], "x": digest(rep.solution)}
        arrays[f"solve/{name}/x"] = rep.solution
    meta["solves"] = solves

    # ---- frozen-lambda path (precompute_lambda / correction_sweeps / error correction) ------
    frozen = {}
    for name in ("poisson9_rb", "poisson9_flood", "dd25_nonsym_seq"):
        A, b, sched = build_case(R, name)
        e = F.engine(A)
        lam, sig, conv, its = e.precompute_lambda(sched, 1e-10, 500)
        ec = e.correction_sweeps(b, sched, lam, sig, 3)
        rep = e.solve_error_correction(b, sched, 2, lam, sig, tol=1e-10, max_iter=3000)
        frozen[name] = {"converged": conv, "iterations": its, "lam": digest(lam), "sigma": digest(sig),
                        "corr3": digest(ec), "ec_status": rep.status, "ec_iterations": rep.iterations,
                        "ec_history": [float(v).hex() for v in rep.residual_history]}
        arrays[f"frozen/{name}/lam"] = lam
        arrays[f"frozen/{name}/sigma"] = sig
        arrays[f"frozen/{name}/corr3"] = ec
    meta["frozen"] = frozen

    # ---- computation-tree values (analysis.cpp:196-215) -----------------------------------
    rng = R.rng(29)
    ctree = []
    for trial in range(4):
        A = rng.diag_dominant(6 + trial % 3, trial % 2 == 0, 0.5)
        b = rng.vector(A.n)
        ctree.append([[float(F.computation_tree_solve(A, b, root, d)).hex() for root in range(A.n)]
                      for d in range(1, 6)])
    meta["computation_tree"] = ctree

    # ---- multigrid transfers + small V-cycle solves ------------------------------------------
    g = R.rng(33)
    u = g.vector(49)
    v = g.vector(9)
    arrays["mg/restrict7"] = F.mg_restrict(u, 7)
    arrays["mg/prolong3"] = F.mg_prolong(v, 3)
    mg = {}
    for prob, J1, J2, sm, pre, post in [("poisson", 5, 3, MG_GABP_RB, 2, 2), ("poisson", 5, 3, MG_GABP_SEQ, 1, 1),
                                        ("poisson", 5, 3, MG_GABP_FC, 1, 1), ("poisson", 5, 3, MG_GS_RB, 2, 2),
                                        ("poisson", 5, 3, MG_GABP_FLOOD, 2, 2),
                                        ("boundary-layer", 6, 6, MG_GABP_RB, 5, 0)]:
        levels, nxs = [], []
        for J in range(J1, J1 - J2, -1):
            Al, bl, _, nx, _ = F.assemble(prob, J, {"eps": 0.01} if prob == "boundary-layer" else {})
            levels.append(Al)
            nxs.append(nx)
            if J == J1:
                b = bl
        H = F.hierarchy(levels, nxs, sm)
        rep = H.solve(pre, post, b, tol=1e-8 * np.abs(b).max(), max_cycles=60)
        key = f"{prob}/{J1}/{J2}/{sm}/{pre}{post}"
        mg[key] = {"levels": H.num_levels, "status": rep.status, "iterations": rep.iterations,
                   "history": [float(h).hex() for h in rep.residual_history], "x": digest(rep.solution)}
    meta["mg"] = mg

    # ---- problem assembly (problems.cpp:161-226) ------------------------------------------
    asm = {}
    for prob, params in [("poisson", {}), ("anisotropic", {}), ("general", {}), ("mixed", {}),
                         ("boundary-layer", {"eps": 0.01}), ("inner-layer", {}), ("stretched", {})]:
        A, b, exact, nx, h = F.assemble(prob, 4, params)
        asm[prob] = {"params": params, "nx": nx, "h": h, "ro": digest(A.row_offsets), "ci": digest(A.col_indices),
                     "v": digest(A.values), "b": digest(b), "exact": digest(exact)}
    meta["assemble"] = asm

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays;", os.path.getsize(os.path.join(HERE, "golden.npz")) // 1024, "KiB")


if __name__ == "__main__":
    main()
