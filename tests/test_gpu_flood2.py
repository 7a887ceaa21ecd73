"""The two-iteration flood solve launches (flood2_kernels.cuh: the column-walking k_flood2_grid5
and the banded k_flood2b_grid5) against the CPU oracle and against the one-iteration fused step: GabpEngine::solve
(gabp.cpp:174-219) statuses, iteration counts, details, residual histories and x, bit for bit, on
5-point grids of every tile-boundary shape, uniform / variable / nonsymmetric coefficients,
convergence at odd and even iterations, max_iter caps, pivot breakdowns and residual blowups."""
import os

import numpy as np
import pytest

import paper_1904_04093_b200 as g
from oracle.oracle import Csr, Schedule as OSched

pytestmark = pytest.mark.gpu


def _csr_to_orc(A):
    return Csr(A.n, A.row_offsets, A.col_indices, A.values)


def _triplets(A):
    rows, cols, vals = [], [], []
    for i in range(A.n):
        for p in range(A.row_offsets[i], A.row_offsets[i + 1]):
            rows.append(i)
            cols.append(int(A.col_indices[p]))
            vals.append(float(A.values[p]))
    return rows, cols, vals


def _solve(A, b, tol, max_iter, kind):
    """kind: "single" (one iteration per launch), "col" (k_flood2_grid5), "band" (k_flood2b_grid5)"""
    os.environ["BGABP_FLOOD2"] = "0" if kind == "single" else "1"
    os.environ["BGABP_FLOOD2_KIND"] = kind
    try:
        eng = g.GabpEngine(A)
        return eng.solve(b, g.Schedule.parallel_flood(), g.GabpOptions(tol=tol, max_iter=max_iter))
    finally:
        os.environ.pop("BGABP_FLOOD2", None)
        os.environ.pop("BGABP_FLOOD2_KIND", None)


def _check(orc, A, b, tol, max_iter):
    reps = [_solve(A, b, tol, max_iter, k) for k in ("col", "band", "single")]
    want = orc.engine(_csr_to_orc(A)).solve(b, OSched.parallel_flood(), tol=tol, max_iter=max_iter)
    d = reps[0]
    for got in reps:
        assert (int(got.status), got.iterations, got.detail) == (want.status, want.iterations, want.detail)
        assert np.array_equal(got.residual_history, want.residual_history)
        assert np.array_equal(got.solution, want.solution)
    return d


@pytest.mark.parametrize("nx,ny", [(5, 3), (40, 30), (124, 7), (125, 66), (130, 129), (251, 64), (300, 200)])
def test_poisson_grids_match_oracle(orc, nx, ny):
    A = g.poisson5(nx, ny)
    b = orc.rng(nx * 1000 + ny).vector(A.n)
    for tol_rel, cap in ((1e-3, 20000), (1e-8, 20000), (0.0, 37), (0.0, 38)):
        _check(orc, A, b, tol_rel * np.abs(b).max(), cap)


def test_convergence_at_odd_and_even_iterations(orc):
    A = g.poisson5(48, 40)
    b = orc.rng(9).vector(A.n)
    parities = set()
    for tol_rel in (1e-2, 3e-3, 1e-3, 3e-4, 1e-4, 3e-5):
        rep = _check(orc, A, b, tol_rel * np.abs(b).max(), 20000)
        assert int(rep.status) == 0
        parities.add(rep.iterations % 2)
    assert parities == {0, 1}


@pytest.mark.parametrize("cfg,size", [(3, 96), (3, 130), (5, 0)])
def test_variable_and_nonsymmetric_coefficients(orc, cfg, size):
    P = g.config_problem(3, size) if cfg == 3 else g.config5_level(8, 1, sigma=1.0)
    b = P.b if P.b is not None else orc.rng(5).vector(P.A.n)
    for tol_rel, cap in ((1e-8, 20000), (0.0, 51)):
        _check(orc, P.A, b, tol_rel * np.abs(b).max(), cap)


def test_pivot_breakdown_matches_reference(orc):
    """poisson5(30, 20) with an isolated pair p-q (A_pp = A_qq = A_pq = A_qp = 1): q's precision
    cancels in sweep 2 exactly as test_gabp.cpp:73-85's 2x2 system."""
    A = g.poisson5(30, 20)
    rows, cols, vals = _triplets(A)
    p, q = 7 * 30 + 11, 7 * 30 + 12
    keep = [(r, c, v) for r, c, v in zip(rows, cols, vals) if r not in (p, q) and c not in (p, q)]
    keep += [(p, p, 1.0), (q, q, 1.0), (p, q, 1.0), (q, p, 1.0)]
    r, c, v = zip(*keep)
    B = orc.make_csr(A.n, r, c, v)
    Bg = g.SparseMatrix(B.n, B.row_offsets, B.col_indices, B.values)
    b = orc.rng(4).vector(A.n)
    rep = _check(orc, Bg, b, 1e-8, 100)
    assert int(rep.status) == 1 and "pivot" in rep.detail


def test_residual_blowup_matches_reference(orc):
    """An indefinite 5-point operator (diagonal 2.5): flood GaBP diverges."""
    A = g.poisson5(33, 21)
    vals = np.where(A.col_indices == np.repeat(np.arange(A.n), np.diff(A.row_offsets)), 2.5, A.values)
    B = g.SparseMatrix(A.n, A.row_offsets, A.col_indices, vals)
    b = orc.rng(8).vector(A.n)
    rep = _check(orc, B, b, 1e-8, 3000)
    assert int(rep.status) == 1
