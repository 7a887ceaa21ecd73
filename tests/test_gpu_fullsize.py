"""Full-size parity of BASELINE.json configs 2-4: the GPU solve loop against the
CPU oracle at the configured sizes, bit for bit -- every iteration's residual, the status, the
iteration count and x.

The checker is the restatement (oracle/gabp_restate.cpp) with its flood sweep evaluated by OpenMP
threads: the same per-node arithmetic on the same snapshot, pinned bitwise to the
reference's compiled engine by tests/test_oracle.py.  With BGABP_FULLSIZE_REF=1 the checker is the
reference's own compiled engine (oracle/_ref, one thread; ~10 min on the GPU box's host) instead.
"""
import os

import numpy as np
import pytest

import paper_1904_04093_b200 as g
from oracle.oracle import Oracle, Schedule as OSched

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def checker():
    if os.environ.get("BGABP_FULLSIZE_REF") == "1":
        o = Oracle.reference()
        if o is None:
            pytest.skip("oracle/_ref not built")
        return o
    o = Oracle.restatement()
    o.set_threads(os.cpu_count() or 1)
    return o


def _compare(checker, P, tol, cap, stop=0, config=None):
    # the checker's input from the oracle's own generators (equal to the product's, bit for bit)
    A, b = Oracle.restatement().config_problem(config)
    assert np.array_equal(A.row_offsets, P.A.row_offsets) and np.array_equal(A.col_indices, P.A.col_indices)
    assert A.values.tobytes() == P.A.values.tobytes() and b.tobytes() == P.b.tobytes()
    got = g.GabpEngine(P.A).solve(P.b, g.Schedule.parallel_flood(), g.GabpOptions(tol=tol, max_iter=cap, stop=stop))
    want = checker.engine(A).solve(b, OSched.parallel_flood(), tol=tol, max_iter=cap, stop=stop)
    assert (int(got.status), got.iterations, got.detail) == (want.status, want.iterations, want.detail)
    assert got.residual_history.tobytes() == want.residual_history.tobytes()
    assert got.solution.tobytes() == want.solution.tobytes()
    assert got.flop_estimate == want.flop_estimate
    return got


@pytest.mark.parametrize("checkpoint", [100, 500])
def test_config2_checkpoints(checker, checkpoint):
    """poisson5(2048, 2048), b ~ U[-1,1] seed 1: iterations 1..100 and 1..500 of the solve loop
    (the tolerance 1e-8 ||b|| needs ~6.7M sweeps, so both stop at the cap)."""
    P = g.config_problem(2)
    rep = _compare(checker, P, 1e-8 * np.abs(P.b).max(), checkpoint, config=2)
    assert rep.status == g.SolveStatus.MaxIter and rep.iterations == checkpoint


def test_config3_full_solve_to_1e8(checker):
    """1024^2 upwind convection-diffusion, nonsymmetric GaBP to rel. residual 1e-8: the same
    iteration count (1967) and every residual of the way, bit for bit."""
    P = g.config_problem(3)
    rep = _compare(checker, P, 1e-8 * np.abs(P.b).max(), 20000, config=3)
    assert rep.status == g.SolveStatus.Converged and rep.iterations == 1967


def test_config4_twenty_sweeps(checker):
    """256^3 anisotropic lognormal diffusion (100M edges), 20 sweeps of the solve loop."""
    P = g.config_problem(4)
    rep = _compare(checker, P, 0.0, 20, config=4)
    assert rep.iterations == 20
