"""BASELINE.json configs 2-4 on the GPU against the CPU oracle: full-solve parity at reduced sizes,
checkpoint parity and size-independent properties at the configured sizes."""
import numpy as np
import pytest

import paper_1904_04093_b200 as g
from oracle.oracle import Csr, Schedule as OSched
from tests.parity import assert_close

pytestmark = pytest.mark.gpu


def ocsr(A):
    return Csr(A.n, A.row_offsets, A.col_indices, A.values)


def _oracle(orc, ref):
    return ref if ref is not None else orc


@pytest.mark.parametrize("N", [48, 96])
def test_config3_nonsymmetric_full_solve_bitwise(orc, ref, N):
    """Config 3 recipe (upwind, cell Peclet 2, nonsymmetric values): flood solve to 1e-8 equal to
    the reference sweep for sweep -- iterations, full residual history, solution."""
    O = _oracle(orc, ref)
    p = g.config_problem(3, size=N)
    eng = g.GabpEngine(p.A)
    assert eng.info["symmetric_values"] == 0 and eng.layout == g.Layout.Dia
    tol = 1e-8 * np.abs(p.b).max()
    got = eng.solve(p.b, g.Schedule.parallel_flood(), g.GabpOptions(tol=tol, max_iter=20000))
    want = O.engine(ocsr(p.A)).solve(p.b, OSched.parallel_flood(), tol=tol, max_iter=20000)
    assert got.status == g.SolveStatus.Converged
    assert (int(got.status), got.iterations) == (want.status, want.iterations)
    assert got.residual_history.tobytes() == want.residual_history.tobytes()
    assert got.solution.tobytes() == want.solution.tobytes()


def test_config3_full_size_checkpoints_and_solve(orc, ref):
    """Config 3 at 1024^2: the first sweeps bit-identical to the oracle; the solve reaches
    rel. residual 1e-8 and the CPU-evaluated residual of the returned x confirms it."""
    O = _oracle(orc, ref)
    p = g.config_problem(3)
    assert p.A.n == 1024 * 1024
    eng = g.GabpEngine(p.A)
    oe = O.engine(ocsr(p.A))
    lam, m = oe.make_state()
    xr = np.zeros(p.A.n)
    x = np.zeros(p.A.n)
    for s in range(3):
        assert eng.sweep_resident(p.b, g.Schedule.parallel_flood(), x)[0]
        oe.sweep(p.b, OSched.parallel_flood(), lam, m, xr)
        st = eng.get_state()
        assert_close(st.lambda_tilde, lam, f"lambda@{s + 1}", bitwise=True)
        assert_close(st.m, m, f"m@{s + 1}", bitwise=True)
        assert_close(x, xr, f"x@{s + 1}", bitwise=True)
    tol = 1e-8 * np.abs(p.b).max()
    rep = eng.solve(p.b, g.Schedule.parallel_flood(), g.GabpOptions(tol=tol, max_iter=20000))
    assert rep.status == g.SolveStatus.Converged
    r = O.residual_inf_norm(ocsr(p.A), rep.solution, p.b)
    assert r == rep.residual_history[-1] and r <= tol
    assert rep.residual_history[-2] > tol  # it stopped at the first iteration below tol


def test_config4_small_300_sweeps_bitwise(orc, ref):
    """Config 4 recipe (3D 7-point, lognormal K, harmonic faces, (1,1,0.01)) at 20^3: 300 flood
    sweeps, x and the residual bit-identical to the oracle at every 50th sweep."""
    O = _oracle(orc, ref)
    p = g.config_problem(4, size=20)
    eng = g.GabpEngine(p.A)
    assert eng.layout == g.Layout.Dia and eng.info["num_slots"] == 6 and eng.info["symmetric_values"] == 1
    oe = O.engine(ocsr(p.A))
    lam, m = oe.make_state()
    xr = np.zeros(p.A.n)
    x = np.zeros(p.A.n)
    for s in range(300):
        eng.sweep_resident(p.b, g.Schedule.parallel_flood(), x)
        oe.sweep(p.b, OSched.parallel_flood(), lam, m, xr)
        if (s + 1) % 50 == 0:
            assert x.tobytes() == xr.tobytes(), s + 1
            st = eng.get_state()
            assert st.m.tobytes() == m.tobytes() and st.lambda_tilde.tobytes() == lam.tobytes()
    rep = eng.solve(p.b, g.Schedule.parallel_flood(), g.GabpOptions(tol=0.0, max_iter=300))
    want = oe.solve(p.b, OSched.parallel_flood(), tol=0.0, max_iter=300)
    assert rep.iterations == want.iterations == 300
    assert rep.residual_history.tobytes() == want.residual_history.tobytes()


def test_config4_full_size_checkpoint(orc, ref):
    """Config 4 at 256^3 (16.8M unknowns, 117M nonzeros): sweeps 1-2 bit-identical to the oracle
    (the CPU needs ~3 s per sweep), then the fixed 300-sweep run: residual history finite and the
    CPU residual of the returned x equal to the last entry."""
    O = _oracle(orc, ref)
    p = g.config_problem(4)
    assert p.A.n == 256 ** 3 and p.A.nnz == 117047296
    eng = g.GabpEngine(p.A)
    assert eng.num_edges == 100270080
    oe = O.engine(ocsr(p.A))
    lam, m = oe.make_state()
    xr = np.zeros(p.A.n)
    x = np.zeros(p.A.n)
    for s in range(2):
        assert eng.sweep_resident(p.b, g.Schedule.parallel_flood(), x)[0]
        oe.sweep(p.b, OSched.parallel_flood(), lam, m, xr)
    assert x.tobytes() == xr.tobytes()
    st = eng.get_state()
    assert st.m.tobytes() == m.tobytes()
    del lam, m, st
    rep = eng.solve(p.b, g.Schedule.parallel_flood(), g.GabpOptions(tol=0.0, max_iter=300))
    assert rep.status == g.SolveStatus.MaxIter and rep.iterations == 300
    assert np.all(np.isfinite(rep.residual_history))
    assert O.residual_inf_norm(ocsr(p.A), rep.solution, p.b) == rep.residual_history[-1]
    assert rep.residual_history[-1] < 0.2 * rep.residual_history[0]  # 0.12 r0 after 300 sweeps


def test_config2_full_size_checkpoints(orc, ref):
    """Config 2 at 2048^2: sweeps 1 and 10 bit-identical (SURVEY §8(d) checkpoint parity) and the
    device residual equal to the CPU residual of the same x."""
    O = _oracle(orc, ref)
    p = g.config_problem(2)
    eng = g.GabpEngine(p.A)
    oe = O.engine(ocsr(p.A))
    lam, m = oe.make_state()
    xr = np.zeros(p.A.n)
    x = np.zeros(p.A.n)
    for s in range(10):
        eng.sweep_resident(p.b, g.Schedule.parallel_flood(), x)
        oe.sweep(p.b, OSched.parallel_flood(), lam, m, xr)
        if s in (0, 9):
            st = eng.get_state()
            assert st.lambda_tilde.tobytes() == lam.tobytes() and st.m.tobytes() == m.tobytes()
            assert x.tobytes() == xr.tobytes()
    assert eng.residual_inf_norm(x, p.b) == O.residual_inf_norm(ocsr(p.A), xr, p.b)
    tol = 1e-8 * np.abs(p.b).max()
    rep = eng.solve(p.b, g.Schedule.parallel_flood(), g.GabpOptions(tol=tol, max_iter=60))
    want = oe.solve(p.b, OSched.parallel_flood(), tol=tol, max_iter=60)
    assert (int(rep.status), rep.iterations) == (want.status, want.iterations) == (2, 60)
    assert rep.residual_history.tobytes() == want.residual_history.tobytes()
