"""Optional message damping (BASELINE.json north_star "optional damping"; the reference has none,
SPEC.md:197).  Off (the default, or set back to 0) must be the reference bit for bit; on, every
flood sweep and solve must equal the restated damped oracle (oracle/gabp_restate.cpp emit: new <-
(1 - a) new + a old, products rounded before the add) bit for bit, on both device layouts and on
every fused-step variant (symmetric, nonsymmetric, constant-coefficient, message-delta stop)."""
import numpy as np
import pytest

import paper_1904_04093_b200 as g
from oracle.oracle import Schedule as OSched
from tests.cases import CASES, build_case

pytestmark = pytest.mark.gpu
LAYOUTS = [g.Layout.Auto, g.Layout.Csr]
FLOOD = [n for n in sorted(CASES) if n.endswith("_flood") or n == "config1"]


def _pair(orc, A, alpha, layout):
    eng = g.GabpEngine(A, layout)
    eng.set_damping(alpha)
    ref = orc.engine(A)
    ref.set_damping(alpha)
    return eng, ref


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("alpha", [0.25, 0.5, 0.7])
def test_damped_sweeps_match_damped_oracle(orc, layout, alpha):
    for name in FLOOD:
        A, b, sched = build_case(orc, name)
        if sched.kind != 0:
            continue
        eng, ref = _pair(orc, A, alpha, layout)
        st = eng.make_state()
        lam, m = ref.make_state()
        x, xr = np.zeros(A.n), np.zeros(A.n)
        for s in range(12):
            ok = eng.sweep(b, g.Schedule.parallel_flood(), st, x)
            okr = ref.sweep(b, OSched.parallel_flood(), lam, m, xr)
            assert tuple(ok) == tuple(okr), (name, s)
            assert st.lambda_tilde.tobytes() == lam.tobytes() and st.m.tobytes() == m.tobytes(), (name, s)
            assert x.tobytes() == xr.tobytes(), (name, s)
            if not ok[0]:
                break


def _problems(orc):
    yield "poisson5 48^2 (constant stencil)", g.config_problem(2, size=48).A, orc.rng(1).vector(48 * 48)
    p3 = g.config_problem(3, size=40)
    yield "upwind 40^2 (nonsymmetric)", p3.A, p3.b
    p4 = g.config_problem(4, size=12)
    yield "3-D lognormal 12^3 (7-point)", p4.A, p4.b


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("stop", [g.StopCriterion.Residual, g.StopCriterion.MessageDelta])
def test_damped_solves_match_damped_oracle(orc, layout, stop):
    """The fused DIA solve step (damped variant) and the union-CSR solve loop."""
    for name, A, b in _problems(orc):
        from oracle.oracle import Csr
        Ao = Csr(A.n, A.row_offsets, A.col_indices, A.values)
        for alpha in (0.3, 0.6):
            eng, ref = _pair(orc, Ao, alpha, layout)
            tol = 1e-8 * np.abs(b).max()
            got = eng.solve(b, g.Schedule.parallel_flood(), g.GabpOptions(tol=tol, max_iter=400, stop=stop))
            want = ref.solve(b, OSched.parallel_flood(), tol=tol, max_iter=400, stop=int(stop))
            assert (int(got.status), got.iterations, got.detail) == (want.status, want.iterations, want.detail), name
            assert got.residual_history.tobytes() == want.residual_history.tobytes(), name
            assert got.solution.tobytes() == want.solution.tobytes(), name


def test_damping_off_is_the_reference_bitwise(orc, golden):
    """Setting damping and then 0 again leaves the reference's results (golden solve reports)."""
    A, b, _ = build_case(orc, "config1")
    eng = g.GabpEngine(A)
    tol = 1e-8 * np.abs(b).max()
    plain = eng.solve(b, g.Schedule.parallel_flood(), g.GabpOptions(tol=tol, max_iter=300))
    eng.set_damping(0.5)
    damped = eng.solve(b, g.Schedule.parallel_flood(), g.GabpOptions(tol=tol, max_iter=300))
    eng.set_damping(0.0)
    again = eng.solve(b, g.Schedule.parallel_flood(), g.GabpOptions(tol=tol, max_iter=300))
    assert plain.residual_history.tobytes() == again.residual_history.tobytes()
    assert plain.solution.tobytes() == again.solution.tobytes()
    assert damped.residual_history.tobytes() != plain.residual_history.tobytes()
    want = orc.engine(A).solve(b, OSched.parallel_flood(), tol=tol, max_iter=300)
    assert again.residual_history.tobytes() == want.residual_history.tobytes()


def test_damping_rejects_ordered_schedules_and_bad_factors(orc):
    A, b, _ = build_case(orc, "config1")
    eng = g.GabpEngine(A)
    for bad in (-0.1, 1.0, float("nan")):
        with pytest.raises(ValueError, match="damping"):
            eng.set_damping(bad)
    eng.set_damping(0.5)
    with pytest.raises(ValueError, match="flood schedule only"):
        eng.solve(b, g.Schedule.red_black_grid(64, 64), g.GabpOptions(max_iter=3))
    st = eng.make_state()
    with pytest.raises(ValueError, match="flood schedule only"):
        eng.sweep(b, g.Schedule.sequential(), st, np.zeros(A.n))
