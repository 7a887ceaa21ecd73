"""The device build of the DIA layout (build_kernels.cuh) against the host build of the same
matrix (BGABP_HOST_BUILD=1, the engine's original host layout code): identical device arrays,
slot map and derived facts (bit-symmetry, constant-coefficient stencil, 5-point grid), and
identical solves.  The host build follows make_csr/transpose_pos (sparse.cpp:36-75) and
build_message_graph (gabp.cpp:8-27) literally; the device build scatters each entry A_ij into
node i's in-slot and node j's out-slot instead of searching for transpose partners."""
import os

import numpy as np
import pytest

import paper_1904_04093_b200 as g
from tests.cases import CASES, build_case

pytestmark = pytest.mark.gpu


def _digest(A, host):
    old = os.environ.pop("BGABP_HOST_BUILD", None)
    try:
        if host:
            os.environ["BGABP_HOST_BUILD"] = "1"
        eng = g.GabpEngine(A)
        return eng.layout_digest(), eng.info
    finally:
        os.environ.pop("BGABP_HOST_BUILD", None)
        if old is not None:
            os.environ["BGABP_HOST_BUILD"] = old


def _wrapped_grid(orc):
    """poisson5(8, 8) plus couplings between the last node of a row and the first of the next:
    the offsets stay {-8, -1, 1, 8} but the sequential pipeline's grid assumption fails."""
    A = orc.poisson5(8, 8)
    rows, cols, vals = [], [], []
    for i in range(A.n):
        for p in range(A.row_offsets[i], A.row_offsets[i + 1]):
            rows.append(i)
            cols.append(int(A.col_indices[p]))
            vals.append(float(A.values[p]))
    for r in range(7):
        i = 8 * r + 7
        rows += [i, i + 1]
        cols += [i + 1, i]
        vals += [-0.5, -0.5]
    return orc.make_csr(A.n, rows, cols, vals)


def _matrices(orc):
    out = {name: build_case(orc, name)[0] for name in sorted(CASES)}
    out["wrapped_grid"] = _wrapped_grid(orc)
    out["poisson_33x17"] = g.poisson5(33, 17)
    out["config3_64"] = g.config_problem(3, 64).A
    out["config4_12"] = g.config_problem(4, 12).A
    out["config5_J7_l0"] = g.config5_level(7, 0).A
    out["config5_J7_l2"] = g.config5_level(7, 2).A
    return out


def test_device_build_equals_host_build(orc):
    seen_dia = 0
    for name, A in _matrices(orc).items():
        dd, info_d = _digest(A, False)
        dh, info_h = _digest(A, True)
        info_d.pop("device_bytes"), info_h.pop("device_bytes")  # the device build keeps the CSR in HBM
        assert info_d == info_h, name
        assert dd == dh, f"{name}: device layout differs from the host build"
        seen_dia += info_d["layout"] == int(g.Layout.Dia)
    assert seen_dia >= 10


def test_device_build_facts(orc):
    """Facts the kernel variants key on, as the host build derives them."""
    e = g.GabpEngine(g.poisson5(64, 64))
    assert e.info["symmetric_values"] == 1 and e.info["uniform_coefficients"] == 1
    e = g.GabpEngine(g.config_problem(3, 32).A)
    assert e.info["symmetric_values"] == 0 and e.info["uniform_coefficients"] == 0
    e = g.GabpEngine(g.config5_level(6, 0).A)
    assert e.info["symmetric_values"] == 1 and e.info["uniform_coefficients"] == 0


def test_device_built_engine_solves_like_host_built(orc):
    """A solve on a lazily host-materialised engine (greedy colouring needs the host union lists)
    equals one on the host-built engine, bit for bit."""
    A = g.config_problem(3, 24).A
    b = orc.rng(5).vector(A.n)
    reps = []
    for host in (False, True):
        if host:
            os.environ["BGABP_HOST_BUILD"] = "1"
        try:
            eng = g.GabpEngine(A)
        finally:
            os.environ.pop("BGABP_HOST_BUILD", None)
        perm = np.random.RandomState(3).permutation(A.n)
        scheds = (g.Schedule.parallel_flood(), g.Schedule.red_black(), g.Schedule.red_black_grid(24, 24),
                  g.Schedule.sequential(), g.Schedule.custom(perm))
        for sched in scheds:
            rep = eng.solve(b, sched, g.GabpOptions(tol=1e-8 * np.abs(b).max(), max_iter=4000))
            st = eng.get_state()
            reps.append((int(rep.status), rep.iterations, rep.solution.tobytes(), st.m.tobytes()))
    assert reps[:5] == reps[5:]


@pytest.mark.parametrize("cfg", [2, 4])
def test_device_build_equals_host_build_full_size(cfg):
    """BASELINE.json configs 2 (4.2M nodes, 21M entries) and 4 (16.8M nodes, 117M entries, 7-point,
    variable coefficients): the device-built layout equals the host-built one bit for bit."""
    A = g.config_problem(cfg).A
    dd, info_d = _digest(A, False)
    dh, info_h = _digest(A, True)
    info_d.pop("device_bytes"), info_h.pop("device_bytes")
    assert info_d == info_h
    assert dd == dh
