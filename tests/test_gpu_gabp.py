"""GPU parity of the GaBP engine against the CPU oracle and the golden vectors.

Mirrors the reference's own tests (proj/tests/test_gabp.cpp, test_sparse.cpp,
acceptance.cpp criterion 10) with the CUDA path as the system under test and the restated /
reference CPU code as the checker.
"""
import hashlib

import numpy as np
import pytest

import paper_1904_04093_b200 as g
from oracle.oracle import Schedule as OSched
from tests.cases import CASES, build_case, one_way_4x4, tree_5x5
from tests.parity import assert_close

pytestmark = pytest.mark.gpu


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gsched(s: OSched) -> g.Schedule:
    return g.Schedule(s.kind, s.nx, s.ny, s.order)


LAYOUTS = [g.Layout.Auto, g.Layout.Csr]


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("name", sorted(CASES))
def test_per_sweep_state_matches_golden_bitwise(orc, golden, name, layout):
    """GabpEngine::sweep after every sweep: lambda, m (CSR order), beta, x and the residual."""
    meta, arrays = golden
    rec = meta["cases"][name]
    A, b, sched = build_case(orc, name)
    eng = g.GabpEngine(A, layout)
    x = np.zeros(A.n)
    for s, want in enumerate(rec["digests"]):
        ok, err = eng.sweep_resident(b, gsched(sched), x)
        assert [ok, err] == rec["ok"][s], f"sweep {s + 1}"
        if not ok:  # the reference's partly updated x (gabp.cpp:71-87, 126-130, 155-158)
            assert digest(x) == want[2], f"{name} sweep {s + 1}: x after the breakdown"
            break
        st = eng.get_state()
        beta = eng.node_precisions()
        r = eng.residual_inf_norm(x, b)
        got = [digest(st.lambda_tilde), digest(st.m), digest(x), digest(beta), float(r).hex()]
        if got != want:  # report with the elementwise bar before failing on bits
            keep = f"{name}/{s + 1}"
            if keep + "/x" in arrays:
                for k, v in (("lam", st.lambda_tilde), ("m", st.m), ("x", x), ("beta", beta)):
                    assert_close(v, arrays[f"{keep}/{k}"], f"{name} sweep {s + 1} {k}")
        assert got == want, f"{name} sweep {s + 1}: not bit-identical to the reference"


def test_config1_full_state_every_sweep_against_oracle(orc):
    """Config 1 (BASELINE.json): poisson5(64,64), b~U[-1,1] seed 0, 200 flood sweeps, lambda, m,
    beta and x compared with the oracle after every sweep (rel 1e-10; expected bit-identical)."""
    A, b, sched = build_case(orc, "config1")
    eng = g.GabpEngine(A)
    assert eng.layout == g.Layout.Dia and eng.info["num_slots"] == 4
    ref = orc.engine(A)
    lam, m = ref.make_state()
    xr = np.zeros(A.n)
    x = np.zeros(A.n)
    nonbit = 0
    for s in range(200):
        ok, _ = eng.sweep_resident(b, g.Schedule.parallel_flood(), x)
        assert ok
        ref.sweep(b, sched, lam, m, xr)
        st = eng.get_state()
        nonbit += assert_close(st.lambda_tilde, lam, f"lambda@{s + 1}")
        nonbit += assert_close(st.m, m, f"m@{s + 1}")
        nonbit += assert_close(x, xr, f"x@{s + 1}")
        nonbit += assert_close(eng.node_precisions(), ref.node_precisions(lam, m), f"beta@{s + 1}")
    assert nonbit == 0
    rel = ref.o.residual_inf_norm(A, xr, b) / np.abs(b).max()
    assert abs(rel - 2.33e-2) < 1e-3  # rel. residual ~2.3e-2 after 200 sweeps


def test_sweep_with_caller_state_roundtrip(orc):
    """The reference signature sweep(b, sched, state, x) with a caller-owned MessageState."""
    A, b, sched = build_case(orc, "dd25_nonsym_flood")
    eng = g.GabpEngine(A)
    ref = orc.engine(A)
    st = eng.make_state()
    lam, m = ref.make_state()
    x, xr = np.zeros(A.n), np.zeros(A.n)
    for _ in range(7):
        assert eng.sweep(b, g.Schedule.parallel_flood(), st, x)[0]
        ref.sweep(b, sched, lam, m, xr)
    assert st.lambda_tilde.tobytes() == lam.tobytes() and st.m.tobytes() == m.tobytes()
    assert x.tobytes() == xr.tobytes()


SOLVES = ["poisson9_flood", "poisson9_rb", "dd25_nonsym_flood", "dd25_nonsym_seq", "dd20_sym_flood", "ex7x7_flood",
          "ex7x7_seq", "pivot2_seq", "pivot2_flood", "poisson64_flood"]


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("name", SOLVES)
def test_solve_report_matches_golden(orc, golden, name, layout):
    """solve(): status, iterations, detail, flop estimate and the whole residual history."""
    meta, _ = golden
    rec = meta["solves"][name]
    A, b, sched = build_case(orc, name)
    eng = g.GabpEngine(A, layout)
    rep = eng.solve(b, gsched(sched), g.GabpOptions(tol=rec["tol"], max_iter=rec["max_iter"], stop=rec["stop"]))
    assert (int(rep.status), rep.iterations, rep.detail) == (rec["status"], rec["iterations"], rec["detail"])
    assert [float(v).hex() for v in rep.residual_history] == rec["history"]
    assert rep.flop_estimate == rec["flops"]
    # on a pivot stop the reference returns a partly updated x (gabp.cpp:71-87, 126-130, 155-158):
    # every solve path keeps x(k-1) in a two-slot ring and composes it exactly
    assert digest(rep.solution) == rec["x"]


def test_solve_stop_rules_and_edges(orc):
    A = orc.poisson5(6, 6)
    b = orc.rng(3).vector(A.n)
    eng = g.GabpEngine(A)
    ref = orc.engine(A)
    # r0 <= tol: converged after 0 iterations, x = 0 (gabp.cpp:179-185)
    rep = eng.solve(b, g.Schedule.parallel_flood(), g.GabpOptions(tol=10.0))
    assert (rep.status, rep.iterations) == (g.SolveStatus.Converged, 0) and not rep.solution.any()
    # max_iter = 0 -> MaxIter immediately
    rep = eng.solve(b, g.Schedule.parallel_flood(), g.GabpOptions(tol=1e-30, max_iter=0))
    assert (rep.status, rep.iterations) == (g.SolveStatus.MaxIter, 0)
    # MessageDelta stop and tiny caps, every schedule
    for sched in (OSched.parallel_flood(), OSched.sequential(), OSched.red_black_grid(6, 6),
                  OSched.four_color_grid(6, 6)):
        for stop, tol, cap in ((1, 1e-9, 500), (0, 1e-9, 7), (0, 1e-9, 1), (1, 0.5, 50)):
            want = ref.solve(b, sched, tol=tol, max_iter=cap, stop=stop)
            got = eng.solve(b, gsched(sched), g.GabpOptions(tol=tol, max_iter=cap, stop=stop))
            assert (int(got.status), got.iterations) == (want.status, want.iterations), (sched.kind, stop, cap)
            assert got.residual_history.tobytes() == want.residual_history.tobytes()
            assert got.solution.tobytes() == want.solution.tobytes()


def test_diagonal_system_solves_in_one_sweep():
    """test_gabp.cpp:63-71"""
    D = g.SparseMatrix(2, np.array([0, 1, 2], np.int32), np.array([0, 1], np.int32), np.array([2.0, 4.0]))
    rep = g.GabpEngine(D).solve(np.array([2.0, 8.0]), g.Schedule.sequential(2), g.GabpOptions(tol=1e-14))
    assert rep.status == g.SolveStatus.Converged and rep.iterations == 1
    assert np.allclose(rep.solution, [1.0, 2.0])


def test_pivot_breakdown_is_divergence(orc):
    """test_gabp.cpp:73-85 through solve() and sweep()."""
    from tests.cases import pivot_2x2
    A = pivot_2x2(orc)
    eng = g.GabpEngine(A)
    rep = eng.solve(np.ones(2), g.Schedule.sequential(2), g.GabpOptions())
    assert rep.status == g.SolveStatus.Diverged and "pivot" in rep.detail
    x = np.zeros(2)
    eng.reset_state()
    ok, err = eng.sweep_resident(np.ones(2), g.Schedule.parallel_flood(), x)
    assert not ok and err == "zero pivot at node 0"


def test_schedule_errors_match_reference(orc):
    A = orc.poisson5(3, 3)
    eng = g.GabpEngine(A)
    x = np.zeros(9)
    with pytest.raises(ValueError, match="does not cover every node"):
        eng.sweep_resident(np.ones(9), g.Schedule.red_black_grid(4, 3), x)
    with pytest.raises(ValueError, match="not a permutation"):
        eng.sweep_resident(np.ones(9), g.Schedule.custom([0, 0, 1, 2, 3, 4, 5, 6, 7]), x)


def test_tree_exactness_and_hand_elimination(orc):
    """test_gabp.cpp:87-111: saturated tree messages equal hand elimination; x equals A^-1 b."""
    A = tree_5x5(orc)
    eng = g.GabpEngine(A)
    st = eng.make_state()
    x = np.zeros(5)
    for _ in range(10):
        assert eng.sweep(np.ones(5), g.Schedule.sequential(5), st, x)[0]
    D = A.dense()
    lam13 = -D[2, 0] * D[0, 2] / D[0, 0]
    lam23 = -D[2, 1] * D[1, 2] / D[1, 1]
    expected = -D[4, 2] * D[2, 4] / (D[2, 2] + lam13 + lam23)
    pos = int(np.where((np.repeat(np.arange(5), np.diff(A.row_offsets)) == 4) & (A.col_indices == 2))[0][0])
    assert abs(st.lambda_tilde[pos] * D[2, 4] - expected) <= 1e-12 * abs(expected)
    assert np.max(np.abs(x - np.linalg.solve(D, np.ones(5)))) < 1e-12
    rng = orc.rng(101)
    for trial in range(5):
        n = 20 + 36 * trial
        T, edges = rng.tree(n)
        diam = orc.tree_diameter(n, edges)
        bb = rng.vector(n)
        eng = g.GabpEngine(T)
        st = eng.make_state()
        x = np.zeros(n)
        for _ in range(2 * diam):
            assert eng.sweep(bb, g.Schedule.sequential(n), st, x)[0]
        assert np.max(np.abs(x - orc.dense_solve(T, bb))) < 1e-10


def test_flood_iterate_equals_computation_tree(orc):
    """acceptance.cpp:296-316 (criterion 10) with the GPU flood sweep."""
    rng = orc.rng(1010)
    for trial in range(10):
        n = rng.uniform_int(4, 8)
        A = rng.diag_dominant(n, trial % 2 == 0, 0.5)
        b = rng.vector(A.n)
        eng = g.GabpEngine(A)
        x = np.zeros(A.n)
        for depth in range(1, 6):
            assert eng.sweep_resident(b, g.Schedule.parallel_flood(), x)[0]
            for root in range(A.n):
                t = orc.computation_tree_solve(A, b, root, depth, 2000000)
                assert abs(t - x[root]) <= 1e-12 * max(1.0, abs(x[root]))


def test_message_graph_one_way_edges(orc):
    """test_gabp.cpp:43-61: 7 edges, node 3 sends but never receives."""
    A = one_way_4x4(orc)
    eng = g.GabpEngine(A)
    assert eng.num_edges == 7
    x = np.zeros(4)
    b = np.arange(1.0, 5.0)
    for _ in range(30):
        eng.sweep_resident(b, g.Schedule.parallel_flood(), x)
    assert np.max(np.abs(x - np.linalg.solve(A.dense(), b))) < 1e-10


def test_frozen_path_matches_golden(orc, golden):
    """precompute_lambda / correction_sweeps / solve_error_correction (gabp.cpp:221-401)."""
    meta, arrays = golden
    for name, rec in meta["frozen"].items():
        A, b, sched = build_case(orc, name)
        for layout in LAYOUTS:
            eng = g.GabpEngine(A, layout)
            fz = eng.precompute_lambda(gsched(sched), 1e-10, 500)
            assert (fz.converged, fz.iterations) == (rec["converged"], rec["iterations"])
            assert digest(fz.lambda_tilde) == rec["lam"], name
            assert digest(fz.sigma) == rec["sigma"], name
            e = eng.correction_sweeps(b, gsched(sched), fz, 3)
            assert digest(e) == rec["corr3"], name
            rep = eng.solve_error_correction(b, gsched(sched), 2, fz, g.GabpOptions(tol=1e-10, max_iter=3000))
            assert (int(rep.status), rep.iterations) == (rec["ec_status"], rec["ec_iterations"])
            assert [float(v).hex() for v in rep.residual_history] == rec["ec_history"]


def test_error_correction_known_answers(orc):
    """test_gabp.cpp:310-336: exact solution untouched; cold correction replays the iteration."""
    A = orc.poisson5(5, 5)
    b = orc.rng(13).vector(A.n)
    xs = orc.dense_solve(A, b)
    eng = g.GabpEngine(A)
    fz = eng.precompute_lambda(g.Schedule.sequential())
    assert np.max(np.abs(eng.error_correction_apply(b, xs, 3, g.Schedule.sequential(), fz) - xs)) < 1e-12
    A4 = orc.poisson5(4, 4)
    b4 = orc.rng(21).vector(A4.n)
    e4 = g.GabpEngine(A4)
    for k in (1, 3, 7):
        cold = e4.error_correction_apply(b4, np.zeros(A4.n), k, g.Schedule.sequential())
        st = e4.make_state()
        x = np.zeros(A4.n)
        for _ in range(k):
            e4.sweep(b4, g.Schedule.sequential(), st, x)
        assert np.max(np.abs(cold - x)) < 1e-14


def test_residual_inf_norm_known_answers(orc):
    """test_sparse.cpp:96-104"""
    I3 = g.SparseMatrix(3, np.array([0, 1, 2, 3], np.int32), np.arange(3, dtype=np.int32), np.ones(3))
    assert g.GabpEngine(I3).residual_inf_norm([1, 2, 3], [1, 2, 3]) == 0.0
    E = orc.example7x7()
    assert g.GabpEngine(E).residual_inf_norm(np.zeros(7), np.ones(7)) == 1.0


def test_empty_and_single_node_systems():
    E0 = g.SparseMatrix(0, np.array([0], np.int32), np.zeros(0, np.int32), np.zeros(0))
    rep = g.GabpEngine(E0).solve(np.zeros(0), g.Schedule.parallel_flood(), g.GabpOptions())
    assert rep.status == g.SolveStatus.Converged and rep.iterations == 0
    one = g.SparseMatrix(1, np.array([0, 1], np.int32), np.array([0], np.int32), np.array([4.0]))
    rep = g.GabpEngine(one).solve(np.array([2.0]), g.Schedule.parallel_flood(), g.GabpOptions(tol=1e-15))
    assert rep.status == g.SolveStatus.Converged and rep.solution[0] == 0.5


def test_device_stepping_api_equals_host_solve(orc):
    import torch
    A = orc.poisson5(40, 40)
    b = orc.rng(8).vector(A.n)
    eng = g.GabpEngine(A)
    tol = 1e-8 * np.abs(b).max()
    want = eng.solve(b, g.Schedule.parallel_flood(), g.GabpOptions(tol=tol, max_iter=100000))
    bd = torch.tensor(b, device="cuda")
    xd = torch.zeros(A.n, dtype=torch.float64, device="cuda")
    eng.solve_device_begin(bd.data_ptr(), g.Schedule.parallel_flood(), g.GabpOptions(tol=tol, max_iter=100000))
    eng.solve_device_steps(want.iterations + 40)
    status, its, _, _ = eng.solve_device_end(xd.data_ptr())
    assert (status, its) == (want.status, want.iterations)
    assert xd.cpu().numpy().tobytes() == want.solution.tobytes()


@pytest.mark.parametrize("kind", ["chain", "mixed9", "general", "zeros4"])
def test_fused_solve_every_slot_count(orc, ref, kind):
    """The fused DIA solve step for S = 2 (1-D chain), 8 (9-point 'mixed' problem, nonsymmetric
    'general' convection) and tiny explicit-zero matrices: whole solve report bit-identical."""
    O = ref if ref is not None else orc
    if kind == "chain":
        n = 300
        rows = [i for i in range(n) for _ in range(3)]
        cols = [min(max(i + d, 0), n - 1) for i in range(n) for d in (-1, 0, 1)]
        vals = [(2.5 if d == 0 else -1.0) for i in range(n) for d in (-1, 0, 1)]
        A = orc.make_csr(n, rows, cols, vals)
        b = orc.rng(2).vector(n)
    elif kind == "zeros4":
        from tests.cases import explicit_zeros
        A = explicit_zeros(orc)
        b = orc.rng(4).vector(4)
    else:
        p = g.assemble("mixed" if kind == "mixed9" else "general", 5)
        from oracle.oracle import Csr
        A = Csr(p.A.n, p.A.row_offsets, p.A.col_indices, p.A.values)
        b = p.b
    eng = g.GabpEngine(A)
    tol = 1e-9 * np.abs(b).max()
    for stop in (0, 1):
        got = eng.solve(b, g.Schedule.parallel_flood(), g.GabpOptions(tol=tol, max_iter=4000, stop=stop))
        want = O.engine(A).solve(b, OSched.parallel_flood(), tol=tol, max_iter=4000, stop=stop)
        assert (int(got.status), got.iterations, got.detail) == (want.status, want.iterations, want.detail), kind
        assert got.residual_history.tobytes() == want.residual_history.tobytes()
        if want.status != 1:
            assert got.solution.tobytes() == want.solution.tobytes()


# ---- pipelined lexicographic solve (seqpipe_kernels.cuh): many sweeps per launch ---------------
def _ocsr(orc, A):
    from oracle.oracle import Csr
    return Csr(A.n, A.row_offsets, A.col_indices, A.values)


def _same_report(got, want):
    assert (int(got.status), got.iterations, got.detail) == (want.status, want.iterations, want.detail)
    assert got.residual_history.tobytes() == want.residual_history.tobytes()
    assert got.solution.tobytes() == want.solution.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("stop,tol", [(0, 1e-8), (1, 1e-9)])
def test_sequential_pipeline_nonsymmetric_grid(orc, ref, stop, tol):
    """Config-3 style upwind operator (bit-nonsymmetric): residual rows read A_{j,k}, not A_{k,j}."""
    o = ref or orc
    p = g.config_problem(3, size=40)
    want = o.engine(_ocsr(o, p.A)).solve(p.b, OSched.sequential(), tol=tol, max_iter=5000, stop=stop)
    got = g.GabpEngine(p.A).solve(p.b, g.Schedule.sequential(), g.GabpOptions(tol=tol, max_iter=5000, stop=stop))
    assert want.status == 0
    _same_report(got, want)


@pytest.mark.gpu
def test_sequential_pipeline_long_solve_wraps_the_ring(orc, ref):
    """Poisson 64^2 to 1e-8: ~2900 pipelined sweeps over many launches and ring wrap-arounds."""
    o = ref or orc
    A = orc.poisson5(64, 64)
    b = orc.rng(0).vector(A.n)
    want = o.engine(A).solve(b, OSched.sequential(), tol=1e-8, max_iter=20000)
    got = g.GabpEngine(A).solve(b, g.Schedule.sequential(), g.GabpOptions(tol=1e-8, max_iter=20000))
    assert want.status == 0 and want.iterations > 1000
    _same_report(got, want)


@pytest.mark.gpu
def test_sequential_pipeline_pivot_stop_returns_the_partial_x(orc, ref):
    """Node 1's precision cancels in sweep 1 (A_11 = A_10 A_01 / A_00): the reference stops there
    with x updated at node 0 only; the pipeline composes exactly that x from its ring."""
    o = ref or orc
    D = orc.poisson5(3, 3).dense()
    D[1, 1] = 0.25
    r, c = np.nonzero(D)
    A = orc.make_csr(9, r, c, D[r, c])
    b = np.linspace(1.0, 2.0, 9)
    want = o.engine(A).solve(b, OSched.sequential(), tol=1e-10, max_iter=100)
    got = g.GabpEngine(A).solve(b, g.Schedule.sequential(), g.GabpOptions(tol=1e-10, max_iter=100))
    assert want.status == 1 and "pivot" in want.detail
    _same_report(got, want)


@pytest.mark.parametrize("sched", ["flood", "rb", "seq"])
def test_solve_history_after_growing_max_iter(orc, sched):
    """A second solve with a larger max_iter on the same engine (the history buffer grows; solve
    graphs captured by the first call must not keep writing into the old one) equals the oracle."""
    A = orc.poisson5(40, 30)
    b = orc.rng(21).vector(A.n)
    s = {"flood": OSched.parallel_flood(), "rb": OSched.red_black_grid(40, 30), "seq": OSched.sequential()}[sched]
    eng = g.GabpEngine(A)
    eng.solve(b, gsched(s), g.GabpOptions(tol=0.0, max_iter=40))
    rep = eng.solve(b, gsched(s), g.GabpOptions(tol=0.0, max_iter=600))
    want = orc.engine(A).solve(b, s, tol=0.0, max_iter=600)
    assert (int(rep.status), rep.iterations) == (want.status, want.iterations)
    assert np.array_equal(rep.residual_history, want.residual_history)
    assert np.array_equal(rep.solution, want.solution)


def test_solve_pinned_and_pageable_buffers_agree(orc):
    """bgabp_solve copies caller buffers directly when they are pinned and through the staged
    parallel path when pageable (large vectors): both give the oracle's x bit for bit."""
    import torch
    A = orc.poisson5(700, 600)  # 420k unknowns: 3.4 MB vectors take the staged path when pageable
    b = orc.rng(3).vector(A.n)
    opt = g.GabpOptions(tol=0.0, max_iter=60)
    eng = g.GabpEngine(A)
    rep_pageable = eng.solve(b, g.Schedule.parallel_flood(), opt)
    b_pin = torch.from_numpy(b.copy()).pin_memory()
    x_pin = torch.zeros(A.n, dtype=torch.float64).pin_memory()
    rep_pinned = eng.solve(b_pin.numpy(), g.Schedule.parallel_flood(), opt, x_out=x_pin.numpy())
    want = orc.engine(A).solve(b, OSched.parallel_flood(), tol=0.0, max_iter=60)
    assert np.array_equal(rep_pageable.solution, want.solution)
    assert np.array_equal(x_pin.numpy(), want.solution)
    assert np.array_equal(rep_pinned.residual_history, want.residual_history)


@pytest.mark.parametrize("sched", ["rb", "levels"])
def test_ordered_pivot_stop_reports_partial_x(orc, sched):
    """poisson5(12, 9) with an isolated pair whose second node's precision cancels (test_gabp.cpp:
    73-85 embedded in a grid): the ordered solve stops at that visit and reports x(k) for the
    nodes visited before it and x(k-1) for the rest, as gabp.cpp:71-87 leaves it."""
    A0 = orc.poisson5(12, 9)
    rows, cols, vals = [], [], []
    for i in range(A0.n):
        for p in range(A0.row_offsets[i], A0.row_offsets[i + 1]):
            rows.append(i), cols.append(int(A0.col_indices[p])), vals.append(float(A0.values[p]))
    p_, q_ = 4 * 12 + 5, 4 * 12 + 6
    keep = [(r, c, v) for r, c, v in zip(rows, cols, vals) if r not in (p_, q_) and c not in (p_, q_)]
    keep += [(p_, p_, 1.0), (q_, q_, 1.0), (p_, q_, 1.0), (q_, p_, 1.0)]
    r, c, v = zip(*keep)
    A = orc.make_csr(A0.n, r, c, v)
    b = orc.rng(6).vector(A.n)
    s = OSched.red_black_grid(12, 9) if sched == "rb" else OSched.four_color_grid(12, 9)
    rep = g.GabpEngine(A).solve(b, gsched(s), g.GabpOptions(tol=1e-10, max_iter=500))
    want = orc.engine(A).solve(b, s, tol=1e-10, max_iter=500)
    assert (int(rep.status), rep.iterations, rep.detail) == (want.status, want.iterations, want.detail)
    assert want.status == 1 and "pivot" in want.detail
    assert np.array_equal(rep.solution, want.solution)
    assert np.array_equal(rep.residual_history, want.residual_history)


@pytest.mark.parametrize("pivot", [False, True])
def test_sequential_tall_grid_one_sweep_per_launch(orc, pivot):
    """A 5-point grid too tall for the pipeline's ring (ny = 4200 rows of 3: 132 strips) runs one
    cooperative k_seq_grid5 launch per sweep; solve reports (and the partly updated x of a pivot
    stop, composed from the two-slot x ring) equal the oracle's."""
    nx, ny = 3, 4200
    A0 = orc.poisson5(nx, ny)
    A = A0
    if pivot:
        rows, cols, vals = [], [], []
        for i in range(A0.n):
            for p in range(A0.row_offsets[i], A0.row_offsets[i + 1]):
                rows.append(i), cols.append(int(A0.col_indices[p])), vals.append(float(A0.values[p]))
        p_, q_ = 100 * nx, 100 * nx + 1
        keep = [(r, c, v) for r, c, v in zip(rows, cols, vals) if r not in (p_, q_) and c not in (p_, q_)]
        keep += [(p_, p_, 1.0), (q_, q_, 1.0), (p_, q_, 1.0), (q_, p_, 1.0)]
        r, c, v = zip(*keep)
        A = orc.make_csr(A0.n, r, c, v)
    b = orc.rng(12).vector(A.n)
    tol = 1e-6 * np.abs(b).max()
    rep = g.GabpEngine(A).solve(b, g.Schedule.sequential(), g.GabpOptions(tol=tol, max_iter=400))
    want = orc.engine(A).solve(b, OSched.sequential(), tol=tol, max_iter=400)
    assert (int(rep.status), rep.iterations, rep.detail) == (want.status, want.iterations, want.detail)
    assert np.array_equal(rep.residual_history, want.residual_history)
    assert np.array_equal(rep.solution, want.solution)
