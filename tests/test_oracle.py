"""Pin the CPU restatement (oracle/liboracle.so) before trusting it as the checker.

1. against the golden vectors made from the reference's own compiled sources
   (tests/golden/make_golden.py), bit for bit;
2. against oracle/_ref/libbelief_ref.so directly when it is present, bit for bit.
"""
import hashlib

import numpy as np
import pytest

from oracle.oracle import Schedule
from tests.cases import CASES, build_case


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", sorted(CASES))
def test_restatement_matches_golden_per_sweep(orc, golden, name):
    meta, arrays = golden
    rec = meta["cases"][name]
    A, b, sched = build_case(orc, name)
    assert digest(A.values) + digest(b) == rec["input"], "seeded generator drifted"
    e = orc.engine(A)
    assert e.num_edges == rec["num_edges"]
    lam, m = e.make_state()
    x = np.zeros(A.n)
    for s, want in enumerate(rec["digests"]):
        ok, err = e.sweep(b, sched, lam, m, x)
        assert [ok, err] == rec["ok"][s]
        if not ok:
            break
        beta = e.node_precisions(lam, m)
        r = orc.residual_inf_norm(A, x, b)
        assert [digest(lam), digest(m), digest(x), digest(beta), float(r).hex()] == want, f"sweep {s + 1}"


def test_restatement_solves_match_golden(orc, golden):
    meta, _ = golden
    for name, rec in meta["solves"].items():
        A, b, sched = build_case(orc, name)
        rep = orc.engine(A).solve(b, sched, tol=rec["tol"], max_iter=rec["max_iter"], stop=rec["stop"])
        assert (rep.status, rep.iterations, rep.detail) == (rec["status"], rec["iterations"], rec["detail"]), name
        assert [float(v).hex() for v in rep.residual_history] == rec["history"], name
        assert digest(rep.solution) == rec["x"], name
        assert rep.flop_estimate == rec["flops"], name


def test_restatement_frozen_path_matches_golden(orc, golden):
    meta, _ = golden
    for name, rec in meta["frozen"].items():
        A, b, sched = build_case(orc, name)
        e = orc.engine(A)
        lam, sig, conv, its = e.precompute_lambda(sched, 1e-10, 500)
        assert (conv, its) == (rec["converged"], rec["iterations"])
        assert digest(lam) == rec["lam"] and digest(sig) == rec["sigma"]
        assert digest(e.correction_sweeps(b, sched, lam, sig, 3)) == rec["corr3"]
        rep = e.solve_error_correction(b, sched, 2, lam, sig, tol=1e-10, max_iter=3000)
        assert (rep.status, rep.iterations) == (rec["ec_status"], rec["ec_iterations"])
        assert [float(v).hex() for v in rep.residual_history] == rec["ec_history"]


def test_restatement_computation_tree_matches_golden(orc, golden):
    meta, _ = golden
    rng = orc.rng(29)
    for trial, want in enumerate(meta["computation_tree"]):
        A = rng.diag_dominant(6 + trial % 3, trial % 2 == 0, 0.5)
        b = rng.vector(A.n)
        got = [[float(orc.computation_tree_solve(A, b, root, d)).hex() for root in range(A.n)] for d in range(1, 6)]
        assert got == want


def test_restatement_transfers_match_golden(orc, golden):
    _, arrays = golden
    g = orc.rng(33)
    u, v = g.vector(49), g.vector(9)
    assert np.array_equal(orc.mg_restrict(u, 7), arrays["mg/restrict7"])
    assert np.array_equal(orc.mg_prolong(v, 3), arrays["mg/prolong3"])


def test_computation_tree_equals_flood_iterate(orc):
    """acceptance.cpp:296-316 (criterion 10) on the restatement."""
    rng = orc.rng(1010)
    for trial in range(10):
        n = rng.uniform_int(4, 8)
        A = rng.diag_dominant(n, trial % 2 == 0, 0.5)
        b = rng.vector(A.n)
        e = orc.engine(A)
        lam, m = e.make_state()
        x = np.zeros(A.n)
        for depth in range(1, 6):
            ok, _ = e.sweep(b, Schedule.parallel_flood(), lam, m, x)
            assert ok
            for root in range(A.n):
                t = orc.computation_tree_solve(A, b, root, depth, 2000000)
                assert abs(t - x[root]) <= 1e-12 * max(1.0, abs(x[root]))


def test_structure_known_answers(orc):
    """test_sparse.cpp:33-46 and test_gabp.cpp:43-61."""
    A = orc.make_csr(2, [1, 0, 0, 0], [0, 1, 1, 0], [3.0, 1.0, 2.0, 5.0])
    assert A.nnz == 3 and A.values.tolist() == [5.0, 3.0, 3.0]
    assert A.transpose_pos.tolist() == [0, 2, 1]
    from tests.cases import one_way_4x4
    W = one_way_4x4(orc)
    assert orc.engine(W).num_edges == 7
    with pytest.raises(ValueError, match="structurally zero diagonal"):
        orc.engine(orc.make_csr(2, [0, 0, 1], [0, 1, 0], [1.0, 1.0, 1.0]))


def test_restatement_bitwise_equals_reference_library(orc, ref):
    if ref is None:
        pytest.skip("oracle/_ref not built (no /root/reference at build time)")
    for name in sorted(CASES):
        A, b, sched = build_case(orc, name)
        eo, er = orc.engine(A), ref.engine(A)
        so, sr = eo.make_state(), er.make_state()
        xo, xr = np.zeros(A.n), np.zeros(A.n)
        for _ in range(min(CASES[name]["sweeps"], 25)):
            oko = eo.sweep(b, sched, *so, xo)
            okr = er.sweep(b, sched, *sr, xr)
            assert oko == okr
            assert all(np.array_equal(p, q) for p, q in zip(so + (xo,), sr + (xr,))), name
            if not oko[0]:
                break


def test_flop_table_restatement_equals_reference(orc, ref):
    """flop_table (analysis.cpp:135-154): values and the invalid_argument texts."""
    if ref is None:
        pytest.skip("oracle/_ref not built")
    for stencil in (0, 1):
        for sm in (0, 1, 2, 3):
            for sweeps in (0, 1, 2, 3, 6):
                got = want = None
                try:
                    want = ref.flop_table(stencil, sm, sweeps)
                except ValueError as e:
                    want = str(e)
                try:
                    got = orc.flop_table(stencil, sm, sweeps)
                except ValueError as e:
                    got = str(e)
                assert got == want, (stencil, sm, sweeps)


MG_ORACLE_CASES = [("poisson", 5, 3, 1, 2, 2, {}), ("poisson", 5, 3, 0, 1, 1, {}), ("poisson", 5, 3, 7, 2, 2, {}),
                   ("mixed", 5, 3, 2, 0, 4, {}), ("boundary-layer", 6, 6, 3, 2, 2, {"eps": 0.01}),
                   ("general", 5, 3, 3, 2, 2, {})]


@pytest.mark.parametrize("prob,J1,J2,sm,pre,post,params", MG_ORACLE_CASES)
def test_mg_restatement_bitwise_equals_reference_library(orc, ref, prob, J1, J2, sm, pre, post, params):
    """The multigrid restatement (abi_impl.inc) over the restated engine equals it over the
    reference's compiled engine bit for bit: history, x (also after a smoother breakdown, the
    boundary-layer flood case), flop estimate (flop_table of analysis.cpp) and cycle flops."""
    if ref is None:
        pytest.skip("oracle/_ref not built")
    from oracle.oracle import Csr
    levels = [ref.assemble(prob, J, params) for J in range(J1, J1 - J2, -1)]
    mats = [Csr(A.n, A.row_offsets, A.col_indices, A.values) for A, *_ in levels]
    nxs = [nx for _, _, _, nx, _ in levels]
    b = levels[0][1]
    ho, hr = orc.hierarchy(mats, nxs, sm), ref.hierarchy(mats, nxs, sm)
    assert ho.num_levels == hr.num_levels
    assert ho.cycle_flops_per_unknown(pre, post) == hr.cycle_flops_per_unknown(pre, post)
    ro = ho.solve(pre, post, b, tol=1e-8 * np.abs(b).max(), max_cycles=30)
    rr = hr.solve(pre, post, b, tol=1e-8 * np.abs(b).max(), max_cycles=30)
    assert (ro.status, ro.iterations, ro.detail, ro.flop_estimate) == (rr.status, rr.iterations, rr.detail,
                                                                       rr.flop_estimate)
    assert ro.residual_history.tobytes() == rr.residual_history.tobytes()
    assert ro.solution.tobytes() == rr.solution.tobytes()
    if rr.detail.startswith("smoother breakdown"):
        assert rr.residual_history.size == rr.iterations  # the failed cycle has no residual
    else:
        assert rr.residual_history.size == rr.iterations + 1
        assert rr.flop_estimate == rr.iterations * hr.cycle_flops_per_unknown(pre, post) * b.size


@pytest.mark.parametrize("fine_diag,sm,pre,post", [(1.0, 3, 1, 2), (1.0, 3, 2, 2), (2.0, 1, 1, 1), (1.0, 3, 1, 0)])
def test_mg_breakdown_x_restatement_equals_reference_library(orc, ref, fine_diag, sm, pre, post):
    """A smoother breakdown stops the cycle where the reference's exception does: x keeps the
    level-0 updates made before it (multigrid.cpp:290-297; V(1,2) flood breaks in the post-smoothing
    call, after the pre-smoothing and the coarse correction were added)."""
    if ref is None:
        pytest.skip("oracle/_ref not built")
    from tests.cases import mg_breakdown_levels
    mats, nxs = mg_breakdown_levels(orc, fine_diag)
    b = orc.rng(9).vector(49)
    out = []
    for o in (orc, ref):
        h = o.hierarchy(mats, nxs, sm)
        assert h.num_levels == 3
        out.append(h.solve(pre, post, b, tol=1e-10, max_cycles=10))
        try:
            h.v_cycle(pre, post, b, np.zeros(49))
            out.append(None)
        except RuntimeError as e:
            out.append(e.args)
    (ro, eo), (rr, er) = out[:2], out[2:]
    if post == 0:
        assert rr.status != 1 or rr.detail == "residual blowup"
        return
    assert rr.status == 1 and rr.detail.startswith("smoother breakdown on level 0"), rr.detail
    assert (ro.status, ro.iterations, ro.detail, ro.flop_estimate) == (rr.status, rr.iterations, rr.detail,
                                                                       rr.flop_estimate)
    assert ro.residual_history.tobytes() == rr.residual_history.tobytes()
    assert ro.solution.tobytes() == rr.solution.tobytes()
    assert eo[0] == er[0] and eo[1].tobytes() == er[1].tobytes() == rr.solution.tobytes()
    assert (np.abs(rr.solution).max() == 0.0) == (pre >= 2 or fine_diag == 2.0)


def test_restated_damping_zero_is_the_reference(orc, ref):
    """Damping (restatement only) at 0 is the reference's update; the reference build has none."""
    if ref is None:
        pytest.skip("oracle/_ref not built")
    A = orc.poisson5(12, 12)
    b = orc.rng(1).vector(A.n)
    e = orc.engine(A)
    e.set_damping(0.0)
    got = e.solve(b, Schedule.parallel_flood(), tol=1e-8, max_iter=500)
    want = ref.engine(A).solve(b, Schedule.parallel_flood(), tol=1e-8, max_iter=500)
    assert got.residual_history.tobytes() == want.residual_history.tobytes()
    e.set_damping(0.5)
    damped = e.solve(b, Schedule.parallel_flood(), tol=1e-8, max_iter=500)
    assert damped.residual_history.tobytes() != want.residual_history.tobytes()
    with pytest.raises(ValueError):
        ref.engine(A).set_damping(0.5)
