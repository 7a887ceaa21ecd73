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
