"""The restatements against the reference's OWN multigrid.cpp, classic.cpp and region_gabp.cpp.

Those three reference files include <Eigen/Dense>, which this image lacks; oracle/Makefile compiles
them where they lie over a minimal stand-in header (oracle/eigen_shim/Eigen/Dense) whose
factorizations are the ones in oracle/dense_standin.h — the same the restatements use.  Everything
else (hierarchy setup and truncation, the sweeps_expand probe, frozen precisions, smoothing,
transfer operators, the cycle, mg_solve and its report, the point relaxations, region message
updates, direct_message, the flop formulas) is the reference's code, so equality here is bit for
bit.  CPU only (the reference library is built in the build container and travels to the GPU box).
"""
import numpy as np
import pytest

from oracle.oracle import Csr
from oracle.oracle import Schedule as OSched

# belief::MgSmoother numbering (multigrid.hpp:17-31); 9-12 (line GS / zebra) are not restated
SM = {"gabp_seq": 0, "gabp_rb": 1, "gabp_fc": 2, "gabp_flood": 3, "gabp_line": 4, "jacobi": 5, "gs_lex": 6,
      "gs_rb": 7, "gs_fc": 8}

MG_CASES = [
    ("poisson", 5, 4, {}, "gabp_rb", 2, 2, False),
    ("poisson", 5, 4, {}, "gabp_rb", 1, 1, True),
    ("poisson", 5, 3, {}, "gabp_seq", 1, 1, False),
    ("poisson", 5, 3, {}, "gabp_fc", 2, 1, False),
    ("poisson", 5, 3, {}, "gabp_flood", 2, 2, False),
    ("poisson", 4, 3, {}, "gabp_line", 1, 1, False),
    ("poisson", 5, 3, {}, "jacobi", 2, 2, False),
    ("poisson", 5, 3, {}, "gs_lex", 1, 1, False),
    ("poisson", 5, 4, {}, "gs_rb", 2, 2, False),
    ("poisson", 5, 3, {}, "gs_fc", 2, 2, False),
    ("mixed", 5, 3, {}, "gabp_fc", 0, 4, False),
    ("mixed", 5, 3, {}, "gabp_fc", 2, 2, True),
    ("anisotropic", 5, 3, {"eps": 0.01}, "gabp_rb", 2, 2, False),
    ("anisotropic", 4, 3, {"eps": 0.01}, "gabp_line", 1, 1, False),
    ("general", 5, 3, {}, "gabp_flood", 2, 2, False),
    ("general", 5, 3, {}, "gabp_seq", 1, 1, True),
    ("boundary-layer", 6, 6, {"eps": 0.01}, "gabp_flood", 2, 2, False),
    ("boundary-layer", 6, 6, {"eps": 0.01}, "gabp_rb", 2, 2, False),
    ("boundary-layer", 5, 4, {"eps": 0.001}, "gs_rb", 2, 2, False),
]


def _need(ref):
    if ref is None or not ref.has_ref_full:
        pytest.skip("oracle/_ref (with multigrid.cpp over the Eigen stand-in) not built")


def _named_levels(ref, prob, J1, J2, params):
    levels = []
    for J in range(J1, J1 - J2, -1):
        try:
            levels.append(ref.assemble(prob, J, params))
        except ValueError:
            raise
    mats = [Csr(A.n, A.row_offsets, A.col_indices, A.values) for A, *_ in levels]
    return mats, [nx for _, _, _, nx, _ in levels], levels[0][1]


@pytest.mark.parametrize("prob,J1,J2,params,sm,pre,post,frozen", MG_CASES)
def test_mg_restatement_equals_reference_multigrid_cpp(orc, ref, prob, J1, J2, params, sm, pre, post, frozen):
    """orc_mg_* (abi_impl.inc) == belief::Hierarchy + mg_solve (multigrid.cpp:74-318) bit for bit, on
    both oracle builds: level count after the expansion probe, frozen flags, cycle flops, the solve
    report (status, cycles, detail, flop estimate, full history) and x; one extra v_cycle from a
    nonzero start."""
    _need(ref)
    try:
        hr = ref.ref_hierarchy(prob, J1, J2, params, SM[sm])
    except ValueError as e:
        pytest.skip(f"reference rejects the case: {e}")
    mats, nxs, b = _named_levels(ref, prob, J1, J2, params)
    assert hr.fine_rhs()[0].tobytes() == b.tobytes()
    tol = 1e-8 * np.abs(b).max()
    rr = hr.solve(pre, post, b, tol=tol, max_cycles=25, frozen=frozen)
    x0 = np.random.RandomState(5).uniform(-1, 1, b.size)
    for o in (orc, ref):
        ho = o.hierarchy(mats, nxs, SM[sm])
        assert ho.num_levels == hr.num_levels
        assert [ho.frozen_ok(k) for k in range(ho.num_levels)] == [hr.frozen_ok(k) for k in range(hr.num_levels)]
        assert ho.cycle_flops_per_unknown(pre, post) == hr.cycle_flops_per_unknown(pre, post)
        ro = ho.solve(pre, post, b, tol=tol, max_cycles=25, frozen=frozen)
        assert (ro.status, ro.iterations, ro.detail, ro.flop_estimate) == (rr.status, rr.iterations, rr.detail,
                                                                           rr.flop_estimate)
        assert ro.residual_history.tobytes() == rr.residual_history.tobytes()
        assert ro.solution.tobytes() == rr.solution.tobytes()
        try:
            want = hr.v_cycle(pre, post, b, x0, frozen=frozen)
        except RuntimeError as e:
            with pytest.raises(RuntimeError) as got:
                ho.v_cycle(pre, post, b, x0, frozen=frozen)
            assert got.value.args[0] == e.args[0] and got.value.args[1].tobytes() == e.args[1].tobytes()
        else:
            assert ho.v_cycle(pre, post, b, x0, frozen=frozen).tobytes() == want.tobytes()


def test_mg_reference_truncates_where_the_restatement_does(orc, ref):
    """The boundary-layer hierarchy stops coarsening at the first level whose sweeps expand
    (multigrid.cpp:88-92): same depth from the reference's ctor and the restatement."""
    _need(ref)
    hr = ref.ref_hierarchy("boundary-layer", 6, 6, {"eps": 0.01}, SM["gabp_flood"])
    mats, nxs, _ = _named_levels(ref, "boundary-layer", 6, 6, {"eps": 0.01})
    assert hr.num_levels == orc.hierarchy(mats, nxs, SM["gabp_flood"]).num_levels < 6
    assert [hr.level_n(k) for k in range(hr.num_levels)] == [m.n for m in mats[:hr.num_levels]]


@pytest.mark.parametrize("kind,sched", [(1, "seq"), (2, "rb"), (3, "fc")])
def test_gs_restatement_equals_reference_relax(orc, ref, kind, sched):
    """orc_gs_sweeps == belief::relax (classic.cpp:99-118) for the point Gauss-Seidel orders."""
    _need(ref)
    nx, ny = 9, 7
    A = orc.poisson5(nx, ny)
    rng = np.random.RandomState(3)
    b, x0 = rng.uniform(-1, 1, A.n), rng.uniform(-1, 1, A.n)
    s = {"seq": OSched.sequential(), "rb": OSched.red_black_grid(nx, ny), "fc": OSched.four_color_grid(nx, ny)}[sched]
    want = ref.ref_relax(kind, A, b, x0, 3, nx, ny)
    for o in (orc, ref):
        assert o.gs_sweeps(A, b, x0, s, 3).tobytes() == want.tobytes()


def _scaled_grid(o, nx, ny, seed):
    A = o.poisson5(nx, ny)
    s = np.random.RandomState(seed).uniform(0.5, 1.5, A.nnz)
    return o.make_csr(A.n, np.repeat(np.arange(A.n), np.diff(A.row_offsets)), A.col_indices, A.values * s)


@pytest.mark.parametrize("nx,ny,seed,mode", [(5, 4, 0, 0), (5, 4, 1, 1), (8, 8, 2, 0), (3, 9, 3, 1), (12, 6, 4, 0)])
def test_region_restatement_equals_reference_region_gabp_cpp(orc, ref, nx, ny, seed, mode):
    """region_restate.inc == belief::RegionGabpEngine (region_gabp.cpp:30-268) bit for bit: the
    block-message state and x after every sweep, the solve report, direct_message and the flops."""
    _need(ref)
    A = _scaled_grid(orc, nx, ny, seed)
    lines = orc.grid_lines(nx, ny)
    b = np.random.RandomState(seed + 10).uniform(-1, 1, A.n)
    er = ref.ref_region(A, lines)
    for o in (orc, ref):
        eo = o.region(A, lines)
        assert (eo.num_edges, eo.lam_size, eo.m_size) == (er.num_edges, er.lam_size, er.m_size)
        assert eo.flops(False) == er.flops(False) and eo.flops(True) == er.flops(True)
        (lo, mo), (lr, mr) = eo.make_state(), er.make_state()
        xo, xr = np.zeros(A.n), np.zeros(A.n)
        for s in range(6):
            oko, okr = eo.sweep(b, lo, mo, xo, mode), er.sweep(b, lr, mr, xr, mode)
            assert oko == okr
            assert lo.tobytes() == lr.tobytes() and mo.tobytes() == mr.tobytes() and xo.tobytes() == xr.tobytes(), s
        for e in (0, er.num_edges // 2, er.num_edges - 1):
            do, dr = eo.direct_message(b, lo, mo, e), er.direct_message(b, lr, mr, e)
            assert do[0].tobytes() == dr[0].tobytes() and do[1].tobytes() == dr[1].tobytes()
        ro, rr = eo.solve(b, tol=1e-10, max_iter=60, mode=mode), er.solve(b, tol=1e-10, max_iter=60, mode=mode)
        assert (ro.status, ro.iterations, ro.detail, ro.flop_estimate) == (rr.status, rr.iterations, rr.detail,
                                                                           rr.flop_estimate)
        assert ro.residual_history.tobytes() == rr.residual_history.tobytes()
        assert ro.solution.tobytes() == rr.solution.tobytes()


def test_region_reference_singular_region_message(orc, ref):
    """A singular local system: same sweep verdict and text from region_gabp.cpp:91-94 and the restatement."""
    _need(ref)
    D = np.array([[1.0, 1.0, 0.0], [1.0, 1.0, 1.0], [0.0, 1.0, 2.0]])
    r, c = np.nonzero(D)
    A = orc.make_csr(3, r, c, D[r, c])
    large = [[0, 1], [1, 2]]
    out = []
    for e in (orc.region(A, large), ref.region(A, large), ref.ref_region(A, large)):
        lam, m = e.make_state()
        out.append(e.sweep(np.ones(3), lam, m, np.zeros(3), 0))
    assert out[0] == out[1] == out[2] and out[2][0] is False and "singular local system in region 0" in out[2][1]


def test_eigen_standin_block_convergence_against_numpy(orc, ref):
    """check_block_convergence (region_gabp.cpp:276-309) through the stand-in's FullPivLU inverse,
    JacobiSVD and EigenSolver agrees with numpy (tolerance: different dense algorithms)."""
    _need(ref)
    nx, ny = 6, 5
    A = _scaled_grid(orc, nx, ny, 7)
    D = A.dense()
    blocks = [[iy * nx + ix for ix in range(nx)] for iy in range(ny)]
    for spectral in (False, True):
        k = len(blocks)
        N = np.zeros((k, k))
        for i in range(k):
            inv = np.linalg.inv(D[np.ix_(blocks[i], blocks[i])])
            for j in range(k):
                if i != j:
                    R = -inv @ D[np.ix_(blocks[i], blocks[j])]
                    N[i, j] = np.linalg.norm(R, 2) if spectral else np.abs(R).sum(axis=1).max()
        want = np.abs(np.linalg.eigvals(N)).max()
        rho, suf, sing = ref.ref_block_convergence(A, blocks, spectral)
        assert sing == -1 and suf == (want < 1.0)
        assert abs(rho - want) <= 1e-10 * want
