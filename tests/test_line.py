"""Line GaBP (region GaBP over grid lines).

CPU: the oracle's region restatement (oracle/region_restate.inc) is pinned against the reference's
own compiled region.cpp (graph construction, accept/reject and messages) and against the
reference's region tests and acceptance checks (test_region.cpp, acceptance.cpp:118-190); the
device engine's input validation (it runs before any CUDA call) is compared with the oracle's.
GPU: per-sweep block-message state, solves and the GabpLine multigrid smoother against the oracle.
The device solves each line's tridiagonal system in O(N) where the reference uses a dense
FullPivLU, so parity is a tolerance, not bits: relative 1e-9 on every sweep's block messages and
x (the randomly scaled nonsymmetric grids have local systems conditioned to ~1e5, which turns the
two algorithms' rounding into ~3e-10 relative), and 1e-10 on solves of well-conditioned systems.
"""
import numpy as np
import pytest

import paper_1904_04093_b200 as g
from oracle.oracle import Csr
from oracle.oracle import Schedule as OSched

RTOL = 1e-10       # solves, multigrid
RTOL_SWEEP = 1e-9  # per-sweep state on randomly scaled nonsymmetric grids


def _csr_from_dense(o, D):
    r, c = np.nonzero(D)
    return o.make_csr(D.shape[0], r, c, D[r, c])


def _scaled_grid(o, nx, ny, seed):
    """poisson5 with every stored value scaled by U(0.5, 1.5) (acceptance.cpp:124-126): nonsymmetric."""
    A = o.poisson5(nx, ny)
    s = np.random.RandomState(seed).uniform(0.5, 1.5, A.nnz)
    return o.make_csr(A.n, np.repeat(np.arange(A.n), np.diff(A.row_offsets)), A.col_indices, A.values * s)


def _path(o, n):
    D = np.diag(np.full(n, 2.5)) - np.eye(n, k=1) - np.eye(n, k=-1)
    return _csr_from_dense(o, D)


def _complete(o, n, d):
    D = np.ones((n, n)) + (d - 1.0) * np.eye(n)
    return _csr_from_dense(o, D)


def _poisson_levels(Js):
    """Rediscretised Poisson levels from the product's assembly (bitwise-pinned to problems.cpp)."""
    levels, nx = [], []
    for J in Js:
        p = g.assemble("poisson", J)
        levels.append(Csr(p.A.n, p.A.row_offsets, p.A.col_indices, p.A.values))
        nx.append(p.nx)
    return levels, nx, g.assemble("poisson", Js[0]).b


def _norm_graph(gr):
    small, parents, counting = gr
    return [list(map(int, s)) for s in small], [list(map(int, p)) for p in parents], list(map(int, counting))


# ---------------------------------------------------------------------------------------------
# the restatement against the reference's region.cpp and region tests (CPU)
# ---------------------------------------------------------------------------------------------
def _graph_cases(o):
    P = _path(o, 4)
    K = _complete(o, 4, 5.0)
    ex = o.example7x7()
    pairs = [[i, int(j)] for i in range(ex.n) for j in ex.col_indices[ex.row_offsets[i]:ex.row_offsets[i + 1]] if j > i]
    cases = [(o.poisson5(nx, ny), o.grid_lines(nx, ny)) for nx, ny in ((3, 3), (2, 5), (1, 4), (4, 1), (6, 6))]
    cases += [(ex, pairs), (ex, [[0, 1, 2, 3, 4], [0, 1, 2, 5, 6], [3, 4, 5, 6]]), (P, [[1, 0, 2], [1, 2, 3]])]
    bad = [(P, [[0, 1], [2, 3]]), (P, [[0, 1, 2], [1, 2, 3], [0, 3]]), (P, [[0, 1, 2], [1, 2, 7]]),
           (P, [[0, 0, 1], [1, 2, 3]]), (K, [[0, 1, 2], [0, 1, 3], [0, 2, 3]]), (P, [[0, 1, 2]])]
    return cases, bad


def test_region_graph_matches_reference_builder(orc, ref):
    if ref is None or not ref.has_region_graph:
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    cases, bad = _graph_cases(orc)
    for A, large in cases:
        want = _norm_graph(ref.region_graph_ref(A, large))
        got = _norm_graph(orc.region(A, large).small())
        assert got == want
    for A, large in bad:
        with pytest.raises(ValueError) as e_ref:
            ref.region_graph_ref(A, large)
        with pytest.raises(ValueError) as e_orc:
            orc.region(A, large)
        assert str(e_orc.value) == str(e_ref.value)


def test_grid_lines_make_single_node_children(orc):
    # test_region.cpp:40-53
    R = orc.region(orc.poisson5(3, 3), orc.grid_lines(3, 3))
    small, parents, counting = R.small()
    assert len(small) == 9 and all(len(s) == 1 for s in small)
    assert all(len(p) == 2 for p in parents) and all(c == -1 for c in counting)


def test_line_regions_solve_a_grid_system(orc):
    # test_region.cpp:264-278
    A = orc.poisson5(6, 6)
    b = orc.rng(8).vector(A.n)
    xs = np.linalg.solve(A.dense(), b)
    R = orc.region(A, orc.grid_lines(6, 6))
    for mode in (0, 1):
        rep = R.solve(b, tol=1e-11, mode=mode)
        assert rep.status == 0
        assert np.abs(rep.solution - xs).max() < 1e-9


def test_single_covering_region_solves_in_one_sweep(orc):
    # test_region.cpp:155-170
    gen = orc.rng(5)
    A = gen.diag_dominant(8, True, 0.6)
    b = gen.vector(8)
    R = orc.region(A, [list(range(8))])
    assert R.small()[0] == []
    rep = R.solve(b, tol=1e-12)
    assert rep.status == 0 and rep.iterations == 1
    assert np.abs(rep.solution - np.linalg.solve(A.dense(), b)).max() < 1e-12


def test_shared_inverse_matches_direct_route(orc):
    # acceptance.cpp:118-147: one flood sweep from a warmed state equals the per-edge direct route
    rs = np.random.RandomState(1004)
    for trial in range(30):
        nx, ny = rs.randint(2, 6), rs.randint(2, 6)
        A = _scaled_grid(orc, nx, ny, trial)
        R = orc.region(A, orc.grid_lines(nx, ny))
        b = rs.uniform(-1, 1, A.n)
        lam, m = R.make_state()
        x = np.zeros(A.n)
        for _ in range(rs.randint(0, 4)):
            assert R.sweep(b, lam, m, x, 1)[0]
        lam0, m0 = lam.copy(), m.copy()
        assert R.sweep(b, lam, m, x, 1)[0]
        for e in range(R.num_edges):
            L, mm = R.direct_message(b, lam0, m0, e)
            assert abs(L[0] - lam[e]) <= 1e-10 and abs(mm[0] - m[e]) <= 1e-10


def test_pair_regions_reduce_to_scalar_gabp(orc):
    # acceptance.cpp:149-190: pair regions are scalar flood GaBP (Lambda = lambda_tilde * A_from,to)
    for seed in range(4):
        gen = orc.rng(1005 + seed)
        A = gen.cycle_chords(8 + 3 * seed)
        pairs = [[i, int(j)] for i in range(A.n) for j in A.col_indices[A.row_offsets[i]:A.row_offsets[i + 1]] if j > i]
        R = orc.region(A, pairs)
        small, _, _ = R.small()
        el, es = R.edges()
        E = orc.engine(A)
        b = gen.vector(A.n)
        lam, m = R.make_state()
        sl, sm = E.make_state()
        xr, xs = np.zeros(A.n), np.zeros(A.n)
        D = A.dense()
        for _ in range(8):
            assert R.sweep(b, lam, m, xr, 1)[0]
            E.sweep(b, OSched.parallel_flood(), sl, sm, xs)
            for e in range(R.num_edges):
                u, v = pairs[el[e]]
                to = small[es[e]][0]
                frm = v if to == u else u
                pos = next(p for p in range(A.row_offsets[to], A.row_offsets[to + 1]) if A.col_indices[p] == frm)
                assert abs(lam[e] - sl[pos] * D[frm, to]) <= 1e-12
                assert abs(m[e] - sm[pos]) <= 1e-12


def test_multigrid_line_smoother_restatement_converges(orc):
    # test_multigrid.cpp:107-122 (GabpLine): Hierarchy("poisson", 4, 3), V(1,1), tol 1e-9
    levels, nx, b = _poisson_levels((4, 3, 2))
    H = orc.hierarchy(levels, nx, 4)
    rep = H.solve(1, 1, b, tol=1e-9)
    assert rep.status == 0 and rep.iterations <= 25
    assert np.abs(rep.solution - np.linalg.solve(levels[0].dense(), b)).max() < 1e-7


def _bad_line_inputs(o):
    """(matrix, nx, ny) the grid-line region graph rejects."""
    P = o.poisson5(4, 3)
    D = P.dense()
    wrap = D.copy()
    wrap[3, 4] = wrap[4, 3] = -1.0  # couples the end of row 0 to the start of row 1: no line holds it
    cut = D.copy()
    cut[5, 6] = cut[6, 5] = 0.0  # row 1 falls apart
    return [(_csr_from_dense(o, wrap), 4, 3), (_csr_from_dense(o, cut), 4, 3), (P, 4, 4), (P, 3, 3)]


def test_line_engine_rejects_what_the_reference_rejects(orc):
    """bglin_create validates before touching the device, so this runs on the CPU."""
    for A, nx, ny in _bad_line_inputs(orc):
        with pytest.raises(ValueError) as e_orc:
            orc.region(A, orc.grid_lines(nx, ny))
        with pytest.raises(ValueError) as e_dev:
            g.LineGabpEngine(g.SparseMatrix.of(A), nx, ny)
        assert str(e_dev.value) == str(e_orc.value)


# ---------------------------------------------------------------------------------------------
# the device engine against the restatement (GPU)
# ---------------------------------------------------------------------------------------------
def _close(got, want, what, rtol=RTOL):
    np.testing.assert_allclose(got, want, rtol=rtol, atol=rtol * max(1.0, float(np.abs(want).max(initial=0.0))),
                               err_msg=what)


def _checker(orc, ref, A, large):
    """The reference's own RegionGabpEngine (region_gabp.cpp compiled over the Eigen stand-in) when
    oracle/_ref is built, else its restatement (pinned to it bit for bit, tests/test_ref_full.py)."""
    if ref is not None and ref.has_ref_full:
        return ref.ref_region(A, large)
    return orc.region(A, large)


def _mg_checker(orc, ref, levels, nx):
    """The reference's own GabpLine Hierarchy on the Poisson levels, else the restatement."""
    if ref is not None and ref.has_ref_full:
        J1 = int(np.log2(nx[0] + 1))
        return ref.ref_hierarchy("poisson", J1, len(levels), {}, 4)
    return orc.hierarchy(levels, nx, 4)


GRIDS = [(6, 6, 0), (9, 5, 1), (1, 7, 2), (7, 1, 3), (33, 17, 4), (64, 48, 5)]


@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny,seed", GRIDS)
@pytest.mark.parametrize("mode", [0, 1])
def test_gpu_line_sweep_from_the_same_state(orc, ref, nx, ny, seed, mode):
    """Every sweep starts from the oracle's state: one sweep's messages and x, nonsymmetric grids."""
    A = _scaled_grid(orc, nx, ny, seed)
    b = np.random.RandomState(seed).uniform(-1, 1, A.n)
    R = _checker(orc, ref, A, orc.grid_lines(nx, ny))
    D = g.LineGabpEngine(g.SparseMatrix.of(A), nx, ny)
    assert D.num_edges == R.num_edges
    lr, mr = R.make_state()
    xr = np.zeros(A.n)
    for k in range(8):
        ld, md, xd = lr.copy(), mr.copy(), xr.copy()
        assert R.sweep(b, lr, mr, xr, mode)[0]
        assert D.sweep(b, ld, md, xd, mode)[0]
        _close(ld, lr, f"Lambda of sweep {k + 1}", RTOL_SWEEP)
        _close(md, mr, f"m of sweep {k + 1}", RTOL_SWEEP)
        _close(xd, xr, f"x of sweep {k + 1}", RTOL_SWEEP)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1])
def test_gpu_line_sweep_long_lines(orc, ref, mode):
    """Rows longer than one 128-node warp tile and columns cut into many segments, so the scan
    carries between tiles and between segments are exercised (nonsymmetric, from the same state)."""
    nx, ny, seed = 160, 140, 7
    A = _scaled_grid(orc, nx, ny, seed)
    b = np.random.RandomState(seed).uniform(-1, 1, A.n)
    R = _checker(orc, ref, A, orc.grid_lines(nx, ny))
    D = g.LineGabpEngine(g.SparseMatrix.of(A), nx, ny)
    lr, mr = R.make_state()
    xr = np.zeros(A.n)
    for k in range(3):
        ld, md, xd = lr.copy(), mr.copy(), xr.copy()
        assert R.sweep(b, lr, mr, xr, mode)[0]
        assert D.sweep(b, ld, md, xd, mode)[0]
        _close(ld, lr, f"Lambda of sweep {k + 1}", RTOL_SWEEP)
        _close(md, mr, f"m of sweep {k + 1}", RTOL_SWEEP)
        _close(xd, xr, f"x of sweep {k + 1}", RTOL_SWEEP)


@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny", [(6, 6), (31, 17), (64, 64)])
@pytest.mark.parametrize("mode", [0, 1])
def test_gpu_line_sweeps_free_running(orc, ref, nx, ny, mode):
    """Twelve sweeps on their own state (Poisson, well conditioned): relative 1e-10 throughout."""
    A = orc.poisson5(nx, ny)
    b = orc.rng(nx + ny).vector(A.n)
    R = _checker(orc, ref, A, orc.grid_lines(nx, ny))
    D = g.LineGabpEngine(g.SparseMatrix.of(A), nx, ny)
    lr, mr = R.make_state()
    ld, md = D.make_state()
    xr, xd = np.zeros(A.n), np.zeros(A.n)
    for k in range(12):
        assert R.sweep(b, lr, mr, xr, mode)[0]
        assert D.sweep(b, ld, md, xd, mode)[0]
        _close(ld, lr, f"Lambda after sweep {k + 1}")
        _close(md, mr, f"m after sweep {k + 1}")
        _close(xd, xr, f"x after sweep {k + 1}")


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1])
def test_gpu_line_solve_matches_restatement(orc, ref, mode):
    A = orc.poisson5(24, 20)
    b = orc.rng(8).vector(A.n)
    R = _checker(orc, ref, A, orc.grid_lines(24, 20))
    D = g.LineGabpEngine(g.SparseMatrix.of(A), 24, 20)
    want = R.solve(b, tol=1e-10, mode=mode)
    got = D.solve(b, g.RegionSolveOptions(tol=1e-10, mode=mode))
    assert (int(got.status), got.iterations, got.detail) == (want.status, want.iterations, want.detail)
    _close(got.residual_history, want.residual_history, "history")
    _close(got.solution, want.solution, "x")
    assert got.flop_estimate == want.flop_estimate


@pytest.mark.gpu
def test_gpu_line_singular_local_system(orc, ref):
    # row 0 of a 2x2 grid is [[1, 1], [1, 1]]: its local system is singular on the first sweep
    D2 = np.array([[1.0, 1.0, -0.5, 0.0], [1.0, 1.0, 0.0, -0.5], [-0.5, 0.0, 3.0, -1.0], [0.0, -0.5, -1.0, 3.0]])
    A = _csr_from_dense(orc, D2)
    b = np.ones(4)
    want = _checker(orc, ref, A, orc.grid_lines(2, 2)).solve(b)
    got = g.LineGabpEngine(g.SparseMatrix.of(A), 2, 2).solve(b)
    assert want.status == 1 and want.detail.startswith("singular local system")
    assert (int(got.status), got.iterations, got.detail) == (want.status, want.iterations, want.detail)


@pytest.mark.gpu
def test_gpu_line_smoother_multigrid_matches_restatement(orc, ref):
    levels, nx, b = _poisson_levels((5, 4, 3))
    want = _mg_checker(orc, ref, levels, nx).solve(1, 1, b, tol=1e-9)
    H = g.Hierarchy("poisson", 5, 3, smoother=g.MgSmoother.GabpLine)
    got = g.mg_solve(H, g.CycleSpec(1, 1, g.MgSmoother.GabpLine), b, g.MgSolveOptions(tol=1e-9))
    assert (int(got.status), got.iterations) == (want.status, want.iterations)
    _close(got.solution, want.solution, "x")


@pytest.mark.gpu
def test_gpu_line_rejects_like_the_reference_on_the_device_path(orc):
    D = orc.poisson5(4, 4).dense()
    D[3, 4] = D[4, 3] = -1.0
    with pytest.raises(ValueError, match=r"edge \(3,4\) is covered by no large region"):
        g.Hierarchy.from_levels([_csr_from_dense(orc, D)], [4], g.MgSmoother.GabpLine)


@pytest.mark.gpu
@pytest.mark.parametrize("pre,post", [(2, 2), (0, 3), (3, 1)])
def test_gpu_line_smoother_multi_sweep_cycles(orc, ref, pre, post):
    """Recorded factors for several sweeps per smoothing call (mean-only fast path)."""
    levels, nx, b = _poisson_levels((5, 4, 3))
    want = _mg_checker(orc, ref, levels, nx).solve(pre, post, b, tol=1e-9)
    H = g.Hierarchy("poisson", 5, 3, smoother=g.MgSmoother.GabpLine)
    got = g.mg_solve(H, g.CycleSpec(pre, post, g.MgSmoother.GabpLine), b, g.MgSolveOptions(tol=1e-9))
    assert (int(got.status), got.iterations) == (want.status, want.iterations)
    _close(got.solution, want.solution, "x")
