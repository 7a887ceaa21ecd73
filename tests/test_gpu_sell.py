"""General-sparsity fused solve step (SELL layout, sell_kernels.cuh) against the oracle, bit for
bit: GabpEngine::solve (gabp.cpp:174-219 over the flood sweep of gabp.cpp:102-163) on matrices
that are not <= 8-offset stencils -- random diagonally dominant graphs (symmetric and not), a hub
node wider than any register-cached chunk, structurally one-way edges, explicit zeros -- and on
stencils forced off the DIA layout; plus the SELL step against the three-launch union-CSR loop."""
import numpy as np
import pytest

import paper_1904_04093_b200 as g
from oracle.oracle import Csr, Schedule as OSched
from tests.cases import build_case, grid5_const

pytestmark = pytest.mark.gpu


def _hub(orc, n, seed):
    """A random sparse matrix plus a hub row/column coupling node 0 to every 3rd node."""
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for i in range(n):
        for j in rng.choice(n, size=3, replace=False):
            if j != i:
                rows += [i]
                cols += [int(j)]
                vals += [float(rng.uniform(-1, 0))]
    for j in range(3, n, 3):
        rows += [0, j]
        cols += [j, 0]
        vals += [-0.01, -0.02]
    for i in range(n):
        rows.append(i)
        cols.append(i)
        vals.append(12.0 + (i == 0) * n * 0.02)
    return orc.make_csr(n, rows, cols, vals)


def _cases(orc):
    gen = orc.rng(41)
    yield "dd 1000 symmetric (p 0.01)", gen.diag_dominant(1000, True, 0.01), gen.vector(1000)
    yield "dd 777 nonsymmetric (p 0.004)", gen.diag_dominant(777, False, 0.004), gen.vector(777)
    yield "dd 300 nonsymmetric (p 0.05)", gen.diag_dominant(300, False, 0.05), gen.vector(300)
    A = _hub(orc, 2000, 5)
    yield "hub 2000", A, gen.vector(2000)
    yield "cycle + chords 513", gen.cycle_chords(513), gen.vector(513)
    A, b, _ = build_case(orc, "oneway4_flood")
    yield "one-way 4x4", A, b
    A, b, _ = build_case(orc, "zeros4_flood")
    yield "explicit zeros", A, b
    A, b, _ = build_case(orc, "pivot2_flood")
    yield "pivot 2x2", A, b
    A, b, _ = build_case(orc, "ex7x7_flood")
    yield "7x7 non-convergent", A, b


@pytest.mark.parametrize("stop", [0, 1])
def test_sell_solve_matches_oracle(orc, ref, stop):
    O = ref if ref is not None else orc
    for name, A, b in _cases(orc):
        eng = g.GabpEngine(A, g.Layout.Csr)
        want_eng = O.engine(A)
        for tol, cap in ((1e-9 * np.abs(b).max(), 3000), (0.0, 37), (1e-9, 1), (1e-9, 2), (0.5, 9)):
            want = want_eng.solve(b, OSched.parallel_flood(), tol=tol, max_iter=cap, stop=stop)
            got = eng.solve(b, g.Schedule.parallel_flood(), g.GabpOptions(tol=tol, max_iter=cap, stop=stop))
            key = (name, tol, cap)
            assert (int(got.status), got.iterations, got.detail) == (want.status, want.iterations, want.detail), key
            assert got.residual_history.tobytes() == want.residual_history.tobytes(), key
            assert got.solution.tobytes() == want.solution.tobytes(), key
            assert got.flop_estimate == want.flop_estimate, key


def test_sell_step_equals_ucsr_loop(orc, monkeypatch):
    """BGABP_UCSR_SOLVE=1 keeps the earlier three-launch union-CSR solve loop (A/B)."""
    gen = orc.rng(77)
    A, b = gen.diag_dominant(2500, False, 0.003), gen.vector(2500)
    out = []
    for flag in ("1", None):
        if flag:
            monkeypatch.setenv("BGABP_UCSR_SOLVE", flag)
        else:
            monkeypatch.delenv("BGABP_UCSR_SOLVE", raising=False)
        eng = g.GabpEngine(A, g.Layout.Csr)
        r = eng.solve(b, g.Schedule.parallel_flood(), g.GabpOptions(tol=1e-10, max_iter=500))
        out.append((int(r.status), r.iterations, r.residual_history.tobytes(), r.solution.tobytes()))
    assert out[0] == out[1]


@pytest.mark.parametrize("prob", ["mixed", "general", "anisotropic"])
def test_stencil_forced_to_sell_equals_dia(orc, prob):
    """9-point / 5-point stencils: the SELL step and the DIA step give the same bits."""
    p = g.assemble(prob, 6)
    A = Csr(p.A.n, p.A.row_offsets, p.A.col_indices, p.A.values)
    tol = 1e-8 * np.abs(p.b).max()
    r1 = g.GabpEngine(A, g.Layout.Csr).solve(p.b, g.Schedule.parallel_flood(), g.GabpOptions(tol=tol, max_iter=800))
    r2 = g.GabpEngine(A, g.Layout.Dia).solve(p.b, g.Schedule.parallel_flood(), g.GabpOptions(tol=tol, max_iter=800))
    assert (r1.status, r1.iterations) == (r2.status, r2.iterations)
    assert r1.residual_history.tobytes() == r2.residual_history.tobytes()
    assert r1.solution.tobytes() == r2.solution.tobytes()


def test_sell_device_stepping_and_graphs(orc):
    """The device-resident stepping API (graph-replayed chunks) on the SELL step."""
    import torch
    A = grid5_const(orc, 45, 4.5)
    b = orc.rng(4).vector(A.n)
    eng = g.GabpEngine(A, g.Layout.Csr)
    bd = torch.tensor(b, device="cuda")
    eng.solve_device_begin(bd.data_ptr(), g.Schedule.parallel_flood(), g.GabpOptions(tol=0.0, max_iter=300))
    eng.solve_device_steps(37)
    eng.solve_device_steps(16)
    eng.solve_device_steps(300)
    st, its, _, _ = eng.solve_device_end()
    want = orc.engine(A).solve(b, OSched.parallel_flood(), tol=0.0, max_iter=300)
    assert (int(st), its) == (want.status, want.iterations)
