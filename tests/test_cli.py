"""Matrix Market input (sparse.cpp:123-180 semantics, test_sparse.cpp:48-93 cases) and the
gabp_solve command-line front-end (belief_solve.cpp contract: CSV, summary line, exit codes)."""
import os
import subprocess

import numpy as np
import pytest

import paper_1904_04093_b200 as g

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
CLI = os.path.join(ROOT, "paper_1904_04093_b200", "bin", "gabp_solve")


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return p


def test_matrix_market_cases(tmp_path, orc):
    A = g.load_matrix_market(_write(tmp_path, "one.mtx", "%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 4.0\n"))
    assert A.n == 1 and A.nnz == 1 and A.values[0] == 4.0
    A = g.load_matrix_market(_write(tmp_path, "dup.mtx", "%%MatrixMarket matrix coordinate real general\n"
                                                         "2 2 4\n1 1 1\n2 2 1\n1 2 1.0\n1 2 2.0\n"))
    assert A.nnz == 3 and A.values[1] == 3.0
    S = g.load_matrix_market(_write(tmp_path, "sym.mtx", "%%MatrixMarket matrix coordinate real symmetric\n"
                                                         "% comment\n3 3 3\n1 1 2\n2 1 -1\n3 3 5\n"))
    assert S.row_offsets.tolist() == [0, 2, 3, 4] and S.col_indices.tolist() == [0, 1, 0, 2]
    with pytest.raises(RuntimeError, match="not square"):
        g.load_matrix_market(_write(tmp_path, "rect.mtx", "%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1\n"))
    with pytest.raises(RuntimeError, match="out of bounds"):
        g.load_matrix_market(_write(tmp_path, "oob.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n"))
    with pytest.raises(RuntimeError, match="cannot open"):
        g.load_matrix_market(tmp_path / "missing.mtx")
    # round trip of a random nonsymmetric matrix in %.17g equals the reference's make_csr
    R = orc.rng(42).diag_dominant(17, False)
    rows = np.repeat(np.arange(R.n), np.diff(R.row_offsets))
    text = "%%MatrixMarket matrix coordinate real general\n%d %d %d\n" % (R.n, R.n, R.nnz) + "".join(
        "%d %d %.17g\n" % (i + 1, j + 1, v) for i, j, v in zip(rows, R.col_indices, R.values))
    B = g.load_matrix_market(_write(tmp_path, "rt.mtx", text))
    assert np.array_equal(B.row_offsets, R.row_offsets) and np.array_equal(B.col_indices, R.col_indices)
    assert B.values.tobytes() == R.values.tobytes()


def _cli(*args, **kw):
    if not os.path.exists(CLI):
        pytest.skip("gabp_solve not built")
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600, **kw)


def test_cli_argument_errors_exit_1():
    assert _cli("--param", "eps").returncode == 1
    assert _cli("--bogus").returncode == 1
    assert _cli("--solver", "bicgstab").returncode == 1
    assert _cli("--problem", "nope").returncode == 1
    r = _cli("--solver", "mg:red-black-gabp")
    assert r.returncode == 1 and "needs --cycle" in r.stderr


@pytest.mark.gpu
def test_cli_gabp_run_matches_oracle(tmp_path, orc):
    r = _cli("--problem", "poisson", "--J", 5, "--schedule", "parallel-flood", "--tol", 1e-6, "--max-iter", 3000)
    p = g.assemble("poisson", 5)
    from oracle.oracle import Csr, Schedule as OSched
    want = orc.engine(Csr(p.A.n, p.A.row_offsets, p.A.col_indices, p.A.values)).solve(
        p.b, OSched.parallel_flood(), tol=1e-6, max_iter=3000)
    lines = r.stdout.strip().splitlines()
    assert lines[0] == "iteration,residual_inf"
    assert [float(l.split(",")[1]) for l in lines[1:]] == list(want.residual_history)
    assert r.returncode == {0: 0, 1: 2, 2: 3}[want.status]
    assert f"iterations={want.iterations}" in r.stderr


@pytest.mark.gpu
def test_cli_multigrid_and_matrix_market(tmp_path):
    r = _cli("--problem", "poisson", "--solver", "mg:red-black-gabp", "--cycle", "V:6,4", "--pre", 2, "--post", 2,
             "--tol", 1e-9, "--out", tmp_path / "h.csv")
    assert r.returncode == 0 and "status=converged" in r.stderr
    assert (tmp_path / "h.csv").read_text().startswith("iteration,residual_inf\n")
    A = g.poisson5(20, 20)
    rows = np.repeat(np.arange(A.n), np.diff(A.row_offsets))
    mtx = tmp_path / "p.mtx"
    mtx.write_text("%%MatrixMarket matrix coordinate real general\n%d %d %d\n" % (A.n, A.n, A.nnz) + "".join(
        "%d %d %.17g\n" % (i + 1, j + 1, v) for i, j, v in zip(rows, A.col_indices, A.values)))
    r = _cli("--matrix", mtx, "--rhs", "random", "--seed", 3, "--schedule", "parallel-flood", "--tol", 1e-8,
             "--max-iter", 5)
    assert r.returncode == 3 and "status=max_iter iterations=5" in r.stderr


def test_cli_smoother_names_follow_the_reference():
    # belief_solve.cpp:58-75: flood-gabp / line-gabp are accepted names; unknown ones are errors
    r = _cli("--problem", "poisson", "--solver", "mg:parallel-gabp", "--cycle", "V:4,3")
    assert r.returncode == 1 and "unknown multigrid smoother" in r.stderr


@pytest.mark.gpu
def test_cli_generalized_gabp_and_line_smoother(orc):
    r = _cli("--problem", "poisson", "--J", 5, "--solver", "generalized-gabp", "--tol", 1e-6, "--max-iter", 800)
    p = g.assemble("poisson", 5)
    from oracle.oracle import Csr
    want = orc.region(Csr(p.A.n, p.A.row_offsets, p.A.col_indices, p.A.values),
                      orc.grid_lines(p.nx, p.nx)).solve(p.b, tol=1e-6, max_iter=800)
    assert r.returncode == {0: 0, 1: 2, 2: 3}[want.status] and f"iterations={want.iterations}" in r.stderr
    got = [float(l.split(",")[1]) for l in r.stdout.strip().splitlines()[1:]]
    # line solves agree to rounding (O(N) vs dense local solves): relative to r0 for small residuals
    np.testing.assert_allclose(got, want.residual_history, rtol=1e-9, atol=1e-10 * want.residual_history[0])
    r = _cli("--problem", "poisson", "--solver", "mg:line-gabp", "--cycle", "V:6,4", "--tol", 1e-9)
    assert r.returncode == 0 and "status=converged" in r.stderr
    r = _cli("--problem", "poisson", "--solver", "mg:flood-gabp", "--cycle", "V:5,3", "--max-iter", 3)
    assert r.returncode in (0, 2, 3) and "iterations=" in r.stderr
