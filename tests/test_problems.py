"""Input assembly: the product's restated assemble() must equal the reference's own, bit for bit
(problems.cpp:161-226); the config generators must be well formed."""
import numpy as np
import pytest

import paper_1904_04093_b200 as g

NAMED = [("poisson", {}), ("anisotropic", {}), ("anisotropic", {"eps": 1e-2}), ("general", {}), ("mixed", {}),
         ("mixed", {"eps": -0.01}), ("boundary-layer", {"eps": 0.01}), ("inner-layer", {}),
         ("stretched", {}), ("stretched", {"eps": 8e-8})]


@pytest.mark.parametrize("name,params", NAMED)
def test_assemble_bitwise_equals_reference(ref, golden, name, params):
    for J in (1, 2, 4, 6):
        p = g.assemble(name, J, params)
        if ref is not None:
            A, b, exact, nx, h = ref.assemble(name, J, params)
            assert p.nx == nx
            assert np.array_equal(p.A.row_offsets, A.row_offsets)
            assert np.array_equal(p.A.col_indices, A.col_indices)
            assert p.A.values.tobytes() == A.values.tobytes()
            assert p.b.tobytes() == b.tobytes() and p.exact.tobytes() == exact.tobytes()
    meta, _ = golden
    if not params or name == "boundary-layer":
        want = meta["assemble"].get(name)
        if want and want["params"] == params:
            import hashlib
            p = g.assemble(name, 4, params)
            d = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
            assert (d(p.A.row_offsets), d(p.A.col_indices), d(p.A.values), d(p.b)) == \
                (want["ro"], want["ci"], want["v"], want["b"])


def test_assemble_rejects_unknown_names_and_params():
    with pytest.raises(ValueError, match="unknown problem"):
        g.assemble("nope", 3)
    with pytest.raises(ValueError, match="unknown parameter 'eta'"):
        g.assemble("poisson", 3, {"eta": 1.0})
    with pytest.raises(ValueError, match="J must be >= 1"):
        g.assemble("poisson", 0)


def test_poisson5_equals_make_csr(orc):
    for nx, ny in [(1, 1), (3, 2), (64, 64), (7, 13)]:
        P = g.poisson5(nx, ny)
        O = orc.poisson5(nx, ny)
        assert np.array_equal(P.row_offsets, O.row_offsets) and np.array_equal(P.col_indices, O.col_indices)
        assert P.values.tobytes() == O.values.tobytes()


def test_config_1_and_2_rhs_is_the_seeded_random_vector(orc):
    p = g.config_problem(1)
    assert p.A.n == 4096 and p.A.nnz == 20224
    assert p.b.tobytes() == orc.rng(0).vector(4096).tobytes()
    p2 = g.config_problem(2, size=48)
    assert p2.b.tobytes() == orc.rng(1).vector(48 * 48).tobytes()


def _is_m_matrix_rows(A, strict_somewhere=True):
    rows = np.repeat(np.arange(A.n), np.diff(A.row_offsets))
    diag = A.values[rows == A.col_indices]
    off = np.where(rows != A.col_indices, np.abs(A.values), 0.0)
    offsum = np.bincount(rows, weights=off, minlength=A.n)
    assert np.all(diag > 0)
    assert np.all(A.values[rows != A.col_indices] <= 0)
    assert np.all(diag >= offsum * (1 - 1e-14))
    if strict_somewhere:
        assert np.any(diag > offsum * (1 + 1e-12))


def test_config3_upwind_is_nonsymmetric_m_matrix():
    p = g.config_problem(3, size=32)
    A = p.A
    _is_m_matrix_rows(A)
    D = np.zeros((A.n, A.n))
    rows = np.repeat(np.arange(A.n), np.diff(A.row_offsets))
    D[rows, A.col_indices] = A.values
    assert np.array_equal(D != 0, D.T != 0)  # structurally symmetric
    assert not np.allclose(D, D.T)           # numerically nonsymmetric
    # cell Peclet 2: |beta| h / 2 = 2, rows scaled by h^2 -> upwind excess h*|b_x| + h*|b_y|
    assert np.isclose(D[5, 5] - 4.0, 4.0 * (np.cos(0.3) + np.sin(0.3)))
    assert np.all((p.b >= 0) & (p.b <= (1.0 / 33) ** 2))


def test_config4_aniso3d_structure():
    p = g.config_problem(4, size=8)
    A = p.A
    assert A.n == 512 and A.nnz == 7 * 512 - 6 * 64
    _is_m_matrix_rows(A)
    D = np.zeros((A.n, A.n))
    rows = np.repeat(np.arange(A.n), np.diff(A.row_offsets))
    D[rows, A.col_indices] = A.values
    assert np.array_equal(D, D.T)
    # z couplings carry the 0.01 anisotropy weight relative to x couplings (same K field scale)
    zc = -np.array([D[i, i + 64] for i in range(0, 448, 7)])
    xc = -np.array([D[i, i + 1] for i in range(0, 448, 7) if (i % 8) != 7])
    assert np.median(zc) < 0.05 * np.median(xc)
    assert np.all(np.abs(p.b) <= 1.0)


def test_config5_levels_coarsen_consistently():
    fine = g.config5_level(6, 0)
    assert fine.A.n == 63 * 63 and fine.nx == 63 and fine.b is not None
    for k in range(1, 5):
        c = g.config5_level(6, k)
        m = (1 << (6 - k)) - 1
        assert c.A.n == m * m and c.nx == m
        _is_m_matrix_rows(c.A)
    _is_m_matrix_rows(fine.A)
    # rows scaled by 1/h^2: the coarse operator of a constant K would be 1/4 of the fine one
    assert fine.A.values.max() > 100.0


@pytest.mark.parametrize("config,size", [(3, 40), (3, 1), (4, 12), (4, 3), (1, 0), (2, 48)])
def test_config_generators_equal_the_oracles(orc, config, size):
    """The product's config generators (direct CSR) equal the oracle's independent restatement of
    the SURVEY.md 8(d) recipes (triplets through make_csr), bit for bit -- so the reference arm and
    the CPU checks take their inputs from the oracle alone."""
    p = g.config_problem(config, size=size)
    A, b = orc.config_problem(config, size=size)
    assert np.array_equal(p.A.row_offsets, A.row_offsets) and np.array_equal(p.A.col_indices, A.col_indices)
    assert p.A.values.tobytes() == A.values.tobytes()
    assert p.b.tobytes() == b.tobytes()


@pytest.mark.parametrize("sigma", [2.0, 1.0])
def test_config5_levels_equal_the_oracles(orc, sigma):
    for k in range(4):
        p = g.config5_level(7, k, sigma=sigma)
        A, b = orc.config5_level(7, k, sigma=sigma)
        assert np.array_equal(p.A.row_offsets, A.row_offsets) and np.array_equal(p.A.col_indices, A.col_indices)
        assert p.A.values.tobytes() == A.values.tobytes()
        if k == 0:
            assert p.b.tobytes() == b.tobytes()
