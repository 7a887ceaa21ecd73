"""Seeded parity cases shared by the golden generator, the oracle tests and the GPU tests.

Each case builds (A, b, schedule) from the generators restated from proj/tests/oracles.hpp
(seeded std::mt19937, libstdc++ distributions) or from hand-written matrices that appear in
the reference's own tests.  `sweeps` is how many GabpEngine::sweep calls the per-sweep parity
check runs; `keep` lists sweeps whose full state is stored in tests/golden/golden.npz.
"""
from __future__ import annotations

import numpy as np

import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from oracle.oracle import Schedule  # noqa: E402


def tree_5x5(o):
    # test_gabp.cpp:18-23
    rows = [0, 0, 1, 1, 2, 2, 2, 2, 3, 3, 4, 4, 4]
    cols = [0, 2, 1, 2, 0, 1, 2, 4, 3, 4, 2, 3, 4]
    vals = [4.0, 1.0, 5.0, -1.5, 0.8, 1.2, 6.0, 2.0, 3.0, 0.7, -1.0, 0.9, 4.5]
    return o.make_csr(5, rows, cols, vals)


def one_way_4x4(o):
    # test_gabp.cpp:27-39 — one-way couplings: node 3 sends but never receives
    M = [[5, 1, 1, 0], [0, 6, 1, 1], [1, 1, 7, 1], [0, 0, 0, 2]]
    r, c, v = zip(*[(i, j, float(M[i][j])) for i in range(4) for j in range(4) if M[i][j] != 0])
    return o.make_csr(4, r, c, v)


def pivot_2x2(o):
    # test_gabp.cpp:73-85 — eliminating node 0 cancels node 1's diagonal exactly
    return o.make_csr(2, [0, 0, 1, 1], [0, 1, 0, 1], [1.0, 1.0, 1.0, 1.0])


def explicit_zeros(o):
    # structural zeros create edges (sparse.hpp:10-13); duplicates are summed (sparse.cpp:56-66)
    rows = [0, 0, 1, 1, 1, 2, 2, 3, 3, 0, 2]
    cols = [0, 1, 0, 1, 2, 2, 3, 3, 1, 1, 0]
    vals = [4.0, 0.0, -1.0, 5.0, 0.0, 6.0, 1.5, 3.0, -0.5, 0.25, 0.0]
    return o.make_csr(4, rows, cols, vals)


def _b(o, n, seed):
    return o.rng(seed).vector(n)


def _build(o, name):
    if name == "config1":
        A = o.poisson5(64, 64)
        return A, _b(o, A.n, 0), Schedule.parallel_flood()
    if name == "poisson64_flood":
        A = o.poisson5(64, 64)
        return A, _b(o, A.n, 0), Schedule.parallel_flood()
    if name == "tree5_seq":
        A = tree_5x5(o)
        return A, np.ones(5), Schedule.sequential()
    if name == "tree5_flood":
        A = tree_5x5(o)
        return A, np.ones(5), Schedule.parallel_flood()
    if name in ("oneway4_flood", "oneway4_seq"):
        A = one_way_4x4(o)
        return A, _b(o, 4, 3), Schedule.parallel_flood() if name.endswith("flood") else Schedule.sequential()
    if name == "dd15_sym_flood":  # test_gabp.cpp:233-247 (symmetric reduction)
        g = o.rng(31)
        A = g.diag_dominant(15, True)
        return A, g.vector(A.n), Schedule.parallel_flood()
    if name in ("dd25_nonsym_flood", "dd25_nonsym_seq"):  # test_gabp.cpp:159-172
        g = o.rng(77)
        A = g.diag_dominant(25, False)
        b = g.vector(A.n)
        return A, b, Schedule.parallel_flood() if name.endswith("flood") else Schedule.sequential()
    if name == "dd20_sym_flood":
        g = o.rng(202)
        A = g.diag_dominant(20, True)
        return A, g.vector(A.n), Schedule.parallel_flood()
    if name == "dd30_nonsym_rbgreedy":
        g = o.rng(11)
        A = g.diag_dominant(30, False)
        return A, g.vector(A.n), Schedule(5)
    if name == "dd20_custom":
        g = o.rng(19)
        A = g.diag_dominant(20, False, 0.3)
        b = g.vector(A.n)
        perm = np.random.RandomState(19).permutation(A.n)
        return A, b, Schedule.custom(perm)
    if name in ("ex7x7_flood", "ex7x7_seq"):  # test_gabp.cpp:249-259
        A = o.example7x7()
        return A, np.ones(7), Schedule.parallel_flood() if name.endswith("flood") else Schedule.sequential()
    if name in ("poisson9_rb", "poisson9_fc", "poisson9_flood", "poisson9_seq"):
        A = o.poisson5(9, 9)
        sched = {"rb": Schedule.red_black_grid(9, 9), "fc": Schedule.four_color_grid(9, 9),
                 "flood": Schedule.parallel_flood(), "seq": Schedule.sequential()}[name.split("_")[1]]
        return A, np.ones(A.n), sched
    if name == "poisson12x7_rb":
        A = o.poisson5(12, 7)
        return A, _b(o, A.n, 12), Schedule.red_black_grid(12, 7)
    if name in ("pivot2_seq", "pivot2_flood"):
        A = pivot_2x2(o)
        return A, np.ones(2), Schedule.parallel_flood() if name.endswith("flood") else Schedule.sequential()
    if name in ("zeros4_flood", "zeros4_seq"):
        A = explicit_zeros(o)
        return A, _b(o, 4, 4), Schedule.parallel_flood() if name.endswith("flood") else Schedule.sequential()
    if name == "cycle12_flood":  # acceptance.cpp:29-49
        g = o.rng(1010)
        A = g.cycle_chords(12)
        return A, g.vector(A.n), Schedule.parallel_flood()
    raise KeyError(name)


CASES = {
    "config1": {"sweeps": 200, "keep": (1, 2, 10, 200)},
    "tree5_seq": {"sweeps": 10, "keep": (10,)},
    "tree5_flood": {"sweeps": 10, "keep": (10,)},
    "oneway4_flood": {"sweeps": 20, "keep": (20,)},
    "oneway4_seq": {"sweeps": 20, "keep": (20,)},
    "dd15_sym_flood": {"sweeps": 12, "keep": (12,)},
    "dd25_nonsym_flood": {"sweeps": 60, "keep": (60,)},
    "dd25_nonsym_seq": {"sweeps": 40, "keep": (40,)},
    "dd20_sym_flood": {"sweeps": 40, "keep": (40,)},
    "dd30_nonsym_rbgreedy": {"sweeps": 30, "keep": (30,)},
    "dd20_custom": {"sweeps": 30, "keep": (30,)},
    "ex7x7_flood": {"sweeps": 50, "keep": (50,)},
    "ex7x7_seq": {"sweeps": 50, "keep": (50,)},
    "poisson9_rb": {"sweeps": 30, "keep": (30,)},
    "poisson9_fc": {"sweeps": 30, "keep": (30,)},
    "poisson9_flood": {"sweeps": 30, "keep": (30,)},
    "poisson9_seq": {"sweeps": 30, "keep": (30,)},
    "poisson12x7_rb": {"sweeps": 20, "keep": (20,)},
    "pivot2_seq": {"sweeps": 3, "keep": ()},
    "pivot2_flood": {"sweeps": 3, "keep": ()},
    "zeros4_flood": {"sweeps": 15, "keep": (15,)},
    "zeros4_seq": {"sweeps": 15, "keep": (15,)},
    "cycle12_flood": {"sweeps": 25, "keep": (25,)},
}


def build_case(o, name):
    """(A, b, schedule) for `name`, built with the restatement's generators (oracle `o`)."""
    return _build(o, name)


def grid5_const(orc, nx, d):
    """nx x nx 5-point matrix, diagonal d, off-diagonals -1 (canonical CSR)."""
    rows, cols, vals = [], [], []
    for iy in range(nx):
        for ix in range(nx):
            i = iy * nx + ix
            for dx, dy in ((0, -1), (-1, 0), (0, 0), (1, 0), (0, 1)):
                jx, jy = ix + dx, iy + dy
                if 0 <= jx < nx and 0 <= jy < nx:
                    rows.append(i)
                    cols.append(jy * nx + jx)
                    vals.append(d if (dx, dy) == (0, 0) else -1.0)
    return orc.make_csr(nx * nx, rows, cols, vals)


def mg_breakdown_levels(orc, fine_diag):
    """Three levels (7^2, 3^2, 1) whose fine level breaks the GaBP smoother: with diagonal 1 a
    flood sweep hits a zero edge pivot in its second sweep, with diagonal 2 a red-black or flood
    sweep hits a zero node pivot in its first.  The coarse levels are diagonally dominant (the
    setup probe keeps them)."""
    return [grid5_const(orc, 7, fine_diag), grid5_const(orc, 3, 8.0), grid5_const(orc, 1, 8.0)], [7, 3, 1]
