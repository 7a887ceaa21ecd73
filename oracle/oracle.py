"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU oracles (see oracle_abi.h).

    Oracle.restatement()  -> oracle/liboracle.so          (own restatement, always available)
    Oracle.reference()    -> oracle/_ref/libbelief_ref.so  (reference sources compiled here;
                                                           None when it was never built)
                             .ref_hierarchy / .ref_region / .ref_relax run the reference's own
                             multigrid.cpp / region_gabp.cpp / classic.cpp (over oracle/eigen_shim)

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module.  The CUDA
product (paper_1904_04093_b200/) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbelief_ref.so")

# schedule kinds shared with include/gabp_b200.h
FLOOD, SEQUENTIAL, RED_BLACK, FOUR_COLOR, CUSTOM, RED_BLACK_GREEDY, FOUR_COLOR_GREEDY = range(7)
# SolveStatus numbering (report.hpp:10)
CONVERGED, DIVERGED, MAX_ITER = 0, 1, 2
# MgSmoother numbering (multigrid.hpp:17-31)
MG_GABP_SEQ, MG_GABP_RB, MG_GABP_FC, MG_GABP_FLOOD = 0, 1, 2, 3
MG_JACOBI, MG_GS_LEX, MG_GS_RB, MG_GS_FC = 5, 6, 7, 8

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class _Sched(C.Structure):
    _fields_ = [("kind", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("order", _ip)]


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


@dataclass
class Schedule:
    kind: int = SEQUENTIAL
    nx: int = 0
    ny: int = 0
    order: np.ndarray | None = None

    def c(self):
        s = _Sched(self.kind, self.nx, self.ny, None)
        if self.order is not None:
            self._keep = i32(self.order)
            s.order = _i(self._keep)
        return s

    @staticmethod
    def parallel_flood():
        return Schedule(FLOOD)

    @staticmethod
    def sequential():
        return Schedule(SEQUENTIAL)

    @staticmethod
    def red_black_grid(nx, ny):
        return Schedule(RED_BLACK, nx, ny)

    @staticmethod
    def four_color_grid(nx, ny):
        return Schedule(FOUR_COLOR, nx, ny)

    @staticmethod
    def custom(order):
        return Schedule(CUSTOM, order=i32(order))


@dataclass
class Report:
    status: int
    iterations: int
    residual_history: np.ndarray
    flop_estimate: float
    solution: np.ndarray
    detail: str = ""


@dataclass
class Csr:
    """Canonical CSR arrays (sparse.hpp:17-39)."""
    n: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray
    transpose_pos: np.ndarray = field(default=None)

    @property
    def nnz(self):
        return int(self.row_offsets[-1])

    def dense(self):
        D = np.zeros((self.n, self.n))
        for i in range(self.n):
            s, e = self.row_offsets[i], self.row_offsets[i + 1]
            D[i, self.col_indices[s:e]] = self.values[s:e]
        return D

    def num_edges(self):
        rows = np.repeat(np.arange(self.n), np.diff(self.row_offsets))
        return int(np.sum(rows != self.col_indices))


class Oracle:
    """One loaded oracle library."""

    _cache: dict = {}

    def __init__(self, path):
        self.path = path
        L = self.lib = C.CDLL(path)
        vp = C.c_void_p
        sig = {
            "orc_make_csr": (vp, [C.c_int, C.c_long, _ip, _ip, _dp, C.c_char_p, C.c_size_t]),
            "orc_matrix_from_csr": (vp, [C.c_int, _ip, _ip, _dp]),
            "orc_matrix_free": (None, [vp]),
            "orc_matrix_n": (C.c_int, [vp]),
            "orc_matrix_nnz": (C.c_long, [vp]),
            "orc_matrix_export": (None, [vp, _ip, _ip, _dp, _ip]),
            "orc_residual_inf_norm": (C.c_double, [vp, _dp, _dp]),
            "orc_inf_norm": (C.c_double, [_dp, C.c_long]),
            "orc_schedule_order": (C.c_int, [_Sched, vp, _ip, _ip, _ip]),
            "orc_engine_create": (vp, [vp, C.c_char_p, C.c_size_t]),
            "orc_engine_free": (None, [vp]),
            "orc_engine_num_edges": (C.c_long, [vp]),
            "orc_sweep_flops": (C.c_double, [vp]),
            "orc_sweep": (C.c_int, [vp, _dp, _Sched, _dp, _dp, _dp, C.c_char_p, C.c_size_t]),
            "orc_solve": (C.c_int, [vp, _dp, _Sched, C.c_double, C.c_int, C.c_int, C.c_double,
                                    _dp, _dp, _ip, _ip, _dp, C.c_char_p, C.c_size_t]),
            "orc_precompute_lambda": (C.c_int, [vp, _Sched, C.c_double, C.c_int, _dp, _dp, _ip, _ip]),
            "orc_correction_sweeps": (C.c_int, [vp, _dp, _Sched, _dp, _dp, C.c_int, _dp]),
            "orc_error_correction_apply_frozen": (C.c_int, [vp, _dp, _dp, C.c_int, _Sched, _dp, _dp, _dp]),
            "orc_error_correction_apply_cold": (C.c_int, [vp, _dp, _dp, C.c_int, _Sched, _dp,
                                                          C.c_char_p, C.c_size_t]),
            "orc_solve_error_correction": (C.c_int, [vp, _dp, _Sched, C.c_int, _dp, _dp, C.c_double,
                                                     C.c_int, C.c_double, _dp, _dp, _ip, _ip, _dp,
                                                     C.c_char_p, C.c_size_t]),
            "orc_node_precisions": (None, [vp, _dp, _dp, _dp]),
            "orc_computation_tree_solve": (C.c_int, [vp, _dp, C.c_int, C.c_int, C.c_long, _dp,
                                                     C.c_char_p, C.c_size_t]),
            "orc_mg_create": (vp, [C.c_int, C.POINTER(vp), _ip, C.c_int, C.c_char_p, C.c_size_t]),
            "orc_mg_free": (None, [vp]),
            "orc_mg_num_levels": (C.c_int, [vp]),
            "orc_mg_level_frozen_ok": (C.c_int, [vp, C.c_int]),
            "orc_mg_vcycle": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_char_p, C.c_size_t]),
            "orc_mg_solve": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, _dp, C.c_double, C.c_int,
                                       C.c_double, _dp, _dp, _ip, _ip, _dp, _ip, C.c_char_p, C.c_size_t]),
            "orc_mg_cycle_flops": (C.c_double, [vp, C.c_int, C.c_int]),
            "orc_set_damping": (C.c_int, [vp, C.c_double]),
            "orc_set_threads": (C.c_int, [C.c_int]),

            "orc_flop_table": (C.c_double, [C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_size_t]),
            "orc_mg_restrict": (None, [_dp, C.c_int, _dp]),
            "orc_mg_prolong": (None, [_dp, C.c_int, _dp]),
            "orc_gs_sweeps": (C.c_int, [vp, _dp, _dp, _Sched, C.c_int, C.c_char_p, C.c_size_t]),
            "orc_dense_solve": (C.c_int, [vp, _dp, _dp]),
            "orc_region_create": (vp, [vp, C.c_int, _ip, _ip, C.c_char_p, C.c_size_t]),
            "orc_region_free": (None, [vp]),
            "orc_region_num_edges": (C.c_int, [vp]),
            "orc_region_num_small": (C.c_int, [vp]),
            "orc_region_state_size": (C.c_long, [vp, C.POINTER(C.c_long)]),
            "orc_region_edges": (None, [vp, _ip, _ip]),
            "orc_region_small": (C.c_long, [vp, _ip, _ip, _ip, _ip, _ip]),
            "orc_region_sweep": (C.c_int, [vp, _dp, C.c_int, _dp, _dp, _dp, C.c_char_p, C.c_size_t]),
            "orc_region_solve": (C.c_int, [vp, _dp, C.c_double, C.c_int, C.c_int, C.c_double, _dp, _dp, _ip, _ip,
                                           _dp, C.c_char_p, C.c_size_t]),
            "orc_region_direct_message": (C.c_int, [vp, _dp, _dp, _dp, C.c_int, _dp, _dp, C.c_char_p, C.c_size_t]),
            "orc_region_flops": (C.c_double, [vp, C.c_int]),
        }
        gens = {
            "orc_rng_new": (vp, [C.c_uint]),
            "orc_rng_free": (None, [vp]),
            "orc_rng_uniform_int": (C.c_int, [vp, C.c_int, C.c_int]),
            "orc_random_vector": (None, [vp, C.c_int, _dp]),
            "orc_random_diag_dominant": (vp, [vp, C.c_int, C.c_int, C.c_double]),
            "orc_random_tree": (vp, [vp, C.c_int, _ip]),
            "orc_random_cycle_chords": (vp, [vp, C.c_int]),
            "orc_poisson5": (vp, [C.c_int, C.c_int]),
            "orc_config3": (vp, [C.c_int, C.c_double, C.c_double, C.c_uint, _dp]),
            "orc_config4": (vp, [C.c_int, C.c_double, C.c_double, C.c_double, C.c_uint, _dp]),
            "orc_config5_level": (vp, [C.c_int, C.c_int, C.c_uint, C.c_double, _dp]),
            "orc_example7x7": (vp, []),
            "orc_tree_diameter": (C.c_int, [C.c_int, _ip]),
        }
        self.has_generators = hasattr(L, "orc_rng_new")
        if self.has_generators:
            sig.update(gens)
        self.has_region_graph = hasattr(L, "ref_region_graph")
        if self.has_region_graph:  # the reference's own region.cpp builder (reference build only)
            sig["ref_region_graph"] = (C.c_long, [vp, C.c_int, _ip, _ip, _ip, _ip, _ip, _ip, _ip, C.c_char_p,
                                                  C.c_size_t])
        self.has_assemble = hasattr(L, "ref_assemble")
        if self.has_assemble:
            sig["ref_assemble"] = (vp, [C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_char_p), _dp,
                                        _dp, _dp, _ip, _dp, C.c_char_p, C.c_size_t])
        self.has_ref_full = hasattr(L, "ref_hier_create")
        if self.has_ref_full:  # multigrid.cpp / classic.cpp / region_gabp.cpp over the Eigen stand-in
            sig.update({
                "ref_hier_create": (vp, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_char_p), _dp, C.c_int,
                                         C.c_char_p, C.c_size_t]),
                "ref_hier_free": (None, [vp]),
                "ref_hier_num_levels": (C.c_int, [vp]),
                "ref_hier_level_n": (C.c_int, [vp, C.c_int]),
                "ref_hier_level_nx": (C.c_int, [vp, C.c_int]),
                "ref_hier_level_frozen_ok": (C.c_int, [vp, C.c_int]),
                "ref_hier_fine_rhs": (None, [vp, _dp, _dp]),
                "ref_hier_vcycle": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_char_p, C.c_size_t]),
                "ref_hier_cycle_flops": (C.c_double, [vp, C.c_int, C.c_int]),
                "ref_hier_solve": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, _dp, C.c_double, C.c_int, C.c_double,
                                             _dp, _dp, _ip, _ip, _dp, _ip, C.c_char_p, C.c_size_t]),
                "ref_relax": (C.c_int, [C.c_int, vp, _dp, _dp, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_size_t]),
                "ref_region_create": (vp, [vp, C.c_int, _ip, _ip, C.c_char_p, C.c_size_t]),
                "ref_region_free": (None, [vp]),
                "ref_region_num_edges": (C.c_int, [vp]),
                "ref_region_state_size": (C.c_long, [vp, C.POINTER(C.c_long)]),
                "ref_region_sweep": sig["orc_region_sweep"],
                "ref_region_solve": sig["orc_region_solve"],
                "ref_region_direct_message": sig["orc_region_direct_message"],
                "ref_region_flops": (C.c_double, [vp, C.c_int]),
                "ref_block_convergence": (C.c_double, [vp, C.c_int, _ip, _ip, C.c_int, _ip, _ip]),
            })
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args

    # ---- loading --------------------------------------------------------------------------
    @classmethod
    def restatement(cls):
        if RESTATE_SO not in cls._cache:
            if not os.path.exists(RESTATE_SO):
                raise FileNotFoundError(f"{RESTATE_SO} missing: run `make -C oracle` (or __graft_entry__.build())")
            cls._cache[RESTATE_SO] = cls(RESTATE_SO)
        return cls._cache[RESTATE_SO]

    @classmethod
    def reference(cls):
        if not os.path.exists(REF_SO):
            return None
        if REF_SO not in cls._cache:
            cls._cache[REF_SO] = cls(REF_SO)
        return cls._cache[REF_SO]

    # ---- matrices -------------------------------------------------------------------------
    def _export(self, h) -> Csr:
        L = self.lib
        n = L.orc_matrix_n(h)
        nnz = L.orc_matrix_nnz(h)
        ro = np.zeros(n + 1, np.int32)
        ci = np.zeros(nnz, np.int32)
        v = np.zeros(nnz, np.float64)
        tp = np.zeros(nnz, np.int32)
        L.orc_matrix_export(h, _i(ro), _i(ci), _d(v), _i(tp))
        return Csr(n, ro, ci, v, tp)

    def _own(self, h) -> Csr:
        try:
            return self._export(h)
        finally:
            self.lib.orc_matrix_free(h)

    def make_csr(self, n, rows, cols, vals) -> Csr:
        rows, cols, vals = i32(rows), i32(cols), f64(vals)
        err = C.create_string_buffer(256)
        h = self.lib.orc_make_csr(n, len(rows), _i(rows), _i(cols), _d(vals), err, 256)
        if not h:
            raise ValueError(err.value.decode())
        return self._own(h)

    def _handle(self, A: Csr):
        ro, ci, v = i32(A.row_offsets), i32(A.col_indices), f64(A.values)
        return self.lib.orc_matrix_from_csr(A.n, _i(ro), _i(ci), _d(v))

    def canonical(self, A: Csr) -> Csr:
        """Round-trip through this library (recomputes transpose_pos as make_csr does)."""
        return self._own(self._handle(A))

    def residual_inf_norm(self, A: Csr, x, b) -> float:
        h = self._handle(A)
        try:
            return self.lib.orc_residual_inf_norm(h, _d(f64(x)), _d(f64(b)))
        finally:
            self.lib.orc_matrix_free(h)

    def schedule_order(self, A: Csr, sched: Schedule):
        h = self._handle(A)
        order = np.zeros(A.n, np.int32)
        color = np.full(A.n, -1, np.int32)
        nc = C.c_int(0)
        try:
            rc = self.lib.orc_schedule_order(sched.c(), h, _i(order), _i(color), C.byref(nc))
        finally:
            self.lib.orc_matrix_free(h)
        if rc != 1:
            raise ValueError("bad schedule")
        return order, color, nc.value

    def dense_solve(self, A: Csr, b):
        h = self._handle(A)
        x = np.zeros(A.n)
        try:
            self.lib.orc_dense_solve(h, _d(f64(b)), _d(x))
        finally:
            self.lib.orc_matrix_free(h)
        return x

    def computation_tree_solve(self, A: Csr, b, root, depth, node_cap=100000):
        h = self._handle(A)
        out = C.c_double(0)
        err = C.create_string_buffer(256)
        try:
            ok = self.lib.orc_computation_tree_solve(h, _d(f64(b)), root, depth, node_cap, C.byref(out), err, 256)
        finally:
            self.lib.orc_matrix_free(h)
        if not ok:
            raise RuntimeError(err.value.decode())
        return out.value

    def mg_restrict(self, fine, mf):
        mc = (mf - 1) // 2
        out = np.zeros(mc * mc)
        self.lib.orc_mg_restrict(_d(f64(fine)), mf, _d(out))
        return out

    def mg_prolong(self, coarse, mc):
        mf = 2 * mc + 1
        out = np.zeros(mf * mf)
        self.lib.orc_mg_prolong(_d(f64(coarse)), mc, _d(out))
        return out

    def gs_sweeps(self, A: Csr, b, x, sched: Schedule, sweeps):
        h = self._handle(A)
        x = f64(x).copy()
        err = C.create_string_buffer(256)
        try:
            rc = self.lib.orc_gs_sweeps(h, _d(f64(b)), _d(x), sched.c(), sweeps, err, 256)
        finally:
            self.lib.orc_matrix_free(h)
        if rc != 1:
            raise RuntimeError(err.value.decode())
        return x

    def set_threads(self, k):
        """Threads of the restatement's parallel flood evaluation (bit-identical to serial)."""
        return self.lib.orc_set_threads(int(k))

    def flop_table(self, stencil, smoother, sweeps):
        """analysis.cpp:135-154; ValueError on the reference's std::invalid_argument."""
        err = C.create_string_buffer(256)
        v = self.lib.orc_flop_table(stencil, smoother, sweeps, err, 256)
        if v == -1.0 and err.value:
            raise ValueError(err.value.decode())
        return v

    # ---- generators (restatement only) -----------------------------------------------------
    def rng(self, seed):
        return _Rng(self, seed)

    def poisson5(self, nx, ny) -> Csr:
        return self._own(self.lib.orc_poisson5(nx, ny))

    def config_problem(self, config, size=0, seed=None, sigma=2.0):
        """BASELINE.json configs 1-5 from the oracle's own generators (restatement only):
        (A, b).  Config 5 is its finest level (J with 2^J - 1 = size, default 4095)."""
        seed = {1: 0, 2: 1, 3: 2, 4: 3, 5: 4}[config] if seed is None else seed
        if config in (1, 2):
            N = size or (64 if config == 1 else 2048)
            A = self.poisson5(N, N)
            return A, self.rng(seed).vector(A.n)
        if config == 3:
            N = size or 1024
            b = np.zeros(N * N)
            return self._own(self.lib.orc_config3(N, 2.0, 0.3, seed, _d(b))), b
        if config == 4:
            N = size or 256
            b = np.zeros(N ** 3)
            return self._own(self.lib.orc_config4(N, 1.0, 1.0, 0.01, seed, _d(b))), b
        if config == 5:
            return self.config5_level(int(np.log2((size or 4095) + 1)), 0, seed, sigma)
        raise ValueError(f"config {config}")

    def config5_level(self, J, k, seed=4, sigma=2.0):
        m = (1 << (J - k)) - 1
        b = np.zeros(((1 << J) - 1) ** 2) if k == 0 else None
        A = self._own(self.lib.orc_config5_level(J, k, seed, sigma, _d(b) if b is not None else None))
        assert A.n == m * m
        return A, b

    def example7x7(self) -> Csr:
        return self._own(self.lib.orc_example7x7())

    def tree_diameter(self, n, edges):
        e = i32(edges)
        return self.lib.orc_tree_diameter(n, _i(e))

    def assemble(self, name, J, params=None):
        """Reference problem assembly (reference library only)."""
        params = params or {}
        m = (1 << J) - 1
        b = np.zeros(m * m)
        exact = np.zeros(m * m)
        nx = C.c_int(0)
        h = C.c_double(0)
        keys = (C.c_char_p * max(1, len(params)))(*[k.encode() for k in params])
        vals = f64(list(params.values()) or [0.0])
        err = C.create_string_buffer(256)
        H = self.lib.ref_assemble(name.encode(), J, len(params), keys, _d(vals), _d(b), _d(exact),
                                  C.byref(nx), C.byref(h), err, 256)
        if not H:
            raise ValueError(err.value.decode())
        return self._own(H), b, exact, nx.value, h.value

    # ---- engine ---------------------------------------------------------------------------
    def engine(self, A: Csr):
        return _Engine(self, A)

    def region(self, A: Csr, large):
        """RegionGabpEngine(A, build_two_layer_region_graph(A, large)) (region_gabp.cpp:30-198)."""
        return _Region(self, A, large)

    def grid_lines(self, nx, ny):
        """grid_line_regions(nx, ny) (region.cpp:208-221)."""
        rows = [[iy * nx + ix for ix in range(nx)] for iy in range(ny)]
        cols = [[iy * nx + ix for iy in range(ny)] for ix in range(nx)]
        return rows + cols

    def region_graph_ref(self, A: Csr, large):
        """The reference's own build_two_layer_region_graph (ref build): (small, parents, counting)."""
        offs, idx = _flatten_lists(large)
        h = self._handle(A)
        err = C.create_string_buffer(512)
        try:
            ns = self.lib.ref_region_graph(h, len(large), _i(offs), _i(idx), None, None, None, None, None, err, 512)
            if ns < 0:
                raise ValueError(err.value.decode())
            cap = sum(len(r) for r in large) * 2 + 1
            so, sv, po, pv, cnt = (np.zeros(ns + 1, np.int32), np.zeros(cap, np.int32), np.zeros(ns + 1, np.int32),
                                   np.zeros(cap, np.int32), np.zeros(max(ns, 1), np.int32))
            self.lib.ref_region_graph(h, len(large), _i(offs), _i(idx), _i(so), _i(sv), _i(po), _i(pv), _i(cnt),
                                      err, 512)
        finally:
            self.lib.orc_matrix_free(h)
        return ([list(sv[so[k]:so[k + 1]]) for k in range(ns)], [list(pv[po[k]:po[k + 1]]) for k in range(ns)],
                list(cnt[:ns]))

    def hierarchy(self, levels, nx, smoother):
        return _Hierarchy(self, levels, nx, smoother)

    # ---- the reference's own multigrid.cpp / classic.cpp / region_gabp.cpp (reference build only;
    # compiled over oracle/eigen_shim, see oracle/Makefile) ----------------------------------
    def ref_hierarchy(self, problem, J1, J2, params, smoother):
        """belief::Hierarchy(problem, J1, J2, params, smoother) (multigrid.cpp:74-109)."""
        return _RefHierarchy(self, problem, J1, J2, params or {}, smoother)

    def ref_region(self, A: Csr, large):
        """belief::RegionGabpEngine over belief::build_two_layer_region_graph (region_gabp.cpp)."""
        return _Region(self, A, large, prefix="ref_region")

    def ref_relax(self, kind, A: Csr, b, x, sweeps, nx=0, ny=0):
        """belief::relax (classic.cpp:99-146); kind = belief::RelaxKind (0 Jacobi, 1 GsLex, 2 GsRedBlack,
        3 GsFourColor, 4 LineGsX, 5 LineGsY, 6 ZebraX, 7 AlternatingZebra)."""
        x = f64(x).copy()
        h = self._handle(A)
        err = C.create_string_buffer(256)
        rc = self.lib.ref_relax(kind, h, _d(f64(b)), _d(x), sweeps, nx, ny, err, 256)
        self.lib.orc_matrix_free(h)
        if rc != 1:
            raise RuntimeError(err.value.decode())
        return x

    def ref_block_convergence(self, A: Csr, blocks, spectral=False):
        """check_block_convergence (region_gabp.cpp:276-309): (rho, sufficient, singular_block)."""
        offs, idx = _flatten_lists(blocks)
        h = self._handle(A)
        suf, sing = C.c_int(0), C.c_int(0)
        rho = self.lib.ref_block_convergence(h, len(blocks), _i(offs), _i(idx), int(spectral), C.byref(suf),
                                             C.byref(sing))
        self.lib.orc_matrix_free(h)
        return rho, bool(suf.value), sing.value


class _Rng:
    def __init__(self, orc: Oracle, seed):
        self.o = orc
        self.h = orc.lib.orc_rng_new(seed)

    def __del__(self):
        try:
            self.o.lib.orc_rng_free(self.h)
        except Exception:
            pass

    def uniform_int(self, lo, hi):
        return self.o.lib.orc_rng_uniform_int(self.h, lo, hi)

    def vector(self, n):
        out = np.zeros(n)
        self.o.lib.orc_random_vector(self.h, n, _d(out))
        return out

    def diag_dominant(self, n, symmetric, edge_prob=0.25) -> Csr:
        return self.o._own(self.o.lib.orc_random_diag_dominant(self.h, n, int(symmetric), edge_prob))

    def tree(self, n):
        edges = np.zeros(2 * max(n - 1, 1), np.int32)
        A = self.o._own(self.o.lib.orc_random_tree(self.h, n, _i(edges)))
        return A, edges[: 2 * (n - 1)]

    def cycle_chords(self, n) -> Csr:
        return self.o._own(self.o.lib.orc_random_cycle_chords(self.h, n))


class _Engine:
    """GabpEngine (gabp.hpp:58-111) over CSR-position message arrays."""

    def __init__(self, orc: Oracle, A: Csr):
        self.o, self.A = orc, A
        self.mh = orc._handle(A)
        err = C.create_string_buffer(256)
        self.h = orc.lib.orc_engine_create(self.mh, err, 256)
        if not self.h:
            orc.lib.orc_matrix_free(self.mh)
            self.mh = None
            raise ValueError(err.value.decode())

    def __del__(self):
        try:
            if self.h:
                self.o.lib.orc_engine_free(self.h)
            if self.mh:
                self.o.lib.orc_matrix_free(self.mh)
        except Exception:
            pass

    @property
    def num_edges(self):
        return self.o.lib.orc_engine_num_edges(self.h)

    def set_damping(self, alpha):
        """Flood message damping (restatement only; the reference engine accepts just 0)."""
        if self.o.lib.orc_set_damping(self.h, float(alpha)) != 1:
            raise ValueError("damping is not available in the reference engine")

    def sweep_flops(self):
        return self.o.lib.orc_sweep_flops(self.h)

    def make_state(self):
        return np.zeros(self.A.nnz), np.zeros(self.A.nnz)

    def sweep(self, b, sched: Schedule, lam, m, x):
        """In-place on (lam, m, x); returns (ok, err)."""
        err = C.create_string_buffer(512)
        rc = self.o.lib.orc_sweep(self.h, _d(f64(b)), sched.c(), _d(lam), _d(m), _d(x), err, 512)
        if rc < 0:
            raise ValueError(err.value.decode())
        return rc == 1, err.value.decode()

    def solve(self, b, sched: Schedule, tol=2e-4, max_iter=20000, stop=0, divergence_factor=1e12):
        n = self.A.n
        x = np.zeros(n)
        hist = np.zeros(max_iter + 1)
        it, st, fl = C.c_int(0), C.c_int(0), C.c_double(0)
        det = C.create_string_buffer(512)
        rc = self.o.lib.orc_solve(self.h, _d(f64(b)), sched.c(), tol, max_iter, stop, divergence_factor,
                                  _d(x), _d(hist), C.byref(it), C.byref(st), C.byref(fl), det, 512)
        if rc < 0:
            raise ValueError(det.value.decode())
        d = det.value.decode()
        # a pivot stop pushes no residual for its iteration (gabp.cpp:193-199)
        nh = it.value + (0 if st.value == 1 and d.startswith("zero pivot") else 1)
        return Report(st.value, it.value, hist[:nh].copy(), fl.value, x, d)

    def precompute_lambda(self, sched: Schedule, tol=1e-10, max_iter=500):
        lam = np.zeros(self.A.nnz)
        sig = np.zeros(self.A.n)
        cv, it = C.c_int(0), C.c_int(0)
        rc = self.o.lib.orc_precompute_lambda(self.h, sched.c(), tol, max_iter, _d(lam), _d(sig),
                                              C.byref(cv), C.byref(it))
        if rc < 0:
            raise ValueError("schedule order does not cover every node")
        return lam, sig, bool(cv.value), it.value

    def correction_sweeps(self, r, sched, lam, sigma, sweeps):
        e = np.zeros(self.A.n)
        rc = self.o.lib.orc_correction_sweeps(self.h, _d(f64(r)), sched.c(), _d(f64(lam)), _d(f64(sigma)),
                                              sweeps, _d(e))
        if rc < 0:
            raise ValueError("schedule order does not cover every node")
        return e

    def error_correction_apply(self, b, x0, sweeps, sched, lam=None, sigma=None):
        x = np.zeros(self.A.n)
        if lam is not None:
            self.o.lib.orc_error_correction_apply_frozen(self.h, _d(f64(b)), _d(f64(x0)), sweeps, sched.c(),
                                                         _d(f64(lam)), _d(f64(sigma)), _d(x))
            return x
        err = C.create_string_buffer(512)
        rc = self.o.lib.orc_error_correction_apply_cold(self.h, _d(f64(b)), _d(f64(x0)), sweeps, sched.c(),
                                                        _d(x), err, 512)
        if rc != 1:
            raise RuntimeError(err.value.decode())
        return x

    def solve_error_correction(self, b, sched, sweeps, lam, sigma, tol=2e-4, max_iter=20000,
                               divergence_factor=1e12):
        n = self.A.n
        x = np.zeros(n)
        hist = np.zeros(max_iter + 1)
        it, st, fl = C.c_int(0), C.c_int(0), C.c_double(0)
        det = C.create_string_buffer(512)
        self.o.lib.orc_solve_error_correction(self.h, _d(f64(b)), sched.c(), sweeps, _d(f64(lam)),
                                              _d(f64(sigma)), tol, max_iter, divergence_factor, _d(x),
                                              _d(hist), C.byref(it), C.byref(st), C.byref(fl), det, 512)
        return Report(st.value, it.value, hist[: it.value + 1].copy(), fl.value, x, det.value.decode())

    def node_precisions(self, lam, m):
        beta = np.zeros(self.A.n)
        self.o.lib.orc_node_precisions(self.h, _d(f64(lam)), _d(f64(m)), _d(beta))
        return beta


class _Hierarchy:
    """Multigrid restatement (multigrid.cpp:54-318) over caller-supplied levels."""

    def __init__(self, orc: Oracle, levels, nx, smoother):
        self.o = orc
        hs = [orc._handle(A) for A in levels]
        arr = (C.c_void_p * len(hs))(*hs)
        nxa = i32(nx)
        err = C.create_string_buffer(256)
        self.h = orc.lib.orc_mg_create(len(hs), arr, _i(nxa), smoother, err, 256)
        for h in hs:
            orc.lib.orc_matrix_free(h)
        if not self.h:
            raise ValueError(err.value.decode())
        self.n = levels[0].n

    def __del__(self):
        try:
            self.o.lib.orc_mg_free(self.h)
        except Exception:
            pass

    @property
    def num_levels(self):
        return self.o.lib.orc_mg_num_levels(self.h)

    def frozen_ok(self, k):
        return bool(self.o.lib.orc_mg_level_frozen_ok(self.h, k))

    def v_cycle(self, pre, post, b, x, frozen=False):
        """One V-cycle.  Returns x; on a smoother breakdown raises RuntimeError with the
        partly updated x (multigrid.cpp:234-238 updates the caller's x in place) as args[1]."""
        x = f64(x).copy()
        err = C.create_string_buffer(512)
        rc = self.o.lib.orc_mg_vcycle(self.h, pre, post, int(frozen), _d(f64(b)), _d(x), err, 512)
        if rc != 1:
            raise RuntimeError(err.value.decode(), x)
        return x

    def cycle_flops_per_unknown(self, pre, post):
        return self.o.lib.orc_mg_cycle_flops(self.h, pre, post)

    def solve(self, pre, post, b, tol=2e-4, max_cycles=200, divergence_factor=1e6, frozen=False):
        x = np.zeros(self.n)
        hist = np.zeros(max_cycles + 1)
        it, st, hl = C.c_int(0), C.c_int(0), C.c_int(0)
        fl = C.c_double(0.0)
        det = C.create_string_buffer(512)
        self.o.lib.orc_mg_solve(self.h, pre, post, int(frozen), _d(f64(b)), tol, max_cycles,
                                divergence_factor, _d(x), _d(hist), C.byref(it), C.byref(st), C.byref(fl),
                                C.byref(hl), det, 512)
        return Report(st.value, it.value, hist[: hl.value].copy(), fl.value, x, det.value.decode())


class _RefHierarchy:
    """The reference's own belief::Hierarchy / v_cycle / mg_solve (multigrid.cpp), named problems only."""

    def __init__(self, orc: Oracle, problem, J1, J2, params, smoother):
        self.o = orc
        keys = (C.c_char_p * max(1, len(params)))(*[k.encode() for k in params])
        vals = f64(list(params.values()) or [0.0])
        err = C.create_string_buffer(512)
        self.h = orc.lib.ref_hier_create(problem.encode(), J1, J2, len(params), keys, _d(vals), smoother, err, 512)
        if not self.h:
            raise ValueError(err.value.decode())
        self.n = orc.lib.ref_hier_level_n(self.h, 0)

    def __del__(self):
        try:
            self.o.lib.ref_hier_free(self.h)
        except Exception:
            pass

    @property
    def num_levels(self):
        return self.o.lib.ref_hier_num_levels(self.h)

    def level_n(self, k):
        return self.o.lib.ref_hier_level_n(self.h, k)

    def frozen_ok(self, k):
        return bool(self.o.lib.ref_hier_level_frozen_ok(self.h, k))

    def fine_rhs(self):
        b, e = np.zeros(self.n), np.zeros(self.n)
        self.o.lib.ref_hier_fine_rhs(self.h, _d(b), _d(e))
        return b, e

    def v_cycle(self, pre, post, b, x, frozen=False):
        x = f64(x).copy()
        err = C.create_string_buffer(512)
        rc = self.o.lib.ref_hier_vcycle(self.h, pre, post, int(frozen), _d(f64(b)), _d(x), err, 512)
        if rc != 1:
            raise RuntimeError(err.value.decode(), x)
        return x

    def cycle_flops_per_unknown(self, pre, post):
        return self.o.lib.ref_hier_cycle_flops(self.h, pre, post)

    def solve(self, pre, post, b, tol=2e-4, max_cycles=200, divergence_factor=1e6, frozen=False):
        x = np.zeros(self.n)
        hist = np.zeros(max_cycles + 1)
        it, st, hl = C.c_int(0), C.c_int(0), C.c_int(0)
        fl = C.c_double(0.0)
        det = C.create_string_buffer(512)
        rc = self.o.lib.ref_hier_solve(self.h, pre, post, int(frozen), _d(f64(b)), tol, max_cycles,
                                       divergence_factor, _d(x), _d(hist), C.byref(it), C.byref(st), C.byref(fl),
                                       C.byref(hl), det, 512)
        if rc != 1:
            raise RuntimeError(det.value.decode())
        return Report(st.value, it.value, hist[: hl.value].copy(), fl.value, x, det.value.decode())


def _flatten_lists(lists):
    offs = np.zeros(len(lists) + 1, np.int32)
    offs[1:] = np.cumsum([len(r) for r in lists])
    idx = np.array([v for r in lists for v in r] or [0], np.int32)
    return offs, idx


class _Region:
    """Region GaBP restatement (region_gabp.cpp:30-198, region_restate.inc).  State is flat:
    Lambda blocks (row-major |l| x |l|) and m blocks per edge, in the engine's edge order."""

    def __init__(self, orc: Oracle, A: Csr, large, prefix="orc_region"):
        self.o = orc
        self.p = prefix  # "ref_region": the reference's own RegionGabpEngine (same flat state layout)
        offs, idx = _flatten_lists(large)
        h = orc._handle(A)
        err = C.create_string_buffer(512)
        self.h = self._f("create")(h, len(large), _i(offs), _i(idx), err, 512)
        orc.lib.orc_matrix_free(h)
        if not self.h:
            raise ValueError(err.value.decode())
        self.n = A.n
        ms = C.c_long(0)
        self.lam_size = self._f("state_size")(self.h, C.byref(ms))
        self.m_size = ms.value

    def _f(self, name):
        return getattr(self.o.lib, f"{self.p}_{name}")

    def __del__(self):
        try:
            self._f("free")(self.h)
        except Exception:
            pass

    @property
    def num_edges(self):
        return self._f("num_edges")(self.h)

    def edges(self):
        E = self.num_edges
        el, es = np.zeros(max(E, 1), np.int32), np.zeros(max(E, 1), np.int32)
        self.o.lib.orc_region_edges(self.h, _i(el), _i(es))
        return el[:E], es[:E]

    def small(self):
        ns = self.o.lib.orc_region_num_small(self.h)
        nv = self.o.lib.orc_region_small(self.h, None, None, None, None, None)
        so, sv, po, pv, cnt = (np.zeros(ns + 1, np.int32), np.zeros(max(nv, 1), np.int32), np.zeros(ns + 1, np.int32),
                               np.zeros(max(nv * 8, 1), np.int32), np.zeros(max(ns, 1), np.int32))
        self.o.lib.orc_region_small(self.h, _i(so), _i(sv), _i(po), _i(pv), _i(cnt))
        return ([list(sv[so[k]:so[k + 1]]) for k in range(ns)], [list(pv[po[k]:po[k + 1]]) for k in range(ns)],
                list(cnt[:ns]))

    def make_state(self):
        return np.zeros(self.lam_size), np.zeros(self.m_size)

    def sweep(self, b, lam, m, x, mode=0):
        """One sweep (mode 0 Sequential, 1 Flood), in place; returns (ok, err)."""
        err = C.create_string_buffer(512)
        rc = self._f("sweep")(self.h, _d(f64(b)), mode, _d(lam), _d(m), _d(x), err, 512)
        return rc == 1, err.value.decode()

    def solve(self, b, tol=2e-4, max_iter=10000, mode=0, divergence_factor=1e12):
        x = np.zeros(self.n)
        hist = np.zeros(max_iter + 1)
        it, st, fl = C.c_int(0), C.c_int(0), C.c_double(0)
        det = C.create_string_buffer(512)
        self._f("solve")(self.h, _d(f64(b)), tol, max_iter, mode, divergence_factor, _d(x), _d(hist),
                                    C.byref(it), C.byref(st), C.byref(fl), det, 512)
        return Report(st.value, it.value, hist[: it.value + 1].copy(), fl.value, x, det.value.decode())

    def direct_message(self, b, lam, m, edge, nl=1):
        lo, mo = np.zeros(nl * nl), np.zeros(nl)
        err = C.create_string_buffer(512)
        if self._f("direct_message")(self.h, _d(f64(b)), _d(f64(lam)), _d(f64(m)), edge, _d(lo), _d(mo),
                                                err, 512) != 1:
            raise RuntimeError(err.value.decode())
        return lo, mo

    def flops(self, per_child=False):
        return self._f("flops")(self.h, int(per_child))
