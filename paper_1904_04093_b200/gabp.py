"""Python host mirror of the reference's GaBP solver / smoother API over the C-ABI.

Names, argument meaning and error behaviour follow proj/core/include/belief/{gabp,schedule,
report,multigrid,problems}.hpp so tests and drivers read like the reference's own:

    GabpEngine(A).solve(b, Schedule.parallel_flood(), GabpOptions(tol=...))
    Hierarchy("poisson", J1, J2, {}, MgSmoother.GabpRedBlack); mg_solve(h, CycleSpec(...), b, opt)

Every call goes through libgabp_b200.so (include/gabp_b200.h) and runs on the GPU.  There is no
CPU fallback: if the library is missing or no CUDA device is present the calls raise.
std::invalid_argument maps to ValueError, std::runtime_error to RuntimeError.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgabp_b200.so")

_dp, _ip, _vp = C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_void_p

OK, EINVAL, EPIVOT, ECUDA, ERUNTIME = range(5)


class _Sched(C.Structure):
    _fields_ = [("kind", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("order", _ip)]


class _Opts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int), ("stop", C.c_int), ("divergence_factor", C.c_double)]


class _Rep(C.Structure):
    _fields_ = [("status", C.c_int), ("iterations", C.c_int), ("flop_estimate", C.c_double)]


class _LinOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int), ("mode", C.c_int), ("divergence_factor", C.c_double)]


class _Info(C.Structure):
    _fields_ = [("n", C.c_int), ("nnz", C.c_longlong), ("num_edges", C.c_longlong), ("layout", C.c_int),
                ("num_slots", C.c_int), ("symmetric_values", C.c_int), ("bytes_per_sweep", C.c_double),
                ("bytes_per_residual", C.c_double), ("device_bytes", C.c_longlong),
                ("uniform_coefficients", C.c_int), ("sell_slots", C.c_longlong)]


class _Cycle(C.Structure):
    _fields_ = [("pre", C.c_int), ("post", C.c_int), ("frozen", C.c_int)]


class _MgOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_cycles", C.c_int), ("divergence_factor", C.c_double)]


_LIB = None


def lib():
    """The loaded C-ABI library (raises if it was never built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `make -C {_HERE}/csrc` "
                               "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        S = C.POINTER(_Sched)
        sig = {
            "bgabp_version": (C.c_char_p, []),
            "bgabp_create": (C.c_int, [C.c_int, _ip, _ip, _dp, C.c_int, C.POINTER(_vp), C.c_char_p, C.c_size_t]),
            "bgabp_destroy": (None, [_vp]),
            "bgabp_get_info": (C.c_int, [_vp, C.POINTER(_Info)]),
            "bgabp_stream": (_vp, [_vp]),
            "bgabp_layout_digest": (C.c_int, [_vp, C.POINTER(C.c_ulonglong)]),
            "bgabp_reset_state": (C.c_int, [_vp]),
            "bgabp_set_state": (C.c_int, [_vp, _dp, _dp]),
            "bgabp_get_state": (C.c_int, [_vp, _dp, _dp]),
            "bgabp_sweep": (C.c_int, [_vp, _dp, S, _dp, C.c_char_p, C.c_size_t]),
            "bgabp_node_precisions": (C.c_int, [_vp, _dp]),
            "bgabp_sweep_flops": (C.c_double, [_vp]),
            "bgabp_set_damping": (C.c_int, [_vp, C.c_double]),
            "bgabp_dia_offsets": (C.c_int, [_vp, _ip, C.c_int]),
            "bgabp_trim_cache": (None, []),
            "bgabp_solve": (C.c_int, [_vp, _dp, S, C.POINTER(_Opts), C.POINTER(_Rep), _dp, _dp, C.c_char_p,
                                      C.c_size_t]),
            "bgabp_solve_device_begin": (C.c_int, [_vp, _vp, S, C.POINTER(_Opts)]),
            "bgabp_solve_device_steps": (C.c_int, [_vp, C.c_int]),
            "bgabp_solve_device_end": (C.c_int, [_vp, C.POINTER(_Rep), _vp, _vp, C.c_char_p, C.c_size_t]),
            "bgabp_flood_sweeps_device": (C.c_int, [_vp, _vp, C.c_int]),
            "bgabp_solve_device_steps_timed": (C.c_int, [_vp, C.c_int, _dp]),
            "bgabp_residual_inf_norm": (C.c_int, [_vp, _dp, _dp, _dp]),
            "bgabp_precompute_lambda": (C.c_int, [_vp, S, C.c_double, C.c_int, _dp, _dp, _ip, _ip]),
            "bgabp_set_frozen": (C.c_int, [_vp, _dp, _dp]),
            "bgabp_correction_sweeps": (C.c_int, [_vp, _dp, S, C.c_int, _dp]),
            "bgabp_error_correction_apply": (C.c_int, [_vp, _dp, _dp, C.c_int, S, C.c_int, _dp, C.c_char_p,
                                                       C.c_size_t]),
            "bgabp_solve_error_correction": (C.c_int, [_vp, _dp, S, C.c_int, C.POINTER(_Opts), C.POINTER(_Rep),
                                                       _dp, _dp, C.c_char_p, C.c_size_t]),
            "bgmg_create": (C.c_int, [C.c_int, _ip, C.POINTER(_ip), C.POINTER(_ip), C.POINTER(_dp), _ip, C.c_int,
                                      C.POINTER(_vp), C.c_char_p, C.c_size_t]),
            "bgmg_create_named": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_char_p), _dp,
                                            C.c_int, C.POINTER(_vp), C.c_char_p, C.c_size_t]),
            "bgmg_destroy": (None, [_vp]),
            "bgmg_num_levels": (C.c_int, [_vp]),
            "bgmg_level_frozen_ok": (C.c_int, [_vp, C.c_int]),
            "bgmg_level_n": (C.c_int, [_vp, C.c_int]),
            "bgmg_level_nx": (C.c_int, [_vp, C.c_int]),
            "bgmg_cycle_flops_per_unknown": (C.c_int, [_vp, C.POINTER(_Cycle), _dp, C.c_char_p, C.c_size_t]),
            "bgmg_fine_rhs": (C.c_int, [_vp, _dp]),
            "bgmg_vcycle": (C.c_int, [_vp, C.POINTER(_Cycle), _dp, _dp, C.c_char_p, C.c_size_t]),
            "bgmg_solve": (C.c_int, [_vp, C.POINTER(_Cycle), _dp, C.POINTER(_MgOpts), C.POINTER(_Rep), _dp, _dp,
                                     C.c_char_p, C.c_size_t]),
            "bgmg_solve_device": (C.c_int, [_vp, C.POINTER(_Cycle), _vp, C.POINTER(_MgOpts), C.POINTER(_Rep), _vp,
                                            _dp, C.c_char_p, C.c_size_t]),
            "bgmg_stream": (_vp, [_vp]),
            "bgmg_restrict": (C.c_int, [_dp, C.c_int, _dp]),
            "bgmg_prolong": (C.c_int, [_dp, C.c_int, _dp]),
            "bgabp_problem_named": (_vp, [C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_char_p), _dp, C.c_char_p,
                                          C.c_size_t]),
            "bgabp_problem_poisson5": (_vp, [C.c_int, C.c_int]),
            "bgabp_problem_matrix_market": (_vp, [C.c_char_p, C.c_char_p, C.c_size_t]),
            "bgabp_problem_config": (_vp, [C.c_int, C.c_int, C.c_uint]),
            "bgabp_problem_config5_level": (_vp, [C.c_int, C.c_int, C.c_uint]),
            "bgabp_problem_varcoef2d_level": (_vp, [C.c_int, C.c_int, C.c_uint, C.c_double]),
            "bgabp_problem_varcoef2d_rule": (_vp, [C.c_int, C.c_int, C.c_uint, C.c_double, C.c_int]),
            "bgabp_problem_free": (None, [_vp]),
            "bgabp_problem_n": (C.c_int, [_vp]),
            "bgabp_problem_nnz": (C.c_longlong, [_vp]),
            "bgabp_problem_nx": (C.c_int, [_vp]),
            "bgabp_problem_row_offsets": (_ip, [_vp]),
            "bgabp_problem_col_indices": (_ip, [_vp]),
            "bgabp_problem_values": (_dp, [_vp]),
            "bgabp_problem_rhs": (_dp, [_vp]),
            "bgabp_problem_exact": (_dp, [_vp]),
            "bglin_create": (C.c_int, [C.c_int, _ip, _ip, _dp, C.c_int, C.c_int, C.POINTER(_vp), C.c_char_p,
                                       C.c_size_t]),
            "bglin_destroy": (None, [_vp]),
            "bglin_num_edges": (C.c_int, [_vp]),
            "bglin_sweep_flops": (C.c_double, [_vp]),
            "bglin_stream": (_vp, [_vp]),
            "bglin_reset_state": (C.c_int, [_vp]),
            "bglin_set_state": (C.c_int, [_vp, _dp, _dp]),
            "bglin_get_state": (C.c_int, [_vp, _dp, _dp]),
            "bglin_sweep": (C.c_int, [_vp, _dp, C.c_int, _dp, C.c_char_p, C.c_size_t]),
            "bglin_solve": (C.c_int, [_vp, _dp, C.POINTER(_LinOpts), C.POINTER(_Rep), _dp, _dp, C.c_char_p,
                                      C.c_size_t]),
            "bgabp_shard_set_range": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int]),
            "bgabp_shard_solve_begin": (C.c_int, [_vp, _vp, C.POINTER(_Opts), C.c_double]),
            "bgabp_shard_step_compute": (C.c_int, [_vp]),
            "bgabp_shard_reduce_buffer": (_vp, [_vp]),
            "bgabp_shard_step_decide": (C.c_int, [_vp]),
            "bgabp_shard_msg": (_vp, [_vp, C.c_int]),
            "bgabp_shard_x": (_vp, [_vp, C.c_int]),
            "bgabp_shard_pack": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _vp]),
            "bgabp_shard_unpack": (C.c_int, [_vp, C.c_int, _vp, C.c_int, C.c_int, C.c_int, C.c_int]),
            "bgabp_shard_state": (C.c_int, [_vp, _ip, _ip]),
            "bgabp_shard_peer_slots": (C.c_int, [_vp, C.POINTER(_vp)]),
            "bgabp_shard_set_peers": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(_vp), C.c_int, C.c_int,
                                                 C.POINTER(_vp), C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]),
            "bgabp_shard_p2p_compute": (C.c_int, [_vp]),
            "bgabp_shard_p2p_wait": (C.c_int, [_vp, _vp]),
            "bgabp_shard_p2p_decide": (C.c_int, [_vp, C.c_int]),
            "bgabp_shard_p2p_steps": (C.c_int, [C.POINTER(_vp), C.c_int, C.c_int, C.c_int]),
            "bgabp_shard_p2p_steps_ipc": (C.c_int, [_vp, C.c_int]),
            "bgabp_ipc_get": (C.c_int, [_vp, _vp]),
            "bgabp_ipc_open": (C.c_int, [_vp, C.POINTER(_vp)]),
            "bgabp_ipc_close": (C.c_int, [_vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _LIB = L
    return _LIB


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _raise(rc, msg):
    if rc == OK:
        return
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == ECUDA:
        raise RuntimeError("CUDA: " + msg)
    raise RuntimeError(msg)


# ---------------------------------------------------------------------------------------------
# value types (sparse.hpp, schedule.hpp, report.hpp, gabp.hpp)
# ---------------------------------------------------------------------------------------------
@dataclass
class SparseMatrix:
    """Canonical CSR (sparse.hpp:17-39): strictly increasing columns per row."""
    n: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    @property
    def nnz(self):
        return int(self.row_offsets[-1]) if len(self.row_offsets) else 0

    @staticmethod
    def of(A):
        if isinstance(A, SparseMatrix):
            return A
        return SparseMatrix(int(A.n), _i32(A.row_offsets), _i32(A.col_indices), _f64(A.values))


class ScheduleKind(enum.IntEnum):  # schedule.hpp:9-15 (+ how the order was built)
    ParallelFlood = 0
    SequentialLexicographic = 1
    RedBlack = 2
    FourColor = 3
    CustomOrder = 4
    RedBlackGreedy = 5
    FourColorGreedy = 6


@dataclass
class Schedule:
    kind: int = ScheduleKind.SequentialLexicographic
    nx: int = 0
    ny: int = 0
    order: np.ndarray | None = None

    @staticmethod
    def parallel_flood():
        return Schedule(ScheduleKind.ParallelFlood)

    @staticmethod
    def sequential(n=0):
        return Schedule(ScheduleKind.SequentialLexicographic)

    @staticmethod
    def custom(order):
        return Schedule(ScheduleKind.CustomOrder, order=_i32(order))

    @staticmethod
    def red_black_grid(nx, ny):
        return Schedule(ScheduleKind.RedBlack, nx, ny)

    @staticmethod
    def four_color_grid(nx, ny):
        return Schedule(ScheduleKind.FourColor, nx, ny)

    @staticmethod
    def red_black(A=None):
        return Schedule(ScheduleKind.RedBlackGreedy)

    @staticmethod
    def four_color(A=None):
        return Schedule(ScheduleKind.FourColorGreedy)

    def _c(self):
        s = _Sched(int(self.kind), int(self.nx), int(self.ny), None)
        if self.order is not None:
            self._keep = _i32(self.order)
            s.order = _i(self._keep)
        return C.byref(s), s


class SolveStatus(enum.IntEnum):  # report.hpp:10
    Converged = 0
    Diverged = 1
    MaxIter = 2


class StopCriterion(enum.IntEnum):  # gabp.hpp:37
    Residual = 0
    MessageDelta = 1


@dataclass
class GabpOptions:  # gabp.hpp:39-45
    tol: float = 2e-4
    max_iter: int = 20000
    stop: int = StopCriterion.Residual
    divergence_factor: float = 1e12

    def _c(self):
        return _Opts(self.tol, self.max_iter, int(self.stop), self.divergence_factor)


@dataclass
class SolveReport:  # report.hpp:21-28
    status: int = SolveStatus.MaxIter
    iterations: int = 0
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    flop_estimate: float = 0.0
    solution: np.ndarray = field(default_factory=lambda: np.zeros(0))
    detail: str = ""


@dataclass
class MessageState:  # gabp.hpp:31-35, CSR-position indexed
    lambda_tilde: np.ndarray
    m: np.ndarray


@dataclass
class FrozenLambda:  # gabp.hpp:49-54
    lambda_tilde: np.ndarray
    sigma: np.ndarray
    converged: bool = False
    iterations: int = 0


class Layout(enum.IntEnum):
    Auto = 0
    Dia = 1
    Csr = 2


# ---------------------------------------------------------------------------------------------
# GabpEngine (gabp.hpp:58-111)
# ---------------------------------------------------------------------------------------------
class GabpEngine:
    """Device-resident GaBP engine over one matrix; the handle owns the device message state."""

    def __init__(self, A, layout=Layout.Auto):
        L = lib()
        self.A = SparseMatrix.of(A)
        h = _vp()
        err = C.create_string_buffer(512)
        rc = L.bgabp_create(self.A.n, _i(self.A.row_offsets), _i(self.A.col_indices), _d(self.A.values),
                            int(layout), C.byref(h), err, 512)
        _raise(rc, err.value.decode())
        self._h = h
        info = _Info()
        L.bgabp_get_info(h, C.byref(info))
        self.info = {k: getattr(info, k) for k, _ in _Info._fields_}
        self._state_owner = None

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().bgabp_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def num_edges(self):
        return int(self.info["num_edges"])

    @property
    def layout(self):
        return Layout(self.info["layout"])

    def stream(self):
        return lib().bgabp_stream(self._h)

    def layout_digest(self) -> int:
        """FNV-1a digest of the device layout (diagnostic; see bgabp_layout_digest)."""
        out = C.c_ulonglong(0)
        _raise(lib().bgabp_layout_digest(self._h, C.byref(out)), "layout digest")
        return int(out.value)

    def make_state(self) -> MessageState:
        return MessageState(np.zeros(self.A.nnz), np.zeros(self.A.nnz))

    def sweep(self, b, sched: Schedule, state: MessageState, x: np.ndarray):
        """GabpEngine::sweep (gabp.cpp:42-47): updates `state` and `x` in place; returns (ok, err)."""
        L = lib()
        L.bgabp_set_state(self._h, _d(state.lambda_tilde), _d(state.m))
        ok, err = self.sweep_resident(b, sched, x)
        L.bgabp_get_state(self._h, _d(state.lambda_tilde), _d(state.m))
        return ok, err

    def sweep_resident(self, b, sched: Schedule, x: np.ndarray):
        """One sweep on the handle's device-resident state (no state transfer)."""
        if x.dtype != np.float64 or not x.flags.c_contiguous:
            raise ValueError("x must be a contiguous float64 array")
        err = C.create_string_buffer(512)
        sp, _ = sched._c()
        rc = lib().bgabp_sweep(self._h, _d(_f64(b)), sp, _d(x), err, 512)
        if rc == EPIVOT:
            return False, err.value.decode()
        _raise(rc, err.value.decode())
        return True, ""

    def set_state(self, state: MessageState):
        _raise(lib().bgabp_set_state(self._h, _d(_f64(state.lambda_tilde)), _d(_f64(state.m))), "set_state")

    def get_state(self) -> MessageState:
        st = self.make_state()
        _raise(lib().bgabp_get_state(self._h, _d(st.lambda_tilde), _d(st.m)), "get_state")
        return st

    def reset_state(self):
        _raise(lib().bgabp_reset_state(self._h), "reset_state")

    def node_precisions(self, state: MessageState | None = None):
        if state is not None:
            self.set_state(state)
        beta = np.zeros(self.A.n)
        _raise(lib().bgabp_node_precisions(self._h, _d(beta)), "node_precisions")
        return beta

    def sweep_flops(self):
        return lib().bgabp_sweep_flops(self._h)

    def set_damping(self, alpha: float):
        """Optional message damping of flood sweeps and solves (no reference counterpart):
        new <- (1 - alpha) new + alpha old per edge; 0 is the reference's update."""
        _raise(lib().bgabp_set_damping(self._h, float(alpha)), "gabp: damping must lie in [0, 1)")

    def solve(self, b, sched: Schedule, opt: GabpOptions = GabpOptions(), x_out=None) -> SolveReport:
        """GabpEngine::solve (gabp.cpp:174-219).  x_out: optional caller buffer (e.g. pinned) for x."""
        n = self.A.n
        x = np.zeros(n) if x_out is None else x_out
        hist = np.zeros(max(opt.max_iter, 0) + 2)
        rep = _Rep()
        det = C.create_string_buffer(512)
        sp, _ = sched._c()
        o = opt._c()
        rc = lib().bgabp_solve(self._h, _d(_f64(b)), sp, C.byref(o), C.byref(rep), _d(x), _d(hist), det, 512)
        _raise(rc, det.value.decode())
        d = det.value.decode()
        return SolveReport(SolveStatus(rep.status), rep.iterations, hist[: solve_history_len(rep, d)].copy(),
                           rep.flop_estimate, x, d)

    def residual_inf_norm(self, x, b):
        out = C.c_double(0)
        _raise(lib().bgabp_residual_inf_norm(self._h, _d(_f64(x)), _d(_f64(b)), C.byref(out)), "residual")
        return out.value

    def precompute_lambda(self, sched: Schedule, tol=1e-10, max_iter=500) -> FrozenLambda:
        lam = np.zeros(self.A.nnz)
        sig = np.zeros(self.A.n)
        cv, it = C.c_int(0), C.c_int(0)
        sp, _ = sched._c()
        rc = lib().bgabp_precompute_lambda(self._h, sp, tol, max_iter, _d(lam), _d(sig), C.byref(cv), C.byref(it))
        _raise(rc, "gabp: schedule order does not cover every node")
        return FrozenLambda(lam, sig, bool(cv.value), it.value)

    def _load_frozen(self, frozen: FrozenLambda):
        _raise(lib().bgabp_set_frozen(self._h, _d(_f64(frozen.lambda_tilde)), _d(_f64(frozen.sigma))), "frozen")

    def correction_sweeps(self, r, sched: Schedule, frozen: FrozenLambda, sweeps: int):
        self._load_frozen(frozen)
        e = np.zeros(self.A.n)
        sp, _ = sched._c()
        _raise(lib().bgabp_correction_sweeps(self._h, _d(_f64(r)), sp, sweeps, _d(e)),
               "gabp: schedule order does not cover every node")
        return e

    def error_correction_apply(self, b, x0, sweeps, sched: Schedule, frozen: FrozenLambda | None = None):
        if frozen is not None:
            self._load_frozen(frozen)
        x = np.zeros(self.A.n)
        err = C.create_string_buffer(512)
        sp, _ = sched._c()
        rc = lib().bgabp_error_correction_apply(self._h, _d(_f64(b)), _d(_f64(x0)), sweeps, sp,
                                                int(frozen is not None), _d(x), err, 512)
        _raise(rc, err.value.decode())
        return x

    def solve_error_correction(self, b, sched: Schedule, sweeps, frozen: FrozenLambda,
                               opt: GabpOptions = GabpOptions()) -> SolveReport:
        self._load_frozen(frozen)
        x = np.zeros(self.A.n)
        hist = np.zeros(max(opt.max_iter, 0) + 2)
        rep = _Rep()
        det = C.create_string_buffer(512)
        sp, _ = sched._c()
        o = opt._c()
        rc = lib().bgabp_solve_error_correction(self._h, _d(_f64(b)), sp, sweeps, C.byref(o), C.byref(rep), _d(x),
                                                _d(hist), det, 512)
        _raise(rc, det.value.decode())
        return SolveReport(SolveStatus(rep.status), rep.iterations, hist[: rep.iterations + 1].copy(),
                           rep.flop_estimate, x, det.value.decode())

    # ---- device-resident drivers (device pointers as ints, e.g. torch.Tensor.data_ptr()) ----
    def solve_device_begin(self, b_ptr, sched: Schedule, opt: GabpOptions):
        sp, _ = sched._c()
        o = opt._c()
        _raise(lib().bgabp_solve_device_begin(self._h, C.c_void_p(b_ptr), sp, C.byref(o)), "solve_device_begin")

    def solve_device_steps(self, nsteps):
        _raise(lib().bgabp_solve_device_steps(self._h, int(nsteps)), "solve_device_steps")

    def solve_device_steps_timed(self, nsteps):
        """Enqueue nsteps iterations with events around each hot kernel; returns its total ms."""
        ms = C.c_double(0)
        _raise(lib().bgabp_solve_device_steps_timed(self._h, int(nsteps), C.byref(ms)), "solve_device_steps_timed")
        return ms.value

    def solve_device_end(self, x_ptr=None, hist_ptr=None):
        rep = _Rep()
        det = C.create_string_buffer(512)
        rc = lib().bgabp_solve_device_end(self._h, C.byref(rep), C.c_void_p(x_ptr or 0), C.c_void_p(hist_ptr or 0),
                                          det, 512)
        _raise(rc, det.value.decode())
        return SolveStatus(rep.status), rep.iterations, rep.flop_estimate, det.value.decode()

    def flood_sweeps_device(self, b_ptr, nsweeps):
        _raise(lib().bgabp_flood_sweeps_device(self._h, C.c_void_p(b_ptr), int(nsweeps)), "flood_sweeps_device")


# ---------------------------------------------------------------------------------------------
# line GaBP: region GaBP over grid lines (region_gabp.hpp:41-94, region.cpp:208-221)
# ---------------------------------------------------------------------------------------------
class RegionSweepMode(enum.IntEnum):  # region_gabp.hpp:20-23
    Sequential = 0
    Flood = 1


@dataclass
class RegionSolveOptions:  # region_gabp.hpp:25-30
    tol: float = 2e-4
    max_iter: int = 10000
    mode: int = RegionSweepMode.Sequential
    divergence_factor: float = 1e12

    def _c(self):
        return _LinOpts(self.tol, self.max_iter, int(self.mode), self.divergence_factor)


class LineGabpEngine:
    """RegionGabpEngine(A, build_two_layer_region_graph(A, grid_line_regions(nx, ny))) on the device
    for a 5-point operator (x fastest).  Block messages are scalars: 2n edges in the reference's
    edge order (row edges by node, then column edges column by column)."""

    def __init__(self, A, nx, ny):
        L = lib()
        self.A = SparseMatrix.of(A)
        self.nx, self.ny = int(nx), int(ny)
        h = _vp()
        err = C.create_string_buffer(512)
        rc = L.bglin_create(self.A.n, _i(self.A.row_offsets), _i(self.A.col_indices), _d(self.A.values), self.nx,
                            self.ny, C.byref(h), err, 512)
        _raise(rc, err.value.decode())
        self._h = h

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().bglin_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @property
    def num_edges(self):
        return lib().bglin_num_edges(self._h)

    def sweep_flops(self):
        return lib().bglin_sweep_flops(self._h)

    def make_state(self):
        return np.zeros(self.num_edges), np.zeros(self.num_edges)

    def sweep(self, b, lam, m, x, mode=RegionSweepMode.Sequential):
        """RegionGabpEngine::sweep (region_gabp.cpp:145-157): state and x in place; (ok, err)."""
        L = lib()
        _raise(L.bglin_set_state(self._h, _d(lam), _d(m)), "set_state")
        err = C.create_string_buffer(512)
        rc = L.bglin_sweep(self._h, _d(_f64(b)), int(mode), _d(x), err, 512)
        if rc not in (OK, EPIVOT):
            _raise(rc, err.value.decode())
        _raise(L.bglin_get_state(self._h, _d(lam), _d(m)), "get_state")
        return rc == OK, err.value.decode()

    def solve(self, b, opt: RegionSolveOptions = RegionSolveOptions()) -> SolveReport:
        """RegionGabpEngine::solve (region_gabp.cpp:159-198)."""
        n = self.A.n
        x = np.zeros(n)
        hist = np.zeros(max(opt.max_iter, 0) + 2)
        rep = _Rep()
        det = C.create_string_buffer(512)
        o = opt._c()
        rc = lib().bglin_solve(self._h, _d(_f64(b)), C.byref(o), C.byref(rep), _d(x), _d(hist), det, 512)
        _raise(rc, det.value.decode())
        good = rep.iterations - (1 if rep.status == SolveStatus.Diverged and det.value
                                 and det.value != b"residual blowup" else 0)
        return SolveReport(SolveStatus(rep.status), rep.iterations, hist[:good + 1].copy(), rep.flop_estimate, x,
                           det.value.decode())


# ---------------------------------------------------------------------------------------------
# multigrid (multigrid.hpp:17-103)
# ---------------------------------------------------------------------------------------------
class MgSmoother(enum.IntEnum):
    GabpSequential = 0
    GabpRedBlack = 1
    GabpFourColor = 2
    GabpFlood = 3
    GabpLine = 4  # grid-line region GaBP (multigrid.cpp:96-100, 189-204), see LineGabpEngine
    Jacobi = 5
    GsLex = 6
    GsRedBlack = 7
    GsFourColor = 8


@dataclass
class CycleSpec:  # multigrid.hpp:33-40
    pre: int = 1
    post: int = 1
    smoother: int = MgSmoother.GsLex
    frozen: bool = False

    def _c(self):
        return _Cycle(self.pre, self.post, int(self.frozen))


@dataclass
class MgSolveOptions:  # multigrid.hpp:96-100
    tol: float = 2e-4
    max_cycles: int = 200
    divergence_factor: float = 1e6

    def _c(self):
        return _MgOpts(self.tol, self.max_cycles, self.divergence_factor)


class Hierarchy:
    """Hierarchy(problem, J1, J2, params, smoother) (multigrid.hpp:52-86) on the device."""

    def __init__(self, problem, J1, J2, params=None, smoother=MgSmoother.GsLex):
        L = lib()
        params = params or {}
        keys = (C.c_char_p * max(1, len(params)))(*[k.encode() for k in params])
        vals = _f64(list(params.values()) or [0.0])
        h = _vp()
        err = C.create_string_buffer(512)
        rc = L.bgmg_create_named(problem.encode(), J1, J2, len(params), keys, _d(vals), int(smoother), C.byref(h),
                                 err, 512)
        _raise(rc, err.value.decode())
        self._h = h
        self._smoother = smoother

    @classmethod
    def from_levels(cls, levels, nx, smoother):
        """Caller-supplied rediscretised levels, finest first (config 5)."""
        self = cls.__new__(cls)
        L = lib()
        levels = [SparseMatrix.of(A) for A in levels]
        k = len(levels)
        ns = _i32([A.n for A in levels])
        ros = (_ip * k)(*[_i(A.row_offsets) for A in levels])
        cis = (_ip * k)(*[_i(A.col_indices) for A in levels])
        vs = (_dp * k)(*[_d(A.values) for A in levels])
        nxa = _i32(nx)
        h = _vp()
        err = C.create_string_buffer(512)
        rc = L.bgmg_create(k, _i(ns), ros, cis, vs, _i(nxa), int(smoother), C.byref(h), err, 512)
        _raise(rc, err.value.decode())
        self._h = h
        self._smoother = smoother
        return self

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().bgmg_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def num_levels(self):
        return lib().bgmg_num_levels(self._h)

    def level_frozen_ok(self, k):
        return bool(lib().bgmg_level_frozen_ok(self._h, k))

    def level_n(self, k):
        return lib().bgmg_level_n(self._h, k)

    def level_nx(self, k):
        return lib().bgmg_level_nx(self._h, k)

    def cycle_flops_per_unknown(self, spec: CycleSpec) -> float:
        """multigrid.cpp:240-274 (analytic flop_table of the pre + post sweeps)."""
        out = C.c_double(0.0)
        err = C.create_string_buffer(256)
        c = spec._c()
        _raise(lib().bgmg_cycle_flops_per_unknown(self._h, C.byref(c), C.byref(out), err, 256), err.value.decode())
        return out.value

    def smoother(self):
        return self._smoother

    def fine_rhs(self):
        b = np.zeros(self.level_n(0))
        _raise(lib().bgmg_fine_rhs(self._h, _d(b)), "fine_rhs: hierarchy was not built from a named problem")
        return b

    def stream(self):
        return lib().bgmg_stream(self._h)

    def v_cycle(self, spec: CycleSpec, b, x: np.ndarray):
        """One V-cycle, x updated in place; RuntimeError on smoother breakdown (multigrid.cpp:234-238)."""
        err = C.create_string_buffer(512)
        c = spec._c()
        rc = lib().bgmg_vcycle(self._h, C.byref(c), _d(_f64(b)), _d(x), err, 512)
        _raise(rc, err.value.decode())


def mg_solve(hier: Hierarchy, spec: CycleSpec, b, opt: MgSolveOptions = MgSolveOptions()) -> SolveReport:
    """mg_solve (multigrid.cpp:276-318)."""
    n = hier.level_n(0)
    x = np.zeros(n)
    hist = np.zeros(opt.max_cycles + 2)
    rep = _Rep()
    det = C.create_string_buffer(512)
    c, o = spec._c(), opt._c()
    rc = lib().bgmg_solve(hier._h, C.byref(c), _d(_f64(b)), C.byref(o), C.byref(rep), _d(x), _d(hist), det, 512)
    _raise(rc, det.value.decode())
    d = det.value.decode()
    return SolveReport(SolveStatus(rep.status), rep.iterations, hist[: _mg_hist_len(rep, d)].copy(),
                       rep.flop_estimate, x, d)


def solve_history_len(rep, detail):
    """GabpEngine::solve's residual history: iterations + 1 entries, one fewer on a pivot stop
    (the failed sweep pushes no residual, gabp.cpp:193-199)."""
    pivot = rep.status == SolveStatus.Diverged and detail.startswith("zero pivot")
    return rep.iterations + (0 if pivot else 1)


def _mg_hist_len(rep, detail):
    """iterations + 1 residuals, one fewer when the last cycle broke down (multigrid.cpp:288-297)."""
    breakdown = rep.status == SolveStatus.Diverged and detail != "residual blowup"
    return rep.iterations + (0 if breakdown else 1)


def mg_solve_device(hier: Hierarchy, spec: CycleSpec, b_ptr, x_ptr, opt: MgSolveOptions = MgSolveOptions()):
    hist = np.zeros(opt.max_cycles + 2)
    rep = _Rep()
    det = C.create_string_buffer(512)
    c, o = spec._c(), opt._c()
    rc = lib().bgmg_solve_device(hier._h, C.byref(c), C.c_void_p(b_ptr), C.byref(o), C.byref(rep), C.c_void_p(x_ptr),
                                 _d(hist), det, 512)
    _raise(rc, det.value.decode())
    d = det.value.decode()
    return SolveReport(SolveStatus(rep.status), rep.iterations, hist[: _mg_hist_len(rep, d)].copy(),
                       rep.flop_estimate, np.zeros(0), d)


def mg_restrict(fine, mf):
    mc = (mf - 1) // 2
    out = np.zeros(mc * mc)
    _raise(lib().bgmg_restrict(_d(_f64(fine)), mf, _d(out)), "mg_restrict")
    return out


def mg_prolong(coarse, mc):
    mf = 2 * mc + 1
    out = np.zeros(mf * mf)
    _raise(lib().bgmg_prolong(_d(_f64(coarse)), mc, _d(out)), "mg_prolong")
    return out


# ---------------------------------------------------------------------------------------------
# problem assembly (problems.hpp; configs of BASELINE.json)
# ---------------------------------------------------------------------------------------------
@dataclass
class AssembledProblem:  # problems.hpp:16-22
    A: SparseMatrix
    b: np.ndarray
    exact: np.ndarray | None
    nx: int
    h: float = 0.0


def _take_problem(p, h=0.0) -> AssembledProblem:
    L = lib()
    try:
        n, nnz = L.bgabp_problem_n(p), L.bgabp_problem_nnz(p)
        ro = np.ctypeslib.as_array(L.bgabp_problem_row_offsets(p), (n + 1,)).copy()
        ci = np.ctypeslib.as_array(L.bgabp_problem_col_indices(p), (nnz,)).copy() if nnz else np.zeros(0, np.int32)
        v = np.ctypeslib.as_array(L.bgabp_problem_values(p), (nnz,)).copy() if nnz else np.zeros(0)
        rp, ep = L.bgabp_problem_rhs(p), L.bgabp_problem_exact(p)
        b = np.ctypeslib.as_array(rp, (n,)).copy() if rp else None
        ex = np.ctypeslib.as_array(ep, (n,)).copy() if ep else None
        return AssembledProblem(SparseMatrix(n, ro, ci, v), b, ex, L.bgabp_problem_nx(p), h)
    finally:
        L.bgabp_problem_free(p)


def assemble(name, J, params=None) -> AssembledProblem:
    """assemble(name, J, params) (problems.cpp:161-226)."""
    params = params or {}
    keys = (C.c_char_p * max(1, len(params)))(*[k.encode() for k in params])
    vals = _f64(list(params.values()) or [0.0])
    err = C.create_string_buffer(512)
    p = lib().bgabp_problem_named(name.encode(), J, len(params), keys, _d(vals), err, 512)
    if not p:
        raise ValueError(err.value.decode())
    return _take_problem(p, 1.0 / (1 << J))


def load_matrix_market(path) -> SparseMatrix:
    """load_matrix_market (sparse.cpp:123-180): canonical CSR, duplicates summed."""
    L = lib()
    err = C.create_string_buffer(512)
    p = L.bgabp_problem_matrix_market(str(path).encode(), err, 512)
    if not p:
        raise RuntimeError(err.value.decode())
    return _take_problem(p).A


def poisson5(nx, ny) -> SparseMatrix:
    return _take_problem(lib().bgabp_problem_poisson5(nx, ny)).A


def config_problem(config, size=0, seed=None) -> AssembledProblem:
    """BASELINE.json config (1-5) at its own size (size=0) or a reduced one, with its seed."""
    seed = {1: 0, 2: 1, 3: 2, 4: 3, 5: 4}[config] if seed is None else seed
    p = lib().bgabp_problem_config(config, size, seed)
    if not p:
        raise ValueError(f"config {config}: bad size {size}")
    return _take_problem(p)


def varcoef2d_rule_level(J_fine, k, rule, seed=4, sigma=2.0) -> AssembledProblem:
    """Config-5 family level with another coarse-K rule (0 = the generator's full-weighted log K,
    1 = full-weighted K, 2 = full-weighted 1/K, 3 = injection)."""
    p = lib().bgabp_problem_varcoef2d_rule(J_fine, k, seed, sigma, rule)
    if not p:
        raise ValueError(f"varcoef2d: bad level / rule ({J_fine}, {k}, {rule})")
    return _take_problem(p)


def config5_level(J_fine, k, seed=4, sigma=2.0) -> AssembledProblem:
    """Level k (0 = finest) of the config-5 hierarchy; sigma = std of log K (config 5: 2)."""
    p = lib().bgabp_problem_varcoef2d_level(J_fine, k, seed, sigma)
    if not p:
        raise ValueError("config 5 level out of range")
    return _take_problem(p)
