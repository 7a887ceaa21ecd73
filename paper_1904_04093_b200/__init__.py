"""B200 (sm_100a) GaBP hot path of arXiv 1904.04093: synchronous / colour-synchronous Gaussian
belief propagation sweeps, the residual check, and GaBP as a multigrid smoother.

The product is the C-ABI library `libgabp_b200.so` (include/gabp_b200.h) built from csrc/; this
package is its Python host mirror of the reference's proj/core API (see gabp.py).
"""
from .gabp import (AssembledProblem, CycleSpec, FrozenLambda, GabpEngine, GabpOptions, Hierarchy, Layout,  # noqa: F401
                   LineGabpEngine, MessageState, RegionSolveOptions, RegionSweepMode, MgSmoother, MgSolveOptions, Schedule, ScheduleKind, SolveReport, SolveStatus,
                   SparseMatrix, StopCriterion, assemble, config5_level, varcoef2d_rule_level, config_problem, lib, load_matrix_market, mg_prolong,
                   mg_restrict, mg_solve, mg_solve_device, poisson5)

__all__ = [n for n in dir() if not n.startswith("_")]
