"""B200-native inner loop of the inexact Bregman sparse-Newton (IBSN)
optimal-transport solver — a drop-in for the hot path of the reference
package ``otibsn`` (arXiv 2603.07156).

Public API (same names and signatures as the reference):

    from paper_2603_07156_b200 import OtProblem, SolverConfig, ibsn_solve
    res = ibsn_solve(OtProblem(C, a, b), SolverConfig(eta=1e-2, kkt_tol=1e-6))

Solver modules load ``libotb.so`` (hand-written sm_100a CUDA behind a C
ABI, include/otb.h) on first use; there is no CPU fallback.  ``errors``,
``core``, ``trajectory`` and ``instances`` are pure Python.
"""

from __future__ import annotations

import importlib

from . import errors
from .core import (
    LOG_FLOOR,
    InnerScale,
    LogPlan,
    OtProblem,
    SolverConfig,
    initial_plan,
    normalize_cost,
    validate,
)

_LAZY = {
    "ibsn_solve": "bregman_outer",
    "eot_single_solve": "bregman_outer",
    "ibsink_solve": "bregman_outer",
    "OuterResult": "bregman_outer",
    "MuSchedule": "bregman_outer",
    "mu": "bregman_outer",
    "inner_solve": "inner_newton",
    "newton_step": "inner_newton",
    "plan_candidate_log": "inner_newton",
    "InnerReport": "inner_newton",
    "StopReason": "inner_newton",
    "NewtonStepRecord": "inner_newton",
    "DualState": "semidual",
    "RowSoftmaxCache": "semidual",
    "compute_p": "semidual",
    "semidual_value": "semidual",
    "semidual_gradient": "semidual",
    "sparsify_p": "sparsify",
    "SparseHessianOp": "sparsify",
    "SparseRowStochastic": "sparsify",
    "choose_anchor": "sparsify",
    "threshold_rho": "sparsify",
    "hessian_matvec_sparse": "sparsify",
    "cg_solve": "krylov",
    "round_log_plan": "feasibility",
    "round_to_feasible": "feasibility",
    "kkt_residual": "feasibility",
    "bregman_div": "feasibility",
    "c_transform": "feasibility",
    "gap": "feasibility",
    "FeasiblePlan": "feasibility",
    "KktReport": "feasibility",
    "hessian_matvec_exact": "semidual",
    "zeta_from_cache": "semidual",
    "TwoDualState": "sinkhorn",
    "scaled_plan_log": "sinkhorn",
    "zeta_update": "sinkhorn",
    "gamma_update": "sinkhorn",
    "LocalGroup": "distributed",
    "warm_start": "sinkhorn",
    "Trajectory": "trajectory",
    "TrajectoryRecord": "trajectory",
    "RowComm": "distributed",
}

__all__ = ["errors", "LOG_FLOOR", "InnerScale", "LogPlan", "OtProblem", "SolverConfig", "initial_plan",
           "normalize_cost", "validate", *_LAZY]


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    return getattr(importlib.import_module(f".{mod}", __name__), name)
