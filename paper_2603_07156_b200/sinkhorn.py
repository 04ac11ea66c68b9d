"""Warm start by alternating log-domain dual sweeps, on the device.

Drop-in for ``warm_start`` of pkg/src/otibsn/sinkhorn.py:68-103 (called by
the outer loop before every inner solve, bregman_outer.py:106-109).  Each
sweep is two streaming passes of libotb: the zeta pass (row log-sum-exp,
fused with the column-marginal error of sinkhorn.py:61-65) and the gamma
pass (column log-sum-exp as online (max, sum) pairs).  The host reads one
scalar per sweep (the error).
"""

from __future__ import annotations

import numpy as np

from .core import LogPlan, OtProblem, host
from .semidual import DualState
from .session import session_for

DEFAULT_SWEEP_CAP = 100_000   # sinkhorn.py:21


def warm_start(logplan: LogPlan, problem: OtProblem, eta: float, warm_tol: float, gamma0=None, zeta0=None,
               max_sweeps: int = DEFAULT_SWEEP_CAP, generation: int = 0, *, session=None, gamma_buf=None,
               zeta_buf=None, comm=None):
    """sinkhorn.py:68-103 — returns (DualState(gamma recentred), zeta).

    ``zeta0`` is accepted for signature compatibility; like the reference,
    the first sweep overwrites zeta before it is read.  Raises
    WarmStartStalled when the cap is hit.
    """
    s = session if session is not None else session_for(problem, eta, comm)
    plan_t = s.plan(logplan)
    n = s.n
    if gamma_buf is None:
        gamma_buf = s._vec(np.zeros(n) if gamma0 is None else gamma0)
    elif gamma0 is not None and not (hasattr(gamma0, "data_ptr") and gamma0.data_ptr() == gamma_buf.data_ptr()):
        gamma_buf[:n].copy_(s._vec(gamma0)[:n])
    zeta_buf = s.new_vec(s.m_loc) if zeta_buf is None else zeta_buf
    sweeps, err = s.ops.warm_start(plan_t, gamma_buf, zeta_buf, warm_tol, max_sweeps)
    s._last_warm = (sweeps, err)
    if session is not None:
        return DualState(gamma_buf, generation=generation), zeta_buf
    device_in = gamma0 is not None and type(gamma0).__module__.startswith("torch") and gamma0.is_cuda
    if device_in:
        return DualState(gamma_buf[:n], generation=generation), zeta_buf[: s.m_loc]
    return DualState(gamma_buf[:n].cpu().numpy(), generation=generation), zeta_buf[: s.m_loc].cpu().numpy()


# ------------------------------------------- single updates (sinkhorn.py:26-58)
class TwoDualState:
    """sinkhorn.py:26-35 — column dual gamma and row dual zeta."""

    def __init__(self, gamma, zeta):
        self.gamma = np.asarray(host(gamma), dtype=np.float64)
        self.zeta = np.asarray(host(zeta), dtype=np.float64)


def _two_dual_tensors(s, state):
    g = s._vec(state.gamma)
    z = s._vec(state.zeta, s.m_loc)
    return g, z


def scaled_plan_log(logplan: LogPlan, state: TwoDualState, problem: OtProblem, eta: float) -> np.ndarray:
    """sinkhorn.py:41-43 — log X + (zeta_i + gamma_j - C_ij) / eta, one
    device pass (otb_scaled_plan).  Entries below LOG_FLOOR come back
    clamped to it (the device writes a LogPlan); NaN / +inf raise
    InvalidCost."""
    s = session_for(problem, eta)
    plan_t = s.plan(logplan)
    g, z = _two_dual_tensors(s, state)
    out = s.new_plan()
    s.ops.scaled_plan(plan_t, g, z, out)
    return out[:, : s.n].cpu().numpy()


def zeta_update(logplan: LogPlan, state: TwoDualState, problem: OtProblem, eta: float) -> TwoDualState:
    """sinkhorn.py:46-51 — zeta = eta (log a - LSE_j(log X + (gamma - C)/eta)),
    the row pass of otb_sinkhorn_zeta."""
    s = session_for(problem, eta)
    plan_t = s.plan(logplan)
    g, z = _two_dual_tensors(s, state)
    s.ops.sinkhorn_zeta(plan_t, g, z)
    return TwoDualState(state.gamma, z[: s.m_loc].cpu().numpy())


def gamma_update(logplan: LogPlan, state: TwoDualState, problem: OtProblem, eta: float) -> TwoDualState:
    """sinkhorn.py:54-58 — gamma = eta (log b - LSE_i(log X + (zeta - C)/eta)),
    the column pass of otb_sinkhorn_gamma."""
    s = session_for(problem, eta)
    plan_t = s.plan(logplan)
    g, z = _two_dual_tensors(s, state)
    s.ops.sinkhorn_gamma(plan_t, g, z)
    return TwoDualState(g[: s.n].cpu().numpy(), state.zeta)
