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

from .core import LogPlan, OtProblem
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
