"""Rounding onto the transport polytope, Bregman divergence and KKT metrics
(K7-K9, K11) on the device.

The reference computes these on dense host matrices
(pkg/src/otibsn/feasibility.py); here they are fused into the three-pass
``recover_round`` pipeline of libotb, which works on log plans in HBM:

  pass A  candidate log plan (optional), X = exp(logX), row sums -> z,
          column sums of X z                                (44-60)
  pass B  F = (X z) y, row sums -> e_r, column sums -> e_c  (61-66)
  pass C  F^ = F + e_r e_c^T / ||e_r||_1, D_phi(F^, X), and with metrics
          <C, F^> and the KKT sums (c-transform, slack)      (67-122)

``round_log_plan`` is the entry point; ``round_to_feasible`` /
``kkt_residual`` keep the reference signatures for callers holding dense
matrices (the matrix is taken to the log domain first, so entries may
differ from the reference's by one ulp of exp(log x)).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .core import LogPlan, OtProblem, host
from .session import session_for


@dataclass(frozen=True)
class FeasiblePlan:
    """feasibility.py:19-30 — rounded plan; ``entries`` materialised lazily."""

    _session: object = field(repr=False)
    _plan_t: object = field(repr=False)
    _gamma_t: object = field(repr=False)
    bregman: float = 0.0
    objective: float = float("nan")
    delta_p: float = float("nan")
    delta_d: float = float("nan")
    delta_c: float = float("nan")
    delta_kkt: float = float("nan")
    sum_x: float = 0.0
    deficit: float = 0.0

    @property
    def entries(self) -> np.ndarray:
        s = self._session
        s.ops.recover_round(self._plan_t, self._gamma_t, None, recover=False, metrics=False)
        return s.ops.materialize_rounded().cpu().numpy()

    @property
    def shape(self):
        return (self._session.m_loc, self._session.n)


@dataclass(frozen=True)
class KktReport:
    """feasibility.py:33-41 (zeta_used is not materialised on the device path)."""

    delta_p: float
    delta_d: float
    delta_c: float
    delta_kkt: float
    zeta_used: object = None


def round_log_plan(logplan: LogPlan, problem: OtProblem, gamma=None, eta: float = 1.0,
                   metrics: bool = True) -> FeasiblePlan:
    """P_Omega(exp(logplan)) with D_phi(P_Omega(X), X) and, with metrics and
    a column dual ``gamma``, <C, X^> and the relative KKT residual."""
    s = session_for(problem, eta)
    plan_t = s.plan(logplan)
    g = s._vec(np.zeros(s.n) if gamma is None else (gamma if not hasattr(gamma, "gamma") else gamma.gamma))
    r = s.ops.recover_round(plan_t, g, None, recover=False, metrics=metrics)
    return FeasiblePlan(s, plan_t, g, r.bregman, r.objective, r.delta_p, r.delta_d, r.delta_c, r.delta_kkt,
                        r.sum_x, r.deficit)


def _log_of(x) -> LogPlan:
    x = np.asarray(host(x), dtype=np.float64)
    with np.errstate(divide="ignore"):
        return LogPlan(np.log(x))


def round_to_feasible(x, a, b) -> np.ndarray:
    """feasibility.py:44-69 signature; returns the dense rounded matrix."""
    x = np.asarray(host(x), dtype=np.float64)
    prob = OtProblem(np.zeros_like(x), a, b)
    return round_log_plan(_log_of(x), prob, metrics=False).entries


def kkt_residual(x, gamma, cost, a, b) -> KktReport:
    """feasibility.py:93-122 for a matrix that is already feasible: the
    device pipeline rounds first, which leaves a feasible x unchanged up to
    rounding (SPEC: 'An input that is already feasible passes through')."""
    prob = OtProblem(cost, a, b)
    f = round_log_plan(_log_of(x), prob, gamma=np.asarray(host(gamma), dtype=np.float64), metrics=True)
    return KktReport(f.delta_p, f.delta_d, f.delta_c, f.delta_kkt)
