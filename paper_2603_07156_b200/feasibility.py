"""Rounding onto the transport polytope, Bregman divergence and KKT metrics
on the device (drop-in for pkg/src/otibsn/feasibility.py).

Two paths:

* the solver's path works on LOG plans in HBM: ``round_log_plan`` runs the
  fused three-pass ``recover_round`` pipeline of libotb (K7-K9, K11):

    pass A  candidate log plan (optional), X = exp(logX), row sums -> z,
            column sums of X z                                (44-60)
    pass B  F = (X z) y, row sums -> e_r, column sums -> e_c  (61-66)
    pass C  F^ = F + e_r e_c^T / ||e_r||_1, D_phi(F^, X), and with metrics
            <C, F^> and the KKT sums (c-transform, slack)      (67-122)

* the reference's kernel-level functions keep their signatures for callers
  holding a dense LINEAR matrix: ``round_to_feasible`` (returns a
  ``FeasiblePlan``), ``bregman_div``, ``c_transform``, ``kkt_residual`` (on
  x AS GIVEN, including the ||min(x, 0)|| term and ``zeta_used``) and
  ``gap`` run the dense kernels of csrc/dense_api.cuh (otb_round_dense,
  otb_bregman_dense, otb_kkt_dense): numpy's elementwise arithmetic, sums in
  a fixed device order.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib
from .core import LogPlan, OtProblem, _is_torch, host
from .session import session_for


class FeasiblePlan:
    """feasibility.py:19-30 — a nonnegative matrix with exact marginals.

    ``FeasiblePlan(entries)`` as in the reference.  Plans rounded by the
    solver on the device are materialised on first access of ``entries``
    and carry the fused pipeline's scalars (bregman, objective, KKT parts).
    """

    def __init__(self, entries=None, *, _session=None, _plan_t=None, _gamma_t=None, bregman: float = 0.0,
                 objective: float = math.nan, delta_p: float = math.nan, delta_d: float = math.nan,
                 delta_c: float = math.nan, delta_kkt: float = math.nan, sum_x: float = 0.0, deficit: float = 0.0):
        self._entries = None if entries is None else np.asarray(host(entries), dtype=np.float64)
        self._session, self._plan_t, self._gamma_t = _session, _plan_t, _gamma_t
        self.bregman, self.objective = bregman, objective
        self.delta_p, self.delta_d, self.delta_c, self.delta_kkt = delta_p, delta_d, delta_c, delta_kkt
        self.sum_x, self.deficit = sum_x, deficit

    @property
    def entries(self) -> np.ndarray:
        if self._entries is None:
            s = self._session
            s.ops.recover_round(self._plan_t, self._gamma_t, None, recover=False, metrics=False)
            self._entries = s.ops.materialize_rounded().cpu().numpy()
        return self._entries

    @property
    def shape(self) -> tuple[int, int]:
        if self._entries is not None:
            return self._entries.shape
        return (self._session.m_loc, self._session.n)

    def __repr__(self) -> str:
        return f"FeasiblePlan(shape={self.shape})"


class KktReport:
    """feasibility.py:33-41."""

    def __init__(self, delta_p: float, delta_d: float, delta_c: float, delta_kkt: float, zeta_used=None):
        self.delta_p, self.delta_d, self.delta_c, self.delta_kkt = delta_p, delta_d, delta_c, delta_kkt
        self.zeta_used = zeta_used

    def __repr__(self) -> str:
        return (f"KktReport(delta_p={self.delta_p!r}, delta_d={self.delta_d!r}, delta_c={self.delta_c!r}, "
                f"delta_kkt={self.delta_kkt!r})")


def round_log_plan(logplan: LogPlan, problem: OtProblem, gamma=None, eta: float = 1.0,
                   metrics: bool = True) -> FeasiblePlan:
    """P_Omega(exp(logplan)) with D_phi(P_Omega(X), X) and, with metrics and
    a column dual ``gamma``, <C, X^> and the relative KKT residual."""
    s = session_for(problem, eta)
    plan_t = s.plan(logplan)
    g = s._vec(np.zeros(s.n) if gamma is None else (gamma if not hasattr(gamma, "gamma") else gamma.gamma))
    r = s.ops.recover_round(plan_t, g, None, recover=False, metrics=metrics)
    return FeasiblePlan(None, _session=s, _plan_t=plan_t, _gamma_t=g, bregman=r.bregman, objective=r.objective,
                        delta_p=r.delta_p, delta_d=r.delta_d, delta_c=r.delta_c, delta_kkt=r.delta_kkt,
                        sum_x=r.sum_x, deficit=r.deficit)


# ------------------------------------------------------- dense drop-ins
def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2603_07156_b200 needs a CUDA device (sm_100a); there is no CPU path")
    return torch


def _dev(x, torch):
    """Contiguous float64 tensor of x on the current CUDA device."""
    dev = torch.device("cuda", torch.cuda.current_device())
    if _is_torch(x):
        return x.detach().to(device=dev, dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).to(dev)


def _stream(torch) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _matrix(x):
    x2 = x if _is_torch(x) else np.asarray(x, dtype=np.float64)
    if x2.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    return x2


def round_to_feasible(x, a, b) -> FeasiblePlan:
    """feasibility.py:44-69 — capped row scaling, capped column scaling and
    the rank-one correction, on the device (otb_round_dense).  Returns a
    ``FeasiblePlan`` like the reference."""
    torch = _torch()
    x = _matrix(x)
    m, n = x.shape
    xd, ad, bd = _dev(x, torch), _dev(a, torch), _dev(b, torch)
    out = torch.empty((m, n), dtype=torch.float64, device=xd.device)
    deficit = C.c_double()
    _lib.check(_lib.lib.otb_round_dense(xd.data_ptr(), m, n, n, ad.data_ptr(), bd.data_ptr(), out.data_ptr(), n,
                                        C.byref(deficit), _stream(torch)))
    plan = FeasiblePlan(out.cpu().numpy())
    plan.deficit = float(deficit.value)
    return plan


def bregman_div(x, logy: LogPlan) -> float:
    """feasibility.py:72-85 — sum_{x>0} x (log x - log y) - sum x + sum y,
    with log y read from the stored (floored) log entries."""
    torch = _torch()
    x = _matrix(x.entries if isinstance(x, FeasiblePlan) else x)
    m, n = x.shape
    ly = logy.log_entries if isinstance(logy, LogPlan) else logy
    xd, ld = _dev(x, torch), _dev(ly, torch)
    if tuple(ld.shape) != (m, n):
        raise ValueError("x and log y shapes differ")
    out = C.c_double()
    _lib.check(_lib.lib.otb_bregman_dense(xd.data_ptr(), n, ld.data_ptr(), n, m, n, C.byref(out), _stream(torch)))
    return float(out.value)


def _kkt_sums(x, gamma, cost, a, b):
    torch = _torch()
    x = _matrix(x)
    m, n = x.shape
    xd, cd, gd, ad, bd = (_dev(v, torch) for v in (x, cost, gamma, a, b))
    zeta = torch.empty(m, dtype=torch.float64, device=xd.device)
    sums = (C.c_double * 8)()
    _lib.check(_lib.lib.otb_kkt_dense(xd.data_ptr(), n, cd.data_ptr(), n, gd.data_ptr(), ad.data_ptr(), bd.data_ptr(),
                                      m, n, zeta.data_ptr(), sums, _stream(torch)))
    return list(sums), zeta


def c_transform(gamma, cost) -> np.ndarray:
    """feasibility.py:88-90 — row minima of C - gamma."""
    cost = _matrix(cost)
    _, zeta = _kkt_sums(np.zeros(cost.shape) if not _is_torch(cost) else cost * 0, gamma, cost,
                        np.zeros(cost.shape[0]), np.zeros(cost.shape[1]))
    return zeta.cpu().numpy()


def kkt_residual(x, gamma, cost, a, b) -> KktReport:
    """feasibility.py:93-122 — the relative KKT residual of x AS GIVEN (no
    rounding): primal residuals of its marginals and of min(x, 0), the dual
    residual of the c-transform slack and the complementarity <x, slack>."""
    sums, zeta = _kkt_sums(x, gamma, cost, a, b)
    row_sq, col_sq, neg_sq, x_sq, dslack_sq, comp, _, _ = sums
    an = float(np.linalg.norm(host(a)))
    bn = float(np.linalg.norm(host(b)))
    cn = float(np.linalg.norm(host(cost)))
    cost_scale = 1.0 + cn
    delta_p = max(math.sqrt(row_sq) / (1.0 + an), math.sqrt(col_sq) / (1.0 + bn),
                  math.sqrt(neg_sq) / (1.0 + math.sqrt(x_sq)))
    delta_d = math.sqrt(dslack_sq) / cost_scale
    delta_c = abs(comp) / cost_scale
    return KktReport(delta_p, delta_d, delta_c, max(delta_p, delta_d, delta_c), zeta.cpu().numpy())


def gap(x_rounded: FeasiblePlan, cost, optimal_value: float) -> float:
    """feasibility.py:125-127 — |<C, X^> - optimal_value|."""
    x = x_rounded.entries if isinstance(x_rounded, FeasiblePlan) else x_rounded
    x = _matrix(x)
    sums, _ = _kkt_sums(x, np.zeros(x.shape[1]), cost, np.zeros(x.shape[0]), np.zeros(x.shape[1]))
    return abs(sums[6] - optimal_value)
