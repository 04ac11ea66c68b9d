"""Outer inexact Bregman proximal-point loop (IBSN) driving the device path.

Drop-in for ``ibsn_solve`` of pkg/src/otibsn/bregman_outer.py:62-159 (same
signature, same trajectory, same stopping rules).  All iterates stay in
HBM: two padded log-plan buffers (the current X^k and the candidate
X^{k+1}, swapped on acceptance — the "in place" recovery of the north
star), two dual buffers for gamma, one for zeta.  Per outer iteration the
host reads scalars only: warm-start error per sweep, Newton-step scalars,
the inexact-test divergence and the metrics of the accepted candidate.

Superset of the reference result: ``OuterResult`` also carries the final
duals ``gamma`` and ``zeta`` (the reference computes but does not return
them, bregman_outer.py:123-126) and solve counters.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from .core import InnerScale, LogPlan, OtProblem, SolverConfig, _is_torch, validate
from .errors import NumericalFailure
from .inner_newton import NewtonStepRecord, inner_solve
from .semidual import DualState
from .session import session_for
from .sinkhorn import warm_start
from .trajectory import Trajectory, TrajectoryRecord


@dataclass(frozen=True)
class MuSchedule:
    """bregman_outer.py:26-31."""

    mu0: float = 1e-4
    floor: float = 1e-11


def mu(schedule: MuSchedule, k: int) -> float:
    """bregman_outer.py:34-36."""
    return max(schedule.mu0 / (k + 1) ** 2, schedule.floor)


@dataclass
class OuterResult:
    """bregman_outer.py:39-48 plus duals and counters.

    ``rounded_plan`` is produced on first access (one device pass + D2H),
    because at the large configurations it is tens of GB.
    """

    final_logplan: LogPlan
    objective: float = 0.0
    kkt: float = 0.0
    outer_iters: int = 0
    trajectory: Trajectory = field(default_factory=Trajectory)
    gamma: object = None
    zeta: object = None
    newton_iters: int = 0
    cg_iters: int = 0
    warm_sweeps: int = 0
    _session: object = field(default=None, repr=False)
    _gamma_t: object = field(default=None, repr=False)
    _rounded: object = field(default=None, repr=False)

    @property
    def rounded_plan(self) -> np.ndarray:
        if self._rounded is None:
            s = self._session
            plan_t = s.plan(self.final_logplan)
            s.ops.recover_round(plan_t, self._gamma_t, None, recover=False, metrics=False)
            self._rounded = s.ops.materialize_rounded().cpu().numpy()
        return self._rounded


def ibsn_solve(
    problem: OtProblem,
    config: SolverConfig,
    optimal_value: float | None = None,
    observer: Callable[[NewtonStepRecord], None] | None = None,
    on_outer: Callable[[int, LogPlan, np.ndarray], None] | None = None,
    clock: Callable[[], float] | None = None,
    deadline_seconds: float | None = None,
    *,
    comm=None,
) -> OuterResult:
    """bregman_outer.py:62-159 — proximal outer loop with sparsified Newton
    inner solves, entirely on the GPU(s).  ``comm`` (distributed.RowComm)
    shards the rows of C and X over the ranks of one node."""
    validate(problem)
    now = clock if clock is not None else time.perf_counter
    eta = config.eta
    schedule = MuSchedule(config.mu0, config.mu_floor)
    s = session_for(problem, eta, comm)
    n = s.n

    cur, spare = s.new_plan(), s.new_plan()
    s.ops.init_plan(cur)                                   # bregman_outer.py:91-93
    g0, g1 = s.new_vec(), s.new_vec()                      # gamma = 0
    zeta = s.new_vec(s.m_loc)                              # zeta = 0

    traj = Trajectory()
    t0 = now()
    inner_total = cg_total = sweeps_total = 0
    outer_iters = 0
    kkt_value = math.inf
    objective = math.nan
    for k in range(config.max_outer):
        mu_k = mu(schedule, k)
        logplan = LogPlan.from_padded(cur, n)
        warm_start(logplan, problem, eta, config.warm_tol, session=s, gamma_buf=g0, zeta_buf=zeta, generation=k)
        sweeps_total += s._last_warm[0]

        inner_observer = observer
        if config.log_inner_kkt:
            inner_observer = _chain_inner_logger(observer, traj, s, cur, now, t0,
                                                 lambda: (inner_total, cg_total), optimal_value)

        gstate, cand, report = inner_solve(logplan, DualState(g0, generation=k), problem, config, mu_k, k,
                                           observer=inner_observer, session=s, out_plan=spare, gamma_bufs=(g0, g1))
        if gstate.gamma.data_ptr() != g0.data_ptr():
            g0, g1 = g1, g0
        # zeta carried to the next subproblem (bregman_outer.py:123-126): the
        # accepted eval's row log-normalisers, eta (log a - lse).
        s.ops.zeta_from_lse(zeta)
        cur, spare = spare, cur
        outer_iters = k + 1
        if on_outer is not None:
            on_outer(k, LogPlan.from_padded(cur.clone(), n), g0[:n].cpu().numpy())

        inner_total += report.newton_iters
        cg_total += report.cg_iters_total
        objective, kkt_value = report.objective, report.kkt   # _metrics, bregman_outer.py:51-59
        if not math.isfinite(objective):
            raise NumericalFailure(f"non-finite objective {objective!r}")
        traj.record(TrajectoryRecord(
            outer_k=k, inner_total=inner_total, cg_total=cg_total, wall_seconds=now() - t0,
            objective=objective, kkt=kkt_value, grad_norm=report.final_grad_norm,
            gap=None if optimal_value is None else abs(objective - optimal_value)))
        if kkt_value < config.kkt_tol:
            break
        if deadline_seconds is not None and now() - t0 > deadline_seconds:
            break

    device_out = _is_torch(problem.cost)
    gamma_out = g0[:n] if device_out else g0[:n].cpu().numpy()
    zeta_out = zeta[: s.m_loc] if device_out else zeta[: s.m_loc].cpu().numpy()
    return OuterResult(final_logplan=LogPlan.from_padded(cur, n), objective=objective, kkt=kkt_value,
                       outer_iters=outer_iters, trajectory=traj, gamma=gamma_out, zeta=zeta_out,
                       newton_iters=inner_total, cg_iters=cg_total, warm_sweeps=sweeps_total,
                       _session=s, _gamma_t=g0)


def ibsink_solve(
    problem: OtProblem,
    config: SolverConfig,
    optimal_value: float | None = None,
    on_outer: Callable[[int, LogPlan, np.ndarray], None] | None = None,
    clock: Callable[[], float] | None = None,
    deadline_seconds: float | None = None,
    *,
    comm=None,
) -> OuterResult:
    """bregman_outer.py:191-281 — the same outer loop with alternating dual
    sweeps as the inner solver.  Per sweep: zeta update fused with the
    column-marginal error (the pre-check), the scaled plan and its rounding
    / Bregman test when the error is below mu_k, else the gamma update.
    Three device buffers rotate: the reference plan, the scaled candidate,
    and a scratch plan."""
    validate(problem)
    now = clock if clock is not None else time.perf_counter
    eta = config.eta
    schedule = MuSchedule(config.mu0, config.mu_floor)
    s = session_for(problem, eta, comm)
    m, n = s.m, s.n
    scale = float(min(m, n)) if config.inner_scale is InnerScale.MIN_DIM else 1.0
    cur, cand_t, spare = s.new_plan(), s.new_plan(), s.new_plan()
    s.ops.init_plan(cur)                                   # bregman_outer.py:210-212
    gamma = s.new_vec()
    zeta = s.new_vec(s.m_loc)
    traj = Trajectory()
    t0 = now()
    sweep_total = 0
    outer_iters = 0
    kkt_value = math.inf
    objective = math.nan
    err = math.inf
    for k in range(config.max_outer):
        mu_k = mu(schedule, k)
        accepted = False
        sweeps_this = 0
        for _ in range(config.max_inner):
            err = s.ops.sinkhorn_zeta(cur, gamma, zeta)    # zeta_update + column error
            sweeps_this += 1
            if err < mu_k:
                s.ops.scaled_plan(cur, gamma, zeta, cand_t)
                res = s.ops.recover_round(cand_t, gamma, None, recover=False, metrics=False)
                if res.bregman <= scale * mu_k:
                    accepted = True
                    break
            s.ops.sinkhorn_gamma(cur, gamma, zeta)
        if not accepted:
            # sweep cap reached; accept the latest row-exact scaled plan
            err = s.ops.sinkhorn_zeta(cur, gamma, zeta)
            sweeps_this += 1
            s.ops.scaled_plan(cur, gamma, zeta, cand_t)
        cur, cand_t = cand_t, cur
        outer_iters = k + 1
        sweep_total += sweeps_this
        if on_outer is not None:
            on_outer(k, LogPlan.from_padded(cur.clone(), n), gamma[:n].cpu().numpy())
        res = s.ops.recover_round(cur, gamma, None, recover=False, metrics=True)   # _metrics
        objective, kkt_value = float(res.objective), float(res.delta_kkt)
        if not math.isfinite(objective):
            raise NumericalFailure(f"non-finite objective {objective!r}")
        traj.record(TrajectoryRecord(
            outer_k=k, inner_total=sweep_total, cg_total=0, wall_seconds=now() - t0, objective=objective,
            kkt=kkt_value, grad_norm=err, gap=None if optimal_value is None else abs(objective - optimal_value)))
        if kkt_value < config.kkt_tol:
            break
        if deadline_seconds is not None and now() - t0 > deadline_seconds:
            break
    device_out = _is_torch(problem.cost)
    gamma_out = gamma[:n] if device_out else gamma[:n].cpu().numpy()
    zeta_out = zeta[: s.m_loc] if device_out else zeta[: s.m_loc].cpu().numpy()
    return OuterResult(final_logplan=LogPlan.from_padded(cur, n), objective=objective, kkt=kkt_value,
                       outer_iters=outer_iters, trajectory=traj, gamma=gamma_out, zeta=zeta_out,
                       warm_sweeps=sweep_total, _session=s, _gamma_t=gamma)


def eot_single_solve(
    problem: OtProblem,
    config: SolverConfig,
    clock: Callable[[], float] | None = None,
    *,
    comm=None,
) -> OuterResult:
    """bregman_outer.py:284-327 — one entropic (EOT) subproblem: the
    reference log plan is fixed at 0 (the all-ones plan), so the subproblem
    is entropic regularisation of the original cost; warm start, then the
    Newton phase to the gradient-norm target ``config.kkt_tol`` (pre-check
    off), then the metrics of the candidate.  Same kernels as ibsn_solve."""
    validate(problem)
    now = clock if clock is not None else time.perf_counter
    eta = config.eta
    s = session_for(problem, eta, comm)
    n = s.n
    cur, spare = s.new_plan(), s.new_plan()
    cur.zero_()                                            # LogPlan(np.zeros((m, n)))
    g0, g1 = s.new_vec(), s.new_vec()
    zeta = s.new_vec(s.m_loc)
    t0 = now()
    logplan = LogPlan.from_padded(cur, n)
    warm_start(logplan, problem, eta, config.warm_tol, session=s, gamma_buf=g0, zeta_buf=zeta, generation=0)
    gstate, cand, report = inner_solve(logplan, DualState(g0), problem, config, mu_k=0.0, outer_k=0,
                                       grad_target=config.kkt_tol, session=s, out_plan=spare, gamma_bufs=(g0, g1))
    if gstate.gamma.data_ptr() != g0.data_ptr():
        g0, g1 = g1, g0
    objective, kkt_value = report.objective, report.kkt    # _metrics(candidate, gamma)
    if not math.isfinite(objective):
        raise NumericalFailure(f"non-finite objective {objective!r}")
    traj = Trajectory()
    traj.record(TrajectoryRecord(
        outer_k=0, inner_total=report.newton_iters, cg_total=report.cg_iters_total, wall_seconds=now() - t0,
        objective=objective, kkt=kkt_value, grad_norm=report.final_grad_norm))
    device_out = _is_torch(problem.cost)
    gamma_out = g0[:n] if device_out else g0[:n].cpu().numpy()
    return OuterResult(final_logplan=LogPlan.from_padded(spare, n), objective=objective, kkt=kkt_value,
                       outer_iters=1, trajectory=traj, gamma=gamma_out, zeta=None,
                       newton_iters=report.newton_iters, cg_iters=report.cg_iters_total,
                       warm_sweeps=s._last_warm[0], _session=s, _gamma_t=g0)


def _chain_inner_logger(observer, traj, s, plan_t, now, t0, totals, optimal_value):
    """bregman_outer.py:162-188 — one trajectory row per inner step: the
    candidate of the step's dual on the current reference plan, rounded,
    with its objective and KKT residual (recover_round with metrics)."""
    cg_seen = 0
    scratch = s.new_plan()

    def logger(rec: NewtonStepRecord) -> None:
        nonlocal cg_seen
        if observer is not None:
            observer(rec)
        cg_seen += rec.cg_iters
        g = s._vec(rec.gamma)
        s.ops.eval(plan_t, g)
        res = s.ops.recover_round(plan_t, g, scratch, recover=True, metrics=True)
        inner_base, cg_base = totals()
        traj.record(TrajectoryRecord(
            outer_k=rec.outer_k, inner_total=inner_base + rec.inner_v, cg_total=cg_base + cg_seen,
            wall_seconds=now() - t0, objective=res.objective, kkt=res.delta_kkt, grad_norm=rec.grad_norm,
            gap=None if optimal_value is None else abs(res.objective - optimal_value)))

    return logger
