"""Sparsified Newton inner loop (Algorithm 2 inner iterations) on the device.

Drop-in for pkg/src/otibsn/inner_newton.py.  One Newton iteration is one
``otb_newton_step`` call into libotb (sparsify -> device CG -> slope ->
Armijo with the fused eval kernel); the host sees only scalars.  When the
pre-check ``||g|| < mu_k`` passes, ``otb_recover_round`` writes the
candidate log plan into a spare HBM buffer and returns D_phi(P_Omega(X), X)
together with the objective and KKT residual of the rounded candidate, which
the outer loop reuses instead of rounding the accepted plan again
(bregman_outer.py:134 re-rounds the same candidate the test rounded).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from .core import InnerScale, LogPlan, OtProblem, SolverConfig
from .semidual import DualState
from .session import session_for

LINE_SEARCH_CAP = 200        # inner_newton.py:35
GRAD_HARD_FLOOR = 1e-15      # inner_newton.py:39


class StopReason(enum.Enum):
    """inner_newton.py:42-45."""

    INEXACT_CRITERION = "inexact_criterion"
    GRAD_FLOOR = "grad_floor"
    MAX_INNER = "max_inner"


@dataclass(frozen=True)
class InnerReport:
    """inner_newton.py:48-56, plus the metrics of the returned candidate
    (objective / kkt of its rounding against the returned dual) and the
    per-step device counters (nnz of P_rho, rho)."""

    newton_iters: int
    cg_iters_total: int
    final_grad_norm: float
    stop_reason: StopReason
    step_sizes: list[float] = field(default_factory=list)
    objective: float = float("nan")
    kkt: float = float("nan")
    bregman: float = float("nan")
    nnz: list[int] = field(default_factory=list)
    cg_iters: list[int] = field(default_factory=list)
    values: list[float] = field(default_factory=list)
    tests: list[tuple] = field(default_factory=list)   # (inner_v, grad_norm, D_phi) per inexact test


@dataclass(frozen=True)
class NewtonStepRecord:
    """inner_newton.py:59-71 — observer payload after each accepted step."""

    outer_k: int
    inner_v: int
    gamma: np.ndarray = field(repr=False)
    grad_norm: float = 0.0
    step: float = 0.0
    cg_iters: int = 0
    value_before: float = 0.0
    value_after: float = 0.0
    slope: float = 0.0


def newton_step(logplan: LogPlan, gamma: DualState, problem: OtProblem, eta: float, sigma: float = 1e-4,
                beta: float = 0.8, cg_rel_tol: float = 1e-10, cg_max_iters: int | None = None):
    """inner_newton.py:125-148 — returns (new DualState, step, cg_iters)."""
    s = session_for(problem, eta)
    plan_t = s.plan(logplan)
    g_in = s._vec(gamma.gamma)
    value, gnorm = s.ops.eval(plan_t, g_in)
    if gnorm == 0.0:
        return gamma, 0.0, 0
    g_out = s.new_vec()
    r = s.ops.newton_step(plan_t, g_in, g_out, sigma, beta, cg_rel_tol, cg_max_iters)
    out = g_out[: s.n]
    new = out if _is_device(gamma.gamma) else out.cpu().numpy()
    return DualState(new, generation=gamma.generation), float(r.t), int(r.cg_iters)


def _is_device(x) -> bool:
    return type(x).__module__.startswith("torch") and x.is_cuda


def plan_candidate_log(logplan: LogPlan, cache, gamma: DualState, problem: OtProblem, eta: float) -> LogPlan:
    """inner_newton.py:151-167 — log(diag(a) P) on the device (uses the lse
    of ``cache``, which must have been computed at ``gamma``)."""
    s = cache.session
    s.ops.eval(cache.plan_t, cache.gamma_t)
    out = s.new_plan()
    s.ops.recover_round(cache.plan_t, cache.gamma_t, out, recover=True, metrics=False)
    return LogPlan.from_padded(out, s.n)


def inner_solve(logplan: LogPlan, gamma0: DualState, problem: OtProblem, config: SolverConfig, mu_k: float,
                outer_k: int, grad_target: float | None = None, recenter_every: int = 0,
                observer: Callable[[NewtonStepRecord], None] | None = None, *, session=None, out_plan=None,
                gamma_bufs=None, comm=None):
    """inner_newton.py:170-258 — Newton steps until the inexact test passes.

    Returns (DualState, candidate LogPlan, InnerReport).  The keyword-only
    arguments let ``ibsn_solve`` reuse its session and HBM buffers; callers
    of the reference API never pass them.
    """
    s = session if session is not None else session_for(problem, config.eta, comm)
    s.set_precond(getattr(config, "cg_preconditioner", None))
    m, n = s.m, s.n
    eta = config.eta
    scale = float(min(m, n)) if config.inner_scale is InnerScale.MIN_DIM else 1.0
    floor = GRAD_HARD_FLOOR if grad_target is None else max(grad_target, GRAD_HARD_FLOOR)
    plan_t = s.plan(logplan)
    native = observer is None and not recenter_every and config.max_inner >= 1
    g_src = None   # a device dual copied into g_cur by the first native call
    if gamma_bufs is None:
        g_cur, g_nxt = s._vec(gamma0.gamma), s.new_vec()
    else:
        g_cur, g_nxt = gamma_bufs
        if not (_is_device(gamma0.gamma) and gamma0.gamma.data_ptr() == g_cur.data_ptr()):
            src = gamma0.gamma
            if _is_device(src) and native and src.dtype == s.torch.float64 and src.is_contiguous() \
                    and src.device == g_cur.device and src.numel() >= n:
                g_src = src
            elif _is_device(src):
                g_cur[:n].copy_(src.reshape(-1)[:n])
            else:
                g_cur[:n].copy_(s._vec(src)[:n])
    cand_t = out_plan if out_plan is not None else s.new_plan()

    step_sizes: list[float] = []
    nnzs: list[int] = []
    cgs: list[int] = []
    cg_total = 0
    stop = StopReason.MAX_INNER
    tested = None
    tests: list[tuple] = []
    if native:
        # the loop body in native code (otb_inner_iteration): the initial
        # evaluate, the floor stop, the step and the inexact test with no
        # Python round trip between their kernels; same decisions, same order
        test_below = mu_k if grad_target is None else -1.0
        values: list[float] = []
        for v in range(1, config.max_inner + 1):
            r = s.ops.inner_iteration(plan_t, g_cur, g_nxt, config.armijo_sigma, config.armijo_beta,
                                      config.cg_rel_tol, config.cg_max_iters, v == 1, floor, test_below, cand_t,
                                      g_src if v == 1 else None)
            if v == 1:
                value, grad_norm = float(r.value0), float(r.grad_norm0)
                values.append(value)
            if not r.stepped:
                stop = StopReason.GRAD_FLOOR
                break
            nr = r.newton
            g_cur, g_nxt = g_nxt, g_cur
            value, grad_norm = float(nr.value_after), float(nr.grad_norm_after)
            step_sizes.append(float(nr.t))
            nnzs.append(int(nr.nnz))
            cgs.append(int(nr.cg_iters))
            values.append(value)
            cg_total += int(nr.cg_iters)
            if r.tested:
                res = r.test
                tests.append((v, grad_norm, float(res.bregman)))
                if res.bregman <= scale * mu_k:
                    stop = StopReason.INEXACT_CRITERION
                    tested = res
                    break
    else:
        value, grad_norm = s.ops.eval(plan_t, g_cur)
        values = [value]
    for v in range(1, 0 if native else config.max_inner + 1):
        if grad_norm <= floor:
            stop = StopReason.GRAD_FLOOR
            break
        value_before = value
        r = s.ops.newton_step(plan_t, g_cur, g_nxt, config.armijo_sigma, config.armijo_beta, config.cg_rel_tol,
                              config.cg_max_iters)
        g_cur, g_nxt = g_nxt, g_cur
        t = float(r.t)
        value, grad_norm = float(r.value_after), float(r.grad_norm_after)
        step_sizes.append(t)
        nnzs.append(int(r.nnz))
        cgs.append(int(r.cg_iters))
        values.append(value)
        cg_total += int(r.cg_iters)
        if recenter_every and v % recenter_every == 0:
            g_cur[:n] -= g_cur[:n].sum() / n
            value, grad_norm = s.ops.eval(plan_t, g_cur)
        if observer is not None:
            observer(NewtonStepRecord(outer_k=outer_k, inner_v=v, gamma=g_cur[:n].cpu().numpy(),
                                      grad_norm=grad_norm, step=t, cg_iters=int(r.cg_iters),
                                      value_before=value_before, value_after=value, slope=float(r.slope)))
        if grad_target is None and grad_norm < mu_k:
            res = s.ops.recover_round(plan_t, g_cur, cand_t, recover=True, metrics=True)
            tests.append((v, grad_norm, float(res.bregman)))
            if res.bregman <= scale * mu_k:
                stop = StopReason.INEXACT_CRITERION
                tested = res
                break
    if tested is None:
        tested = s.ops.recover_round(plan_t, g_cur, cand_t, recover=True, metrics=True)
    report = InnerReport(
        newton_iters=len(step_sizes),
        cg_iters_total=cg_total,
        final_grad_norm=grad_norm,
        stop_reason=stop,
        step_sizes=step_sizes,
        objective=float(tested.objective),
        kkt=float(tested.delta_kkt),
        bregman=float(tested.bregman),
        nnz=nnzs,
        cg_iters=cgs,
        values=values,
        tests=tests,
    )
    gamma_out = g_cur if (gamma_bufs is not None or _is_device(gamma0.gamma)) else g_cur[:n].cpu().numpy()
    if gamma_bufs is None and _is_device(gamma0.gamma):
        gamma_out = g_cur[:n]
    return DualState(gamma_out, generation=gamma0.generation), LogPlan.from_padded(cand_t, n), report
