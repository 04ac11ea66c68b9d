"""CPU timing of the bench step — TEST INFRASTRUCTURE (bench.py's
``cpu_baseline`` leg and ``--impl reference``; nothing in the package
imports this module).

It runs the REFERENCE implementation itself (``otibsn``, offline-installed
into ``baseline/_ref`` — that directory travels to the GPU box — or taken
from /root/reference/pkg/src in the build container): ``kind = "reference"``.
Where neither exists it falls back to the numpy restatement
oracle/otb_oracle.py: ``kind = "port"``.

The step is the one bench.py times on the GPU: one inner Newton iteration
plus the inexact test and the KKT metrics (``inner_solve(max_inner=1,
mu_k=1e3)`` from the outer-0 warm-started state, S/inner_newton.py:170-258,
then ``round_to_feasible`` + ``kkt_residual``, S/bregman_outer.py:51-59).

* Configs with m n <= SMALL_MN (1-3): the whole step on the whole problem.
* Configs 4-5 (C alone is 8.6 / 20 GB; the reference needs ~10 matrix-sized
  copies, more than the host's RAM): a ROW SAMPLE — rows [0, k) of the
  cost with all n columns.  Every stage of the step is row-parallel (eval,
  sparsify, the K CG products with P_rho, the Armijo trial eval, candidate
  recovery, rounding, D_phi, KKT); the length-n vector work is negligible.
  The sample runs exactly the stages of one step with K CG products (K =
  the GPU arm's CG iterations per step at this config), and the time per
  full step is the sample's time x m / k.  The sample's gamma is its own
  warm start (the rows of a renormalised to sum 1), rho the reference's
  formula with the global m, n (S/sparsify.py:30-32).
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
SMALL_MN = 1.2e8


def load_reference():
    """(modules namespace, kind): otibsn from baseline/_ref or the reference
    tree, else the oracle port."""
    for base in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (base / "otibsn" / "__init__.py").exists() or (base / "otibsn" / "semidual.py").exists():
            if str(base) not in sys.path:
                sys.path.insert(0, str(base))
            try:
                from otibsn import bregman_outer, core, feasibility, inner_newton, krylov, semidual, sinkhorn, sparsify  # noqa: F401

                class R:
                    pass

                for mod in (bregman_outer, core, feasibility, inner_newton, krylov, semidual, sinkhorn, sparsify):
                    setattr(R, mod.__name__.split(".")[-1], mod)
                R.path = str(base)
                return R, "reference"
            except Exception:   # pragma: no cover - a broken install falls back to the port
                continue
    return None, "port"


def blas_threads() -> int:
    return int(os.environ.get("OPENBLAS_NUM_THREADS", os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)))


# ----------------------------------------------------------- full step
class FullStep:
    """The bench step on the whole (small) problem."""

    def __init__(self, cost, a, b, eta, kkt_tol):
        self.R, self.kind = load_reference()
        self.cost, self.a, self.b, self.eta, self.tol = cost, a, b, eta, kkt_tol
        if self.R is not None:
            R = self.R
            self.prob = R.core.OtProblem(cost, a, b)
            self.lp = R.core.initial_plan(self.prob)
            self.g0, _ = R.sinkhorn.warm_start(self.lp, self.prob, eta, 1e-3)
            self.cfg = R.core.SolverConfig(eta=eta, kkt_tol=kkt_tol, max_inner=1)
        else:
            from oracle import otb_oracle as O

            self.O = O
            self.lx = O.product_log_plan(a, b)
            self.g0, _, _ = O.warm_start(self.lx, cost, a, b, eta, 1e-3)

    def step(self):
        if self.R is not None:
            R = self.R
            g, cand, rep = R.inner_newton.inner_solve(self.lp, self.g0, self.prob, self.cfg, mu_k=1e3, outer_k=0)
            f = R.feasibility.round_to_feasible(cand.dense(), self.a, self.b)
            R.feasibility.kkt_residual(f.entries, g.gamma, self.cost, self.a, self.b)
            return
        O = self.O
        m, n = self.cost.shape
        r = O.inner(self.lx, self.cost, self.a, self.b, self.g0, self.eta, 1e3, float(min(m, n)), max_inner=1)
        O.kkt(r.rounded, r.gamma, self.cost, self.a, self.b)

    def describe(self, steps, seconds):
        return (f"{steps} full bench steps (inner_solve(max_inner=1, mu_k=1e3) + round_to_feasible + kkt_residual) "
                f"of the whole problem in {seconds:.1f} s")


# ----------------------------------------------------------- row sample
class RowSampleStep:
    """One step's row-parallel work on rows [0, k), scaled by m / k."""

    def __init__(self, points_cost_rows, a, b, eta, m, cg_iters, k):
        self.R, self.kind = load_reference()
        self.k, self.m = k, m
        self.n = len(b)
        self.eta = eta
        self.K = int(cg_iters)
        self.cost = np.ascontiguousarray(points_cost_rows(k))
        self.a = np.ascontiguousarray(a[:k])
        self.b = b
        aw = self.a / self.a.sum()
        if self.R is not None:
            R = self.R
            self.prob = R.core.OtProblem(self.cost, self.a, b)
            self.lp = R.core.LogPlan(np.log(self.a)[:, None] + np.log(b)[None, :])
            wprob = R.core.OtProblem(self.cost, aw, b)
            st, _ = R.sinkhorn.warm_start(R.core.LogPlan(np.log(aw)[:, None] + np.log(b)[None, :]), wprob, eta, 1e-3)
            self.g0 = st
        else:
            from oracle import otb_oracle as O

            self.O = O
            self.lx = np.log(self.a)[:, None] + np.log(b)[None, :]
            self.g0, _, _ = O.warm_start(np.log(aw)[:, None] + np.log(b)[None, :], self.cost, aw, b, eta, 1e-3)

    def step(self):
        eta, m, n = self.eta, self.m, self.n
        if self.R is not None:
            R = self.R
            S, F, N = R.semidual, R.feasibility, R.inner_newton
            g = self.g0
            cache = S.compute_p(self.lp, g, self.prob, eta)                          # eval
            v0 = S.semidual_value(cache, g, self.prob, eta)
            grad = S.semidual_gradient(cache, self.prob)
            gn = float(np.linalg.norm(grad))
            rho = R.sparsify.threshold_rho(eta, m, n, gn)                           # global m, n
            sp = R.sparsify.sparsify_p(cache, rho, R.sparsify.choose_anchor(self.a))
            op = R.sparsify.SparseHessianOp(p_rho=sp, weights=self.a, eta=eta)
            d, _, _ = R.krylov.cg_solve(op, gn, -grad, 0.0, self.K)                 # exactly K products
            slope = float(grad @ d)
            g2 = S.DualState(g.gamma + d)
            cache2 = S.compute_p(self.lp, g2, self.prob, eta)                        # Armijo t = 1 trial
            v1 = S.semidual_value(cache2, g2, self.prob, eta)
            _ = v1 <= v0 + 1e-4 * slope
            cand = N.plan_candidate_log(self.lp, cache2, g2, self.prob, eta)          # recovery
            f = F.round_to_feasible(cand.dense(), self.a, self.b)                    # rounding
            F.bregman_div(f.entries, cand)                                            # D_phi
            F.kkt_residual(f.entries, g2.gamma, self.cost, self.a, self.b)            # metrics
            return
        O = self.O
        P, lse = O.softmax_rows(self.lx, self.cost, self.g0, eta)
        grad = O.gradient(P, self.a, self.b)
        gn = float(np.linalg.norm(grad))
        rows = O.threshold_rows(P, O.threshold(eta, m, n, gn), O.anchor_index(self.a))
        H = O.SparseHessian(rows, self.a, eta)
        d, _, _ = O.conjugate_gradient(H.matvec, gn, -grad, 0.0, self.K)
        g2 = self.g0 + d
        P2, lse2 = O.softmax_rows(self.lx, self.cost, g2, eta)
        cand = O.candidate_log(self.lx, self.cost, g2, lse2, self.a, eta)
        x = O.round_plan(np.exp(cand), self.a, self.b)
        O.bregman(x, cand)
        O.kkt(x, g2, self.cost, self.a, self.b)

    def describe(self, steps, seconds):
        return (f"{steps} row-sample steps: rows 0..{self.k} of {self.m} (all {self.n} columns) through eval, "
                f"sparsify, {self.K} CG products, the Armijo trial eval, candidate, rounding, D_phi and KKT "
                f"in {seconds:.1f} s; time per full step = sample time x {self.m}/{self.k}")


def make_step(inst_points, full_cost=None, cg_iters=33, budget_s=15.0):
    """The CPU step for a BASELINE configuration (PointInstance): FullStep
    for small configs (``full_cost`` given or buildable), else a RowSampleStep
    whose row count is calibrated so one sample takes about ``budget_s``."""
    pts = inst_points
    m, n = len(pts.a), len(pts.b)
    if m * n <= SMALL_MN:
        cost = full_cost if full_cost is not None else pts.build().cost
        return FullStep(cost, pts.a, pts.b, pts.eta, pts.kkt_tol), 1.0

    from paper_2603_07156_b200 import instances as I

    # the cost rows exactly as the host recipe builds them (normalised by the
    # peak over the sampled rows: uniform points put it within ~1e-3 of the
    # global peak, which does not change the work)
    def rows(k):
        c = I.sq_dist(pts.x[:k], pts.y)
        return I.normalise(c) if pts.normalised else c

    probe = RowSampleStep(rows, pts.a, pts.b, pts.eta, m, cg_iters, 64)
    t0 = time.perf_counter()
    probe.step()
    per_row = (time.perf_counter() - t0) / 64
    k = int(max(64, min(m, budget_s / max(per_row, 1e-9))))
    if k == 64:
        st = probe
    else:
        st = RowSampleStep(rows, pts.a, pts.b, pts.eta, m, cg_iters, k)
    return st, m / st.k
