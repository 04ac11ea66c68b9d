"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``otibsn`` from /root/reference/pkg/src (read-only; nothing is
copied), feeds it seeded inputs and stores inputs + outputs as small .npz
files next to this script.  The GPU box has no /root/reference, so the
parity tests there compare against these files and against the oracle
(oracle/otb_oracle.py), which tests/test_oracle_golden.py pins to them.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.path.insert(0, str(HERE.parents[1]))

from otibsn import bregman_outer, core, data, feasibility, inner_newton, krylov, semidual, sinkhorn, sparsify  # noqa: E402

from paper_2603_07156_b200 import instances  # noqa: E402


def save(name: str, **arrays):
    np.savez_compressed(HERE / f"{name}.npz", **{k: np.asarray(v) for k, v in arrays.items()})


def problem(kind: str, m: int, n: int, seed: int):
    gen = {"uniform": data.gen_uniform, "square": data.gen_square, "spherical": data.gen_spherical}[kind]
    return gen(m, n, seed)


def perturbed_gamma(n, seed, scale=0.05):
    g = np.random.default_rng(seed + 1000).normal(size=n) * scale
    return g - g.mean()


def eval_cases():
    cases = [("uniform", 24, 16, 3, 1e-1), ("uniform", 37, 29, 5, 1e-2), ("square", 64, 48, 1, 1e-2),
             ("spherical", 50, 70, 2, 5e-2), ("uniform", 33, 1, 4, 1e-2), ("uniform", 1, 7, 4, 1e-2)]
    for i, (kind, m, n, seed, eta) in enumerate(cases):
        p = problem(kind, m, n, seed)
        lp = core.initial_plan(p)
        # a non-product plan: one Newton-free perturbation of log X
        lx = lp.log_entries + 0.2 * np.random.default_rng(seed).normal(size=(m, n))
        lp = core.LogPlan(lx)
        g = perturbed_gamma(n, seed)
        st = semidual.DualState(g)
        cache = semidual.compute_p(lp, st, p, eta)
        save(f"eval_{i}", C=p.cost, a=p.source_marginal, b=p.target_marginal, logX=lp.log_entries, gamma=g,
             eta=eta, P=cache.p, lse=cache.row_logsumexp, value=semidual.semidual_value(cache, st, p, eta),
             grad=semidual.semidual_gradient(cache, p))


def sparsify_cases():
    # (kind, m, n, seed, eta, rho_mult, rho_abs)
    cases = [("uniform", 40, 30, 1, 1e-2, 30.0, None), ("square", 64, 48, 2, 1e-2, 10.0, None),
             ("spherical", 30, 50, 3, 5e-2, 100.0, None),
             ("uniform", 6, 4, 0, 10.0, None, 0.5),        # every off-anchor row falls back
             ("uniform", 20, 12, 5, 1e-2, 0.0, None)]      # rho = 0: identity
    for i, (kind, m, n, seed, eta, mult, rho_abs) in enumerate(cases):
        p = problem(kind, m, n, seed)
        lp = core.initial_plan(p)
        g = perturbed_gamma(n, seed, 0.2)
        cache = semidual.compute_p(lp, semidual.DualState(g), p, eta)
        grad = semidual.semidual_gradient(cache, p)
        gn = float(np.linalg.norm(grad))
        rho = rho_abs if rho_abs is not None else mult * sparsify.threshold_rho(eta, m, n, gn)
        anchor = sparsify.choose_anchor(p.source_marginal)
        sp = sparsify.sparsify_p(cache, rho, anchor)
        op = sparsify.SparseHessianOp(p_rho=sp, weights=p.source_marginal, eta=eta)
        v = np.random.default_rng(seed + 7).normal(size=n)
        hv = sparsify.hessian_matvec_sparse(op, v)
        x, it, res = krylov.cg_solve(op, gn, -grad, 1e-10)
        save(f"sparsify_{i}", C=p.cost, a=p.source_marginal, b=p.target_marginal, logX=lp.log_entries, gamma=g,
             eta=eta, rho=rho, anchor=anchor, row_offsets=sp.row_offsets, col_indices=sp.col_indices,
             values=sp.values, anchor_row=sp.anchor_row, d=op.diag_cache, v=v, hv=hv, cg_x=x, cg_iters=it,
             cg_res=res, grad_norm=gn)


def newton_cases():
    cases = [("uniform", 24, 16, 1, 1e-3), ("uniform", 24, 16, 2, 1e-2), ("square", 32, 32, 0, 1e-2),
             ("spherical", 20, 28, 4, 1e-2)]
    for i, (kind, m, n, seed, eta) in enumerate(cases):
        p = problem(kind, m, n, seed)
        lp = core.initial_plan(p)
        st = semidual.DualState(np.zeros(n))
        new, t, its = inner_newton.newton_step(lp, st, p, eta)
        save(f"newton_{i}", C=p.cost, a=p.source_marginal, b=p.target_marginal, logX=lp.log_entries,
             gamma=np.zeros(n), eta=eta, gamma_new=new.gamma, t=t, cg_iters=its)


def rounding_cases():
    for i, (m, n, seed, scale) in enumerate([(20, 15, 0, 0.5), (33, 41, 1, 2.0), (8, 8, 2, 0.0), (5, 9, 3, 30.0)]):
        p = problem("uniform", m, n, seed)
        lx = core.initial_plan(p).log_entries + scale * np.random.default_rng(seed).normal(size=(m, n))
        lp = core.LogPlan(lx)
        g = perturbed_gamma(n, seed)
        rounded = feasibility.round_to_feasible(lp.dense(), p.source_marginal, p.target_marginal)
        dphi = feasibility.bregman_div(rounded.entries, lp)
        rep = feasibility.kkt_residual(rounded.entries, g, p.cost, p.source_marginal, p.target_marginal)
        save(f"round_{i}", C=p.cost, a=p.source_marginal, b=p.target_marginal, logX=lp.log_entries, gamma=g,
             rounded=rounded.entries, bregman=dphi, objective=float((p.cost * rounded.entries).sum()),
             delta_p=rep.delta_p, delta_d=rep.delta_d, delta_c=rep.delta_c, delta_kkt=rep.delta_kkt)


def candidate_cases():
    for i, (m, n, seed, eta) in enumerate([(24, 16, 0, 1e-2), (30, 45, 1, 5e-3)]):
        p = problem("uniform", m, n, seed)
        lp = core.initial_plan(p)
        g = perturbed_gamma(n, seed, 0.5)
        st = semidual.DualState(g)
        cache = semidual.compute_p(lp, st, p, eta)
        cand = inner_newton.plan_candidate_log(lp, cache, st, p, eta)
        save(f"candidate_{i}", C=p.cost, a=p.source_marginal, b=p.target_marginal, logX=lp.log_entries, gamma=g,
             eta=eta, candidate=cand.log_entries)


def warm_cases():
    for i, (kind, m, n, seed, eta) in enumerate([("uniform", 24, 16, 0, 1e-2), ("square", 40, 40, 1, 1e-2),
                                                 ("spherical", 30, 20, 2, 5e-3)]):
        p = problem(kind, m, n, seed)
        lp = core.initial_plan(p)
        st, zeta = sinkhorn.warm_start(lp, p, eta, 1e-3)
        # count sweeps with an instrumented copy of the loop's error sequence
        save(f"warm_{i}", C=p.cost, a=p.source_marginal, b=p.target_marginal, logX=lp.log_entries, eta=eta,
             gamma=st.gamma, zeta=zeta)


def inner_cases():
    for i, (kind, m, n, seed, eta) in enumerate([("uniform", 24, 16, 0, 1e-2), ("square", 32, 32, 1, 1e-2)]):
        p = problem(kind, m, n, seed)
        cfg = core.SolverConfig(eta=eta, kkt_tol=1e-9)
        lp = core.initial_plan(p)
        st, _ = sinkhorn.warm_start(lp, p, eta, cfg.warm_tol)
        g, cand, rep = inner_newton.inner_solve(lp, st, p, cfg, mu_k=1e-4, outer_k=0)
        save(f"inner_{i}", C=p.cost, a=p.source_marginal, b=p.target_marginal, logX=lp.log_entries, eta=eta,
             gamma0=st.gamma, gamma=g.gamma, candidate=cand.log_entries, newton_iters=rep.newton_iters,
             cg_iters_total=rep.cg_iters_total, final_grad_norm=rep.final_grad_norm,
             stop=rep.stop_reason.value, steps=np.asarray(rep.step_sizes))


def solve_cases():
    cases = [("uniform", 12, 10, 0, 1e-2, 1e-9), ("square", 16, 16, 1, 1e-3, 1e-9), ("spherical", 20, 14, 2, 1e-2, 1e-8),
             ("uniform", 32, 32, 3, 1e-3, 1e-10)]
    for i, (kind, m, n, seed, eta, tol) in enumerate(cases):
        p = problem(kind, m, n, seed)
        cfg = core.SolverConfig(eta=eta, kkt_tol=tol)
        res = bregman_outer.ibsn_solve(p, cfg)
        tr = res.trajectory.records
        save(f"solve_{i}", C=p.cost, a=p.source_marginal, b=p.target_marginal, eta=eta, kkt_tol=tol,
             objective=res.objective, kkt=res.kkt, outer_iters=res.outer_iters, rounded=res.rounded_plan,
             final_log=res.final_logplan.log_entries,
             inner_total=np.array([r.inner_total for r in tr]), cg_total=np.array([r.cg_total for r in tr]),
             traj_objective=np.array([r.objective for r in tr]), traj_kkt=np.array([r.kkt for r in tr]))


def eot_cases():
    """eot_single_solve (bregman_outer.py:284-327): one entropic subproblem on
    the all-ones reference plan, Newton to the gradient target kkt_tol."""
    cases = [("uniform", 20, 16, 0, 5e-2, 1e-9), ("square", 24, 24, 1, 2e-2, 1e-10), ("spherical", 18, 30, 2, 1e-1, 1e-9)]
    for i, (kind, m, n, seed, eta, tol) in enumerate(cases):
        p = problem(kind, m, n, seed)
        cfg = core.SolverConfig(eta=eta, kkt_tol=tol)
        res = bregman_outer.eot_single_solve(p, cfg)
        rec = res.trajectory.records[-1]
        save(f"eot_{i}", C=p.cost, a=p.source_marginal, b=p.target_marginal, eta=eta, kkt_tol=tol,
             objective=res.objective, kkt=res.kkt, rounded=res.rounded_plan, final_log=res.final_logplan.log_entries,
             newton_iters=rec.inner_total, cg_total=rec.cg_total, grad_norm=rec.grad_norm)


def ibsink_cases():
    """ibsink_solve (bregman_outer.py:191-281): Sinkhorn sweeps as the inner solver."""
    # truncated at 6 outers: the Sinkhorn inner loop needs 10^4-10^5 sweeps to tol
    cases = [("uniform", 14, 12, 0, 5e-2, 1e-8), ("square", 16, 16, 1, 2e-2, 1e-8), ("spherical", 12, 20, 2, 1e-1, 1e-9)]
    for i, (kind, m, n, seed, eta, tol) in enumerate(cases):
        p = problem(kind, m, n, seed)
        cfg = core.SolverConfig(eta=eta, kkt_tol=tol, max_outer=6)
        res = bregman_outer.ibsink_solve(p, cfg)
        tr = res.trajectory.records
        save(f"ibsink_{i}", C=p.cost, a=p.source_marginal, b=p.target_marginal, eta=eta, kkt_tol=tol,
             objective=res.objective, kkt=res.kkt, outer_iters=res.outer_iters, rounded=res.rounded_plan,
             final_log=res.final_logplan.log_entries, inner_total=np.array([r.inner_total for r in tr]),
             traj_objective=np.array([r.objective for r in tr]), max_outer=6)


def config_scalars():
    """BASELINE configs 1 and 2 (seed 0): the reference's end-to-end numbers."""
    out = {}
    for idx in (1, 2):
        inst = instances.config(idx, 0)
        p = core.OtProblem(inst.cost, inst.a, inst.b)
        res = bregman_outer.ibsn_solve(p, core.SolverConfig(eta=inst.eta, kkt_tol=inst.kkt_tol))
        last = res.trajectory.records[-1]
        out[f"cfg{idx}"] = dict(objective=res.objective, kkt=res.kkt, outer_iters=res.outer_iters,
                                newton_total=last.inner_total, cg_total=last.cg_total,
                                objectives=[r.objective for r in res.trajectory.records],
                                inner_totals=[r.inner_total for r in res.trajectory.records],
                                cg_totals=[r.cg_total for r in res.trajectory.records])
    (HERE / "config_scalars.json").write_text(json.dumps(out, indent=1))


def dense_cases():
    """Kernel-level drop-ins on dense LINEAR matrices (feasibility.py:44-127,
    semidual.py:103-114, sinkhorn.py:41-58): an infeasible x with negative
    entries for kkt_residual (certified as given), round_to_feasible of a
    nonnegative infeasible x, bregman_div, c_transform, gap, the exact Hessian
    product and single Sinkhorn updates."""
    for i, (kind, m, n, seed, eta) in enumerate([("uniform", 23, 17, 0, 1e-2), ("square", 40, 33, 1, 5e-2),
                                                 ("spherical", 9, 50, 2, 1e-2)]):
        p = problem(kind, m, n, seed)
        rng = np.random.default_rng(seed + 50)
        x = rng.random((m, n)) * (2.0 / (m * n))                 # nonnegative, marginals off
        xneg = x - 0.3 / (m * n)                                  # some negative entries
        lp = core.LogPlan(core.initial_plan(p).log_entries + 0.3 * rng.normal(size=(m, n)))
        g = perturbed_gamma(n, seed, 0.1)
        z0 = rng.normal(size=m) * 0.01
        rounded = feasibility.round_to_feasible(x, p.source_marginal, p.target_marginal)
        rep = feasibility.kkt_residual(xneg, g, p.cost, p.source_marginal, p.target_marginal)
        cache = semidual.compute_p(lp, semidual.DualState(g), p, eta)
        v = rng.normal(size=n)
        hv = semidual.hessian_matvec_exact(cache, p, eta, v)
        st = sinkhorn.TwoDualState(gamma=g, zeta=z0)
        zu = sinkhorn.zeta_update(lp, st, p, eta)
        gu = sinkhorn.gamma_update(lp, st, p, eta)
        spl = sinkhorn.scaled_plan_log(lp, st, p, eta)
        save(f"dense_{i}", C=p.cost, a=p.source_marginal, b=p.target_marginal, x=x, xneg=xneg, logY=lp.log_entries,
             gamma=g, zeta0=z0, eta=eta, v=v, rounded=rounded.entries, bregman=feasibility.bregman_div(x, lp),
             kkt=np.array([rep.delta_p, rep.delta_d, rep.delta_c, rep.delta_kkt]), zeta_used=rep.zeta_used,
             c_transform=feasibility.c_transform(g, p.cost), gap=feasibility.gap(rounded, p.cost, 0.01),
             hv=hv, zeta_upd=zu.zeta, gamma_upd=gu.gamma, scaled_log=spl)


def config_seeds():
    """BASELINE configs 1 and 2 at seeds 1 and 2, and config 3 (seed 0)
    truncated at max_outer=2: the reference's scalars per outer."""
    out = {}
    jobs = [(1, 1, None), (1, 2, None), (2, 1, None), (2, 2, None), (3, 0, 2)]
    for idx, seed, max_outer in jobs:
        inst = instances.config(idx, seed)
        p = core.OtProblem(inst.cost, inst.a, inst.b)
        kw = {} if max_outer is None else {"max_outer": max_outer}
        res = bregman_outer.ibsn_solve(p, core.SolverConfig(eta=inst.eta, kkt_tol=inst.kkt_tol, **kw))
        last = res.trajectory.records[-1]
        out[f"cfg{idx}_seed{seed}" + ("" if max_outer is None else f"_outer{max_outer}")] = dict(
            objective=res.objective, kkt=res.kkt, outer_iters=res.outer_iters, max_outer=max_outer,
            newton_total=last.inner_total, cg_total=last.cg_total,
            objectives=[r.objective for r in res.trajectory.records],
            kkts=[r.kkt for r in res.trajectory.records],
            inner_totals=[r.inner_total for r in res.trajectory.records],
            cg_totals=[r.cg_total for r in res.trajectory.records])
        print(idx, seed, out[list(out)[-1]]["objective"], flush=True)
        (HERE / "config_seeds.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    which = sys.argv[1:] or ["eval", "sparsify", "newton", "rounding", "candidate", "warm", "inner", "solve",
                             "eot", "ibsink", "configs"]
    fns = {"eval": eval_cases, "sparsify": sparsify_cases, "newton": newton_cases, "rounding": rounding_cases,
           "candidate": candidate_cases, "warm": warm_cases, "inner": inner_cases, "solve": solve_cases,
           "eot": eot_cases, "ibsink": ibsink_cases, "configs": config_scalars, "dense": dense_cases,
           "seeds": config_seeds}
    for w in which:
        fns[w]()
        print("done", w)
