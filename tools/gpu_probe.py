"""Stage-by-stage GPU probe of libotb against the CPU oracle (debug tool)."""
import sys, time, traceback
import numpy as np
sys.path.insert(0, "/root/repo")
import torch
from oracle import otb_oracle as O
from paper_2603_07156_b200 import instances as I
from paper_2603_07156_b200.core import OtProblem, LogPlan, SolverConfig
from paper_2603_07156_b200 import semidual, sparsify, krylov, inner_newton, feasibility, sinkhorn, bregman_outer
from paper_2603_07156_b200.session import session_for


def rel(a, b):
    a = np.asarray(a); b = np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


def stage(name, fn):
    t = time.time()
    try:
        fn()
        print(f"[ok] {name} ({time.time()-t:.2f}s)", flush=True)
    except Exception:
        print(f"[FAIL] {name}", flush=True)
        traceback.print_exc()


def case(m, n, seed, eta):
    C, a, b = I.small_uniform(m, n, seed)
    prob = OtProblem(C, a, b)
    lx = O.product_log_plan(a, b)
    g = np.random.default_rng(seed + 100).normal(size=n) * 0.01
    g -= g.mean()
    print(f"--- case m={m} n={n} eta={eta}", flush=True)

    def s_eval():
        cache = semidual.compute_p(LogPlan(lx), semidual.DualState(g), prob, eta)
        P, lse = O.softmax_rows(lx, C, g, eta)
        val = O.objective(lse, g, a, b, eta)
        grad = O.gradient(P, a, b)
        print("  info", cache.session.info())
        print("  lse rel", rel(cache.row_logsumexp, lse), "value", cache.value, val, "grad rel", rel(semidual.semidual_gradient(cache, prob), grad))
        print("  P rel", rel(cache.p, P))
        assert rel(cache.row_logsumexp, lse) < 1e-12
    stage("eval", s_eval)

    def s_sparsify():
        cache = semidual.compute_p(LogPlan(lx), semidual.DualState(g), prob, eta)
        P, lse = O.softmax_rows(lx, C, g, eta)
        gn = float(np.linalg.norm(O.gradient(P, a, b)))
        rho = O.threshold(eta, m, n, gn) * 50
        anc = O.anchor_index(a)
        ref = O.threshold_rows(P, rho, anc)
        got = sparsify.sparsify_p(cache, rho, anc)
        print("  nnz", got.values.size, ref.vals.size, "rowptr eq", np.array_equal(got.row_offsets, ref.row_ptr))
        print("  cols eq", np.array_equal(got.col_indices, ref.cols), "vals rel", rel(got.values, ref.vals) if got.values.size == ref.vals.size else None)
        print("  anchor rel", rel(got.anchor_row, ref.anchor_row))
        op = sparsify.SparseHessianOp(got)
        H = O.SparseHessian(ref, a, eta)
        print("  d rel", rel(op.diag_cache, H.d))
        v = np.random.default_rng(1).normal(size=n)
        print("  Hv rel", rel(op.matvec(v), H.matvec(v)))
        rhs = -O.gradient(P, a, b)
        x, it, res = krylov.cg_solve(op, gn, rhs, 1e-10)
        xr, itr, resr = O.conjugate_gradient(H.matvec, gn, rhs, 1e-10)
        print("  cg iters", it, itr, "x rel", rel(x, xr), "res", res, resr)
    stage("sparsify+hv+cg", s_sparsify)

    def s_newton():
        gam, t, its = inner_newton.newton_step(LogPlan(lx), semidual.DualState(g), prob, eta)
        gr, tr, itr = O.newton_step(lx, C, a, b, g, eta)
        print("  t", t, tr, "cg", its, itr, "gamma rel", rel(gam.gamma, gr))
    stage("newton_step", s_newton)

    def s_round():
        fp = feasibility.round_log_plan(LogPlan(lx + 0.3 * np.random.default_rng(2).normal(size=(m, n))), prob, gamma=g, metrics=True)
        L = O.clamp_log_plan(lx + 0.3 * np.random.default_rng(2).normal(size=(m, n)))
        R = O.round_plan(np.exp(L), a, b)
        D = O.bregman(R, L)
        K = O.kkt(R, g, C, a, b)
        print("  D", fp.bregman, D, "obj", fp.objective, float((C * R).sum()), "kkt", fp.delta_kkt, K["delta_kkt"])
        print("  rounded rel", rel(fp.entries, R))
    stage("round", s_round)

    def s_warm():
        ds, z = sinkhorn.warm_start(LogPlan(lx), prob, eta, 1e-3)
        gr, zr, sw = O.warm_start(lx, C, a, b, eta, 1e-3)
        print("  sweeps", sweeps_of(prob, eta), sw, "gamma rel", rel(ds.gamma, gr), "zeta rel", rel(z, zr))
    stage("warm_start", s_warm)


def sweeps_of(prob, eta):
    return session_for(prob, eta)._last_warm


def solve(idx):
    inst = I.config(idx, 0)
    prob = OtProblem(inst.cost, inst.a, inst.b)
    cfg = SolverConfig(eta=inst.eta, kkt_tol=inst.kkt_tol)
    t = time.time()
    r = bregman_outer.ibsn_solve(prob, cfg)
    torch.cuda.synchronize()
    dt = time.time() - t
    print(f"cfg{idx}: obj {r.objective!r} outer {r.outer_iters} newton {r.newton_iters} cg {r.cg_iters} kkt {r.kkt} sweeps {r.warm_sweeps} time {dt:.3f}s", flush=True)
    t = time.time()
    r = bregman_outer.ibsn_solve(prob, cfg)
    torch.cuda.synchronize()
    print(f"   2nd run time {time.time()-t:.3f}s", flush=True)


if __name__ == "__main__":
    print(torch.cuda.get_device_name(), flush=True)
    case(24, 16, 3, 1e-2)
    case(37, 29, 5, 5e-2)
    case(300, 200, 7, 1e-2)
    case(64, 9000, 1, 1e-2)
    case(40, 16400, 2, 1e-2)
    stage("solve cfg1", lambda: solve(1))
    stage("solve cfg2", lambda: solve(2))
