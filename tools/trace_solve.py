"""Per-outer trace of ibsn_solve on the GPU vs the CPU oracle (debug tool)."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from conftest import golden
from oracle import otb_oracle as O
import paper_2603_07156_b200 as P
from paper_2603_07156_b200 import inner_newton as IN

name = sys.argv[1] if len(sys.argv) > 1 else "solve_2"
g = golden(name)
C, a, b, eta, tol = g["C"], g["a"], g["b"], float(g["eta"]), float(g["kkt_tol"])
m, n = C.shape
scale = float(min(m, n))
reports = []
orig = IN.inner_solve
def spy(*args, **kw):
    out = orig(*args, **kw)
    reports.append(out[2])
    return out
import paper_2603_07156_b200.bregman_outer as BO
BO.inner_solve = spy
steps = []
res = P.ibsn_solve(P.OtProblem(C, a, b), P.SolverConfig(eta=eta, kkt_tol=tol),
                   observer=lambda r: steps.append((r.outer_k, r.inner_v, r.grad_norm, r.step, r.cg_iters, r.value_after)))
# oracle trace
lx = O.product_log_plan(a, b); gamma = np.zeros(n); zeta = np.zeros(m)
for k in range(res.outer_iters):
    mu = O.mu(k)
    gamma, zeta, sw = O.warm_start(lx, C, a, b, eta, 1e-3, gamma, zeta)
    ev = O.evaluate(lx, C, a, b, gamma, eta); gr = O.gradient(ev.p, a, b); gn = np.linalg.norm(gr)
    otr = []
    for v in range(1, 501):
        if gn <= 1e-15: break
        ev, info = O.step_from(lx, C, a, b, ev, gr, eta)
        gr = O.gradient(ev.p, a, b); gn = np.linalg.norm(gr)
        rec = [v, gn, info.t, info.cg_iters, ev.value]
        if gn < mu:
            cand = O.candidate_log(lx, C, ev.gamma, ev.lse, a, eta)
            D = O.bregman(O.round_plan(np.exp(cand), a, b), cand)
            rec.append(D / (scale * mu))
            otr.append(rec)
            if D <= scale * mu: break
        else:
            otr.append(rec)
    gamma = ev.gamma
    lx = O.candidate_log(lx, C, gamma, ev.lse, a, eta)
    rep = reports[k]
    gtr = [s for s in steps if s[0] == k]
    same = rep.newton_iters == len(otr)
    if not same or k < 2:
        print(f"outer {k}: mu {mu:.3e} gpu newton {rep.newton_iters} oracle {len(otr)} sweeps {sw}")
        for s in gtr: print("   gpu   v=%d gn=%.6e t=%g cg=%d L=%.17g" % (s[1], s[2], s[3], s[4], s[5]))
        for t in rep.tests: print("   gpu   test v=%d gn=%.6e D/thr=%.6e" % (t[0], t[1], t[2] / (scale * mu)))
        for r in otr: print("   orac  v=%d gn=%.6e t=%g cg=%d L=%.17g %s" % (r[0], r[1], r[2], r[3], r[4], ("D/thr=%.6e" % r[5]) if len(r) > 5 else ""))
print("objective", res.objective, float(g["objective"]))
