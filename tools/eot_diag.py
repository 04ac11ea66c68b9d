"""Step-by-step eot_single_solve trajectory, device vs oracle (debug tool)."""
import os, sys
sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
import numpy as np
from conftest import golden
from oracle import otb_oracle as O

name = sys.argv[1] if len(sys.argv) > 1 else "eot_1"
g = golden(name)
C, a, b, eta, tol = g["C"], g["a"], g["b"], float(g["eta"]), float(g["kkt_tol"])
m, n = C.shape
lx = np.zeros((m, n))
gam, _, sw = O.warm_start(lx, C, a, b, eta, 1e-3)
print("oracle warm sweeps", sw)
res = O.inner(lx, C, a, b, gam, eta, 0.0, float(min(m, n)), grad_target=tol)
for i, st in enumerate(res.steps):
    print("oracle step", i, st)
print("oracle newton", res.newton_iters, "grad", res.grad_norm, "golden", int(g["newton_iters"]), float(g["grad_norm"]))
if os.environ.get("DEV", "1") == "1":
    import torch
    import paper_2603_07156_b200 as P
    recs = []
    prob = P.OtProblem(C, a, b)
    cfg = P.SolverConfig(eta=eta, kkt_tol=tol)
    from paper_2603_07156_b200 import inner_newton
    orig = inner_newton.inner_solve
    def wrapped(*args, **kw):
        kw["observer"] = lambda r: print("device step", r.inner_v, "grad", r.grad_norm, "t", r.step, "cg", r.cg_iters,
                                         "f", r.value_before, r.value_after, "slope", r.slope)
        return orig(*args, **kw)
    import paper_2603_07156_b200.bregman_outer as BO
    BO.inner_solve = wrapped
    out = P.eot_single_solve(prob, cfg)
    print("device newton", out.newton_iters, "warm", out.warm_sweeps)
