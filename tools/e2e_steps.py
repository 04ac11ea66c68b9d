"""Per-step wall time of bench.py's e2e loop (host inputs), to spot drift (debug tool)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_07156_b200 import instances  # noqa: E402
from paper_2603_07156_b200.core import LogPlan, OtProblem, SolverConfig  # noqa: E402
from paper_2603_07156_b200.inner_newton import inner_solve  # noqa: E402
from paper_2603_07156_b200.semidual import DualState  # noqa: E402

inst = instances.config(2, 0)
m, n = inst.cost.shape
cfg = SolverConfig(eta=inst.eta, kkt_tol=inst.kkt_tol, max_inner=1)
C_pin = torch.from_numpy(inst.cost).pin_memory()
lx_pin = torch.from_numpy(np.maximum(np.log(inst.a)[:, None] + np.log(inst.b)[None, :], -1e6)).pin_memory()
g_pin = torch.zeros(n, dtype=torch.float64).pin_memory()
ts = []
for k in range(40):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hprob = OtProblem(C_pin, inst.a, inst.b)
    gs, cand, rep = inner_solve(LogPlan(lx_pin), DualState(g_pin), hprob, cfg, mu_k=1e3, outer_k=0)
    _ = np.asarray(gs.gamma).sum() + rep.objective
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
print(" ".join(f"{t:.1f}" for t in ts))
print("mem allocated MB", torch.cuda.memory_allocated() / 1e6, "reserved", torch.cuda.memory_reserved() / 1e6)

import gc
import weakref
from paper_2603_07156_b200 import session as S

hprob = OtProblem(C_pin, inst.a, inst.b)
gs, cand, rep = inner_solve(LogPlan(lx_pin), DualState(g_pin), hprob, cfg, mu_k=1e3, outer_k=0)
sess = list(getattr(hprob, S._SESSION_ATTR).values())[0]
w = weakref.ref(sess)
del sess, hprob, gs, cand, rep
print("session freed by refcount:", w() is None)
if w() is not None:
    gc.collect()
    print("after gc.collect:", w() is None)
    for r in gc.get_referrers(w())[:5]:
        print("  referrer:", type(r), str(r)[:120])
