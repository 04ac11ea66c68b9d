"""Wall-clock split of one bench step (cfg2) by library call, against the
kernel time the library measures with CUDA events (host-overhead probe)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_07156_b200 import instances  # noqa: E402
from paper_2603_07156_b200.core import LogPlan, OtProblem, SolverConfig  # noqa: E402
from paper_2603_07156_b200.inner_newton import inner_solve  # noqa: E402
from paper_2603_07156_b200.semidual import DualState  # noqa: E402
from paper_2603_07156_b200.session import Ops, session_for  # noqa: E402
from paper_2603_07156_b200.sinkhorn import warm_start  # noqa: E402

inst = instances.config(2, 0)
m, n = inst.cost.shape
dev = torch.device("cuda", 0)
cfg = SolverConfig(eta=inst.eta, kkt_tol=inst.kkt_tol, max_inner=1)
prob = OtProblem(torch.from_numpy(inst.cost).to(dev), inst.a, inst.b)
s = session_for(prob, inst.eta)
X0 = s.new_plan()
s.ops.init_plan(X0)
lp0 = LogPlan.from_padded(X0, n)
gst, _ = warm_start(lp0, prob, inst.eta, cfg.warm_tol, gamma0=torch.zeros(n, dtype=torch.float64, device=dev))
g0 = gst.gamma.clone()
out_plan = s.new_plan()
bufs = (s.new_vec(), s.new_vec())
acc = {}
for name in ("eval", "newton_step", "recover_round"):
    f = getattr(Ops, name)

    def wrap(self, *a, _f=f, _n=name, **k):
        t = time.perf_counter()
        r = _f(self, *a, **k)
        acc[_n] = acc.get(_n, 0.0) + time.perf_counter() - t
        return r
    setattr(Ops, name, wrap)


def step():
    return inner_solve(lp0, DualState(g0), prob, cfg, mu_k=1e3, outer_k=0, session=s, out_plan=out_plan,
                       gamma_bufs=bufs)


for _ in range(5):
    step()
torch.cuda.synchronize()
acc.clear()
K = 20
s.prof_enable(True)
t0 = time.perf_counter()
for _ in range(K):
    step()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / K * 1e6
prof = s.prof_read(reset=True)
kern = sum(v["ms"] for v in prof.values()) / K * 1e3
print(f"step wall {wall:.0f} us; kernels (classes timed by the library) {kern:.0f} us")
for k, v in acc.items():
    print(f"  {k:14s} {v / K * 1e6:8.0f} us wall")
print("  python outside calls", f"{wall - sum(acc.values()) / K * 1e6:.0f} us")
