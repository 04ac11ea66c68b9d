"""CUPTI timeline of one e2e step (host inputs): copies, kernels and gaps (debug tool)."""
import os, sys
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
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


def step():
    hprob = OtProblem(C_pin, inst.a, inst.b)
    gs, cand, rep = inner_solve(LogPlan(lx_pin), DualState(g_pin), hprob, cfg, mu_k=1e3, outer_k=0)
    return np.asarray(gs.gamma).sum() + rep.objective


for _ in range(4):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - e.time_range.start:8.1f}  {e.name[:70]}")
print("span", ev[-1].time_range.end - t0)
