"""Kernel timeline of bench steps (cfg2) from CUPTI via torch.profiler:
per-kernel start/duration and the idle gaps between launches (debug tool)."""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_07156_b200 import instances  # noqa: E402
from paper_2603_07156_b200.core import LogPlan, OtProblem, SolverConfig  # noqa: E402
from paper_2603_07156_b200.inner_newton import inner_solve  # noqa: E402
from paper_2603_07156_b200.semidual import DualState  # noqa: E402
from paper_2603_07156_b200.session import session_for  # noqa: E402
from paper_2603_07156_b200.sinkhorn import warm_start  # noqa: E402

inst = instances.config(int(os.environ.get("CFG", "2")), 0)
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


def step():
    return inner_solve(lp0, DualState(g0), prob, cfg, mu_k=1e3, outer_k=0, session=s, out_plan=out_plan,
                       gamma_bufs=bufs)


for _ in range(5):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = t0
busy = 0.0
gaps = {}
print(f"{'start':>8} {'dur':>7} {'gap':>6}  kernel")
for e in ev:
    st, en = e.time_range.start, e.time_range.end
    gap = st - prev_end
    busy += en - st
    print(f"{st - t0:8.1f} {en - st:7.1f} {gap:6.1f}  {e.name[:90]}")
    gaps[e.name[:60]] = gaps.get(e.name[:60], 0.0) + max(gap, 0.0)
    prev_end = max(prev_end, en)
span = prev_end - t0
print(f"span {span / 3:.0f} us/step, busy {busy / 3:.0f} us/step, idle {(span - busy) / 3:.0f} us/step")
print("idle before (us/step):")
for k, v in sorted(gaps.items(), key=lambda kv: -kv[1])[:12]:
    print(f"  {v / 3:7.1f}  {k}")
