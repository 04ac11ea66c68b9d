"""ibsn_solve timing probe (debug tool): repeats the solve of a BASELINE config from the
bench's device-resident set-up and prints the time of each repeat and the per-kernel-class
profile of the last.   python tools/solve_probe.py CONFIG [REPEATS]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2603_07156_b200.bregman_outer import ibsn_solve
from paper_2603_07156_b200.core import SolverConfig

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
res = bench.Resident(idx, 0, dev, None, 1, 0)
cfg = SolverConfig(eta=res.pts.eta, kkt_tol=res.pts.kkt_tol)
for k in range(reps):
    last = k == reps - 1
    if last:
        res.s.prof_enable(True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = ibsn_solve(res.prob, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"repeat {k}: {dt:.4f} s  outer {r.outer_iters} newton {r.newton_iters} cg {r.cg_iters} "
          f"sweeps {r.warm_sweeps} same_session {r._session is res.s}")
prof = res.s.prof_read(reset=True)
tot = sum(v["ms"] for v in prof.values())
print(f"profiled kernel time {tot:.1f} ms")
for k, v in prof.items():
    if v["launches"]:
        print(f"  {k:12s} {v['ms']:9.2f} ms  {v['launches']:5d} launches  {1e3 * v['ms'] / v['launches']:9.1f} us each")
# kept density and CG iterations per Newton iteration of the last repeat (OTB_PROBE_TRACE=1)
if os.environ.get("OTB_PROBE_TRACE") == "1":
    import paper_2603_07156_b200.bregman_outer as BO
    from paper_2603_07156_b200 import inner_newton as IN

    reports = []
    orig = IN.inner_solve

    def spy(*a, **k):
        out = orig(*a, **k)
        reports.append(out[2])
        return out

    BO.inner_solve = spy
    ibsn_solve(res.prob, cfg)
    m, n = res.m, res.n
    for k, rep in enumerate(reports):
        print(f"  outer {k}: cg {list(rep.cg_iters)} density {[round(z / (m * n), 4) for z in rep.nnz]}")
