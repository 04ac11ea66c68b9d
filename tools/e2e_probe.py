"""Break down one end-to-end step of bench.py's e2e line (host inputs).

    python tools/e2e_probe.py [config]

Times, with a device synchronize around each phase: problem construction,
session (H2D of C, norms, context), log-plan upload + check, the inner step,
and the D2H of the dual and of the candidate plan.
"""

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
from paper_2603_07156_b200.session import session_for  # noqa: E402


def main():
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    inst = instances.config(idx, 0)
    m, n = inst.cost.shape
    cfg = SolverConfig(eta=inst.eta, kkt_tol=inst.kkt_tol, max_inner=1)
    C_pin = torch.from_numpy(inst.cost).pin_memory()
    lx = np.maximum(np.log(inst.a)[:, None] + np.log(inst.b)[None, :], -1e6)
    lx_pin = torch.from_numpy(lx).pin_memory()
    g_pin = torch.zeros(n, dtype=torch.float64).pin_memory()
    torch.cuda.synchronize()
    for it in range(4):
        t = [time.perf_counter()]

        def mark():
            torch.cuda.synchronize()
            t.append(time.perf_counter())

        prob = OtProblem(C_pin, inst.a, inst.b)
        mark()
        s = session_for(prob, inst.eta)
        mark()
        lp = LogPlan(lx_pin)
        s.plan(lp)
        mark()
        gs, cand, _ = inner_solve(lp, DualState(g_pin), prob, cfg, mu_k=1e3, outer_k=0)
        mark()
        _ = np.asarray(gs.gamma).sum()
        mark()
        _ = cand.log_entries[0, 0]
        mark()
        names = ("problem", "session+H2D C", "plan H2D+check", "inner step", "D2H gamma", "D2H plan")
        d = np.diff(t) * 1e3
        print(f"iter {it}: total {1e3 * (t[-1] - t[0]):.2f} ms | " + " ".join(f"{k} {v:.2f}" for k, v in zip(names, d)))
        del prob, s, lp, gs, cand




def h2d_bandwidth():
    """Pinned host -> device copy rate of one 134 MB buffer (the size of C)."""
    src = torch.empty(4096 * 4096, dtype=torch.float64).pin_memory()
    dst = torch.empty_like(src, device="cuda")
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"H2D pinned 134 MB: {dt * 1e3:.2f} ms = {src.numel() * 8 / dt / 1e9:.1f} GB/s")


if __name__ == "__main__":
    h2d_bandwidth()
    main()
