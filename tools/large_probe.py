"""Large-config probe: one Newton step against the oracle, then a few outers.

    python tools/large_probe.py CONFIG [max_outer] [--no-oracle]

Prints the geometry libotb picked, eval/Newton parity against the CPU oracle
on the first step (skipped with --no-oracle), and per-outer timings of a
truncated ibsn_solve.
"""

import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_07156_b200 import instances  # noqa: E402
from paper_2603_07156_b200.bregman_outer import ibsn_solve  # noqa: E402
from paper_2603_07156_b200.core import LogPlan, OtProblem, SolverConfig  # noqa: E402
from paper_2603_07156_b200.session import session_for  # noqa: E402


def main():
    idx = int(sys.argv[1])
    max_outer = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 3
    use_oracle = "--no-oracle" not in sys.argv
    t0 = time.time()
    inst = instances.config(idx, 0)
    m, n = inst.cost.shape
    print(f"cfg{idx} m={m} n={n} eta={inst.eta} built in {time.time() - t0:.1f}s", flush=True)
    dev = torch.device("cuda", 0)
    prob = OtProblem(torch.from_numpy(inst.cost).to(dev), inst.a, inst.b)
    s = session_for(prob, inst.eta)
    print("geometry", s.info(), flush=True)

    # first Newton step from X0 = a b^T, gamma = 0, against the oracle
    X0 = s.new_plan()
    s.ops.init_plan(X0)
    g = s.new_vec()
    v0, gn0 = s.ops.eval(X0, g)
    g2 = s.new_vec()
    torch.cuda.synchronize()
    t = time.time()
    r = s.ops.newton_step(X0, g, g2, 1e-4, 0.8, 1e-10, None)
    torch.cuda.synchronize()
    print(f"newton step: {1e3 * (time.time() - t):.1f} ms  nnz={r.nnz} density={r.nnz / (m * n):.3f} "
          f"cg={r.cg_iters} t={r.t} L {r.value_before:.17g} -> {r.value_after:.17g} |g| {r.grad_norm_after:.6g}",
          flush=True)
    if use_oracle:
        sys.path.insert(0, ROOT)
        from oracle import otb_oracle as O

        lx = np.log(inst.a)[:, None] + np.log(inst.b)[None, :]
        t = time.time()
        res = O.newton_step(lx, inst.cost, inst.a, inst.b, np.zeros(n), inst.eta)
        gam, tt, cg = res[:3]
        print(f"oracle newton step {time.time() - t:.1f}s cg={cg} t={tt}", flush=True)
        gd = g2[:n].cpu().numpy()
        print(f"  |dgamma|/|gamma| = {np.linalg.norm(gd - gam) / np.linalg.norm(gam):.3e}  "
              f"cg {r.cg_iters} vs {cg}", flush=True)
    del s, X0, g, g2

    cfg = SolverConfig(eta=inst.eta, kkt_tol=inst.kkt_tol, max_outer=max_outer)
    times = []
    last = [time.time()]

    def on_outer(*args, **kw):
        torch.cuda.synchronize()
        now = time.time()
        times.append(now - last[0])
        last[0] = now

    torch.cuda.synchronize()
    t = time.time()
    last[0] = t
    res = ibsn_solve(prob, cfg, on_outer=on_outer)
    torch.cuda.synchronize()
    el = time.time() - t
    print(f"ibsn_solve max_outer={max_outer}: {el:.2f}s outer={res.outer_iters} newton={res.newton_iters} "
          f"cg={res.cg_iters} objective={res.objective:.17g} kkt={res.kkt:.3e}", flush=True)
    print("  per-outer s:", " ".join(f"{x:.3f}" for x in times), flush=True)


if __name__ == "__main__":
    main()
