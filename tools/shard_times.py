"""Per-kernel times of ONE rank's row shard (debug / projection tool): the dense passes and
hess_apply depend only on the local row count, n and the kept density, so a problem of m/N rows
and the same n shows what each of N ranks launches.  Not a multi-GPU measurement: the all-reduces
are absent.   python tools/shard_times.py CONFIG "1 2 4 8" """
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2603_07156_b200 import instances

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 5
worlds = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1 2 4 8").split()]
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
full = instances.CONFIGS[idx]
base = None
orig = instances.config_points
for N in worlds:
    m = full["m"] // N
    if idx == 5:
        pts = instances.uniform2d_points(m, full["n"], 0, eta=full["eta"], tol=full["tol"])
    elif idx == 4:
        pts = instances.colour_points(m, full["n"], 0, eta=full["eta"], tol=full["tol"])
    else:
        raise SystemExit("configs 4 and 5 only")
    instances.config_points = lambda i, s=0, _p=pts: _p
    res = bench.Resident(idx, 0, dev, None, 1, 0)
    ms, launches, rep, clocks = bench.timed_steps(res, 3, 3, 1, dev, 0)
    roof = bench.roofline(res, idx, 3)
    per = {k: round(v["us_per_launch"], 1) for k, v in roof["per_kernel"].items()}
    cg = rep.cg_iters[-1] if rep.cg_iters else 0
    line = {"rows": m, "n": full["n"], "world": N, "ms_per_step": round(ms / 3, 2), "cg_iters": cg,
            "density": round((rep.nnz[-1] if rep.nnz else 0) / (m * full["n"]), 4), "us_per_launch": per,
            "sm_mhz": clocks["sm_mhz"]}
    if base is None:
        base = line
    # (time at the first row count) x (rows share) / time: 1.0 = the kernel scales with the local rows
    line["compute_efficiency"] = {k: round(base["us_per_launch"][k] * m / base["rows"] / per[k], 3)
                                  for k in per if k != "cg_vector" and base["us_per_launch"].get(k, 0) > 0}
    line["step_efficiency"] = round(base["ms_per_step"] * m / base["rows"] / line["ms_per_step"], 3)
    print(json.dumps(line), flush=True)
    res.s.close()
    del res
    torch.cuda.empty_cache()
instances.config_points = orig
