"""hess_apply time against the kept density, dense P_rho vs the sparse format of the context
(debug tool): the thresholds of the dense mode.   python tools/hv_density_sweep.py CONFIG"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
res = bench.Resident(idx, 0, dev, None, 1, 0)
s, m, n = res.s, res.m, res.n
g0 = res.g0
v = s._vec(np.random.default_rng(0).normal(size=n))
out = s.new_vec()
val, gn = s.ops.eval(res.X0, g0)
rho0 = res.pts.eta * gn / (m * n)
print(f"config {idx}: m {m} n {n} rho0 {rho0:.3e} geometry", {k: s.info()[k] for k in ("hv_mode", "wc_nq", "wc_win", "wc_ncl")})
for mult in (1.0, 1e2, 1e3, 3e3, 1e4, 3e4, 1e5, 1e6):
    row = []
    for mode in ("1", "0"):
        os.environ["OTB_HV_DENSE"] = mode
        s.ops.eval(res.X0, g0)
        nnz = s.ops.sparsify(res.X0, g0, rho0 * mult)
        for _ in range(3):
            s.ops.hess_apply(v, 0.0, out)
        s.prof_enable(True)
        for _ in range(10):
            s.ops.hess_apply(v, 0.0, out)
        h = s.prof_read(reset=True)["hess_apply"]
        s.prof_enable(False)
        row.append(1e3 * h["ms"] / h["launches"])
    print(f"  rho x {mult:8.0e}: kept {nnz / (m * n):7.4f}   dense {row[0]:8.1f} us   sparse format {row[1]:8.1f} us")
os.environ.pop("OTB_HV_DENSE", None)
