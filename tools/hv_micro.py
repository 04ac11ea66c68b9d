"""Micro-benchmark of hess_apply / CG variants on the cfg2 first Newton step (debug tool)."""
import os, sys, time, json
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2603_07156_b200 import instances
from paper_2603_07156_b200.core import OtProblem, LogPlan, SolverConfig
from paper_2603_07156_b200.session import session_for, _CTX_POOL
from paper_2603_07156_b200.sinkhorn import warm_start

cfgi = int(os.environ.get("CFG", "2"))
inst = instances.config(cfgi, 0)
m, n = inst.cost.shape
dev = torch.device("cuda", 0)
prob = OtProblem(torch.from_numpy(inst.cost).to(dev), inst.a, inst.b)
s = session_for(prob, inst.eta)
X0 = s.new_plan(); s.ops.init_plan(X0)
gst, _ = warm_start(LogPlan.from_padded(X0, n), prob, inst.eta, 1e-3, gamma0=torch.zeros(n, dtype=torch.float64, device=dev))
g0 = s._vec(gst.gamma)
val, gn = s.ops.eval(X0, g0)
rho = inst.eta * gn / (m * n)
nnz = s.ops.sparsify(X0, g0, rho)
info = s.info()
print(json.dumps({k: info[k] for k in ("hv_groups", "cg_fused", "hv_grid", "nnz")}), "nnz/(mn)", nnz / (m * n))
v = s._vec(np.random.default_rng(0).normal(size=n))
out = s.new_vec()
def timeit(fn, reps):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
t_hv = timeit(lambda: s.ops.hess_apply(v, 0.0, out), 50)
print(f"hess_apply (k_hv_grp + k_hv_out + sync): {t_hv:.1f} us  -> {10*nnz/t_hv/1e3:.0f} GB/s algorithmic")
s.prof_enable(True)
for _ in range(20): s.ops.hess_apply(v, 0.0, out)
pr = s.prof_read()
s.prof_enable(False)
h = pr["hess_apply"]; print(f"  k_hv_grp event-timed: {1e3*h['ms']/h['launches']:.1f} us")
rhs = s.new_vec(); rhs[:n] = -torch.from_numpy(np.random.default_rng(1).normal(size=n)).to(dev); rhs[:n] -= rhs[:n].mean()
def cg():
    return s.ops.cg(gn, rhs, 1e-10, 2 * n)
x, its, res = cg()
t_cg = timeit(cg, 5)
print(f"cg: {its} iterations, {t_cg:.0f} us total, {t_cg/its:.1f} us/iteration")
if os.environ.get("OTB_CG_TRACE") == "1":
    import ctypes as C
    from paper_2603_07156_b200 import _lib
    cnt = C.c_int64()
    _lib.check(_lib.lib.otb_cg_trace(s.ctx, None, 0, C.byref(cnt)))
    buf = (C.c_uint64 * cnt.value)()
    _lib.check(_lib.lib.otb_cg_trace(s.ctx, buf, cnt.value, C.byref(cnt)))
    t = np.array(buf, dtype=np.float64).reshape(-1, 16, 6)          # [cta][iteration][stamp], ns
    iters = min(its, 16) - 1
    t = t[:, 1:iters, :]                                             # skip the first iteration
    names = ("hess_apply", "barrier 1", "column slice", "barrier 2", "vectors")
    d = np.diff(t, axis=2)                                           # [cta][it][5]
    print("CG phases (us, mean over CTAs and iterations; max over CTAs in brackets):")
    for k, nm in enumerate(names):
        print(f"  {nm:13s} {d[:, :, k].mean() / 1e3:7.2f}  [{d[:, :, k].max(axis=0).mean() / 1e3:7.2f}]")
    per_it = np.diff(t[:, :, 0], axis=1)
    print(f"  iteration     {per_it.mean() / 1e3:7.2f}")
