#!/usr/bin/env python
"""Benchmark of the IBSN inner loop on B200 (driver contract: one JSON line).

Metric (BASELINE.json): Newton inner iterations per second, OT solve time to
tol, kernel HBM GB/s vs peak.  Workload: BASELINE config 5 by default — the
largest configuration that fits one GPU (m = n = 50000, C and X 20 GB each,
points uniform in [0,1]^2, C normalised, eta = 1e-2, tol 1e-6), seeded
synthetic data built on the GPU bit-identically to the host numpy recipe
(tests: test_device_cost_construction_is_bitwise_numpy).  ``--config``
selects another configuration.

One *step* = one inner iteration of ``inner_solve`` started from the same
state every step — the product plan X^0 = a b^T after the outer-0 warm start —
through the public API ``inner_solve(..., max_inner=1, mu_k=1e3)``: eval of
the current dual, sparsify, device CG, Armijo line search, candidate
recovery, rounding, Bregman inexact test and KKT metrics.

Keys of the line:
  value         steps/s with inputs resident in HBM (CUDA events, max over ranks)
  e2e           the same public call with pinned HOST C, log X, marginals and
                dual: every step copies them in (40 GB at config 5) and reads
                the dual and report scalars back
  roofline      the dominant kernel (time share of a profiled pass of the same
                steps): algorithmic bytes / CUDA-event launch time vs the
                measured HBM copy peak; per_kernel lists every kernel class
                with its fraction and the ncu DRAM bytes (profiles/traffic.json)
  cpu_baseline  the reference itself (otibsn from baseline/_ref) on the box's
                host cores, on a bounded sample of the same step (a row sample
                for configs 4-5, scaled to Newton it/s), rank 0 at N = 1
  solve         OT solve time to tol: ibsn_solve from device-resident inputs
  secondary     configs 2 and 3 (value + solve) when the default config runs

Multi-GPU (torchrun, one rank per GPU): rows sharded over the ranks, each rank
builds only its own rows of C on its GPU; the length-n vectors are combined by
NCCL all-reduce inside libotb.  The problem is fixed: ``"scaling": "strong"``.

``--impl reference`` times the reference's CPU implementation (oracle/cpu_step.py:
otibsn itself from baseline/_ref, else the numpy port) on the same config,
metric and unit, rank 0 only, all host threads for BLAS.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

if "--impl" in sys.argv and "reference" in sys.argv:
    _threads = str(os.cpu_count() or 1)
    for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "NUMEXPR_NUM_THREADS"):
        os.environ.setdefault(_v, _threads)

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0
DEFAULT_CONFIG = 5
CG_ITERS_HINT = {1: 196, 2: 32, 3: 23, 4: 28, 5: 33}   # GPU arm's CG iterations per step (row-sample size)
METRIC = "newton_inner_iterations_per_s"
UNIT = "newton_it/s"
STEP = "inner_solve(max_inner=1, mu_k=1e3) from the outer-0 warm-started state"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--config", type=int, default=DEFAULT_CONFIG)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--cpu-sample", type=float, default=15.0, help="seconds of CPU reference work (cpu_baseline)")
    p.add_argument("--no-solve", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--secondary", default=None, help="comma list of extra configs (default 2,3 with config 5)")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured", d
    except Exception:
        return HBM_FALLBACK_GBS, "fallback", {}


def config_dict(idx, pts):
    """The ``config`` object, identical in both arms."""
    m, n = len(pts.a), len(pts.b)
    return {"workload": f"BASELINE config {idx}: {pts.name}: m={m} n={n} eta={pts.eta} tol={pts.kkt_tol}",
            "step": STEP,
            "l2": f"inputs larger than L2 (C + log X = {2 * 8 * m * n / 1e6:.0f} MB > 126 MB)"
            if 16 * m * n > 126e6 else f"C + log X = {2 * 8 * m * n / 1e6:.0f} MB (L2-resident)"}


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """Polls NVML every 10 ms while active (SM clock + throttle reasons)."""

    REASONS = {
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
        0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting", 0x1: "gpu_idle",
    }

    def __init__(self, index):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------- CPU reference
def cpu_measure(idx, pts, steps, warmup, budget_s, full_cost=None):
    """Time the CPU step (oracle/cpu_step.py) -> (Newton it/s, description, kind)."""
    from oracle import cpu_step

    st, scale = cpu_step.make_step(pts, full_cost=full_cost, cg_iters=CG_ITERS_HINT.get(idx, 32),
                                   budget_s=budget_s)
    for _ in range(warmup):
        st.step()
    t0 = time.perf_counter()
    for _ in range(steps):
        st.step()
    el = time.perf_counter() - t0
    per_step = el / steps * scale
    return 1.0 / per_step, st.describe(steps, el), st.kind


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import cpu_step
    from paper_2603_07156_b200 import instances

    pts = instances.config_points(args.config, args.seed)
    budget = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    value, sample, kind = cpu_measure(args.config, pts, args.steps, args.warmup, budget)
    cores = cpu_step.blas_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / value, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.config, pts),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": sample + f"; BLAS threads {cores} (numpy ufuncs and scipy sparse "
                                           f"products are single-threaded)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
class Resident:
    """Device-resident problem + the warm-started state of the bench step."""

    def __init__(self, idx, seed, dev, comm, world, rank):
        import torch

        from paper_2603_07156_b200 import instances
        from paper_2603_07156_b200.core import LogPlan, OtProblem, RowShardCost, SolverConfig
        from paper_2603_07156_b200.distributed import row_range
        from paper_2603_07156_b200.session import session_for
        from paper_2603_07156_b200.sinkhorn import warm_start

        self.pts = pts = instances.config_points(idx, seed)
        self.m, self.n = m, n = len(pts.a), len(pts.b)
        self.ld = ld = (n + 31) // 32 * 32
        self.r0, self.r1 = row_range(m, rank, world)
        # C on the GPU: this rank's rows only, bit-identical to the host recipe
        local = instances.device_cost(pts, dev, rows=(self.r0, self.r1), ld=ld, comm=comm)
        self.cost_local = local
        cost = RowShardCost(local, self.r0, m) if comm is not None else local
        self.prob = OtProblem(cost, pts.a, pts.b)
        self.cfg = SolverConfig(eta=pts.eta, kkt_tol=pts.kkt_tol, max_inner=1)
        self.s = s = session_for(self.prob, pts.eta, comm)
        self.X0 = s.new_plan()
        s.ops.init_plan(self.X0)
        self.lp0 = LogPlan.from_padded(self.X0, n)
        gst, _ = warm_start(self.lp0, self.prob, pts.eta, self.cfg.warm_tol,
                            gamma0=torch.zeros(n, dtype=torch.float64, device=dev), comm=comm)
        self.g0 = gst.gamma.clone()
        self.out_plan = s.new_plan()
        self.bufs = (s.new_vec(), s.new_vec())
        self.comm = comm

    def step(self):
        from paper_2603_07156_b200.inner_newton import inner_solve
        from paper_2603_07156_b200.semidual import DualState

        return inner_solve(self.lp0, DualState(self.g0), self.prob, self.cfg, mu_k=1e3, outer_k=0, session=self.s,
                           out_plan=self.out_plan, gamma_bufs=self.bufs)


def timed_steps(res, steps, warmup, world, dev, local):
    import torch
    import torch.distributed as dist

    for _ in range(max(warmup, 3)):
        _, _, rep = res.step()
    torch.cuda.synchronize()
    l0 = res.s.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(steps):
            _, _, rep = res.step()
        ev1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms, res.s.launches() - l0, rep, clocks.summary()


def roofline(res, idx, steps):
    """Profiled pass of the same steps: per-kernel-class CUDA-event times on
    the library's stream, algorithmic bytes, fraction of the
    measured HBM peak, ncu DRAM bytes per launch from profiles/traffic.json."""
    s = res.s
    s.prof_enable(True)
    for _ in range(max(2, min(steps, 5))):
        res.step()
    prof = s.prof_read(reset=True)
    s.prof_enable(False)
    hbm, peak_kind, _ = peaks()
    traffic = {}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"cfg{idx}", {})
        except Exception:
            traffic = {}
    total_ms = sum(v["ms"] for v in prof.values())
    per = {}
    for k, v in prof.items():
        if not v["launches"]:
            continue
        us = 1e3 * v["ms"] / v["launches"]
        bpl = v["bytes"] / v["launches"]
        gbs = bpl / (us * 1e-6) / 1e9 if us > 0 else 0.0
        tr = traffic.get(k)
        dram = (tr / (us * 1e-6) / 1e9) if (tr and us > 0) else None
        per[k] = {"us_per_launch": us, "launches": v["launches"], "bytes_per_launch": bpl, "GB/s": gbs,
                  "frac": gbs / hbm, "share": v["ms"] / total_ms if total_ms else 0.0,
                  "traffic": tr, "dram_GB/s": dram, "dram_frac": (dram / hbm) if dram else None}
    dom = max(per, key=lambda k: per[k]["share"])
    d = per[dom]
    out = {"bound": "hbm", "kernel": dom, "achieved": d["GB/s"], "peak": hbm, "unit": "GB/s", "frac": d["frac"],
           "peak_kind": peak_kind, "traffic": d["traffic"], "bytes_per_launch": d["bytes_per_launch"],
           "us_per_launch": d["us_per_launch"], "time_share": d["share"], "dram_GB/s": d["dram_GB/s"],
           "dram_frac": d["dram_frac"], "per_kernel": per}
    if dom == "hess_apply":
        out["note"] = ("hess_apply streams the dense P_rho (sparsify's dense mode): algorithmic bytes per launch = "
                       "8 m n + 8 (m + 1) + 16 n, one pass over the matrix and no column indices (SURVEY 8(d)'s CSR "
                       "figure 12 nnz + 8(m+1) + 16n applies to the CSR/bitmap formats); dram_GB/s is the ncu DRAM "
                       "bytes per launch over the same time")
    return out


def e2e_measure(res, steps, world, dev, comm):
    """inner_solve through the public API with pinned HOST inputs: every step
    copies C, log X (local rows), the marginals and the dual in, and reads the
    dual and the report scalars back.  The resident step's buffers are freed
    first (the e2e call allocates its own device copies, like a user's)."""
    import torch
    import torch.distributed as dist

    from paper_2603_07156_b200.core import LogPlan, OtProblem, RowShardCost
    from paper_2603_07156_b200.inner_newton import inner_solve
    from paper_2603_07156_b200.semidual import DualState

    n, m, ml = res.n, res.m, res.r1 - res.r0
    C_pin = torch.empty((ml, n), dtype=torch.float64, pin_memory=True)
    C_pin.copy_(res.cost_local[:, :n])
    lx_pin = torch.empty((ml, n), dtype=torch.float64, pin_memory=True)
    lx_pin.copy_(torch.from_numpy(np.log(res.pts.a[res.r0:res.r1]))[:, None]
                 + torch.from_numpy(np.log(res.pts.b))[None, :])
    lx_pin.clamp_(min=-1e6)
    g_pin = res.g0[:n].cpu().pin_memory()
    a, b = res.pts.a, res.pts.b
    cfg = res.cfg
    # free the resident step (its session, plans, CSR) before the e2e copies
    for attr in ("out_plan", "X0", "bufs", "lp0"):
        setattr(res, attr, None)
    res.s.close()
    res.s = None
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    def one():
        # a sharded host cost is wrapped like the device one: rows of this rank
        cost = C_pin if comm is None else RowShardCost(C_pin, res.r0, m)
        hprob = OtProblem(cost, a, b)
        gs, cand, rep = inner_solve(LogPlan(lx_pin), DualState(g_pin), hprob, cfg, mu_k=1e3, outer_k=0, comm=comm)
        return np.asarray(gs.gamma).sum() + rep.objective + rep.kkt

    one()                     # first call: context creation, pinned staging
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([el], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    return {"value": steps / el, "unit": UNIT, "h2d_bytes_per_step": int(8 * ml * n * 2 + 8 * (m + 2 * n)),
            "d2h_bytes_per_step": int(8 * n + 8 * 16), "steps": steps,
            "path": "inner_solve(LogPlan(pinned host log X), DualState(pinned host), OtProblem(pinned host C), "
                    "max_inner=1): H2D of C, log X, marginals, dual; D2H of the dual and the report scalars"}


def solve_measure(prob, pts, comm, world, warm):
    import torch
    import torch.distributed as dist

    from paper_2603_07156_b200.bregman_outer import ibsn_solve
    from paper_2603_07156_b200.core import SolverConfig

    full = SolverConfig(eta=pts.eta, kkt_tol=pts.kkt_tol)
    first = None
    for _ in range(2 if warm else 1):   # the first call grows the CSR capacity and captures the CG graphs
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = ibsn_solve(prob, full, comm=comm)
        e1.record()
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) / 1e3
        if first is None:
            first = sec
    return {"time_s": sec, "first_call_s": first, "outer": r.outer_iters, "newton": r.newton_iters, "cg": r.cg_iters,
            "warm_sweeps": r.warm_sweeps, "objective": r.objective, "kkt": r.kkt,
            "newton_it_per_s": r.newton_iters / sec if sec > 0 else None,
            "from": "device-resident C; ibsn_solve(OtProblem, SolverConfig(eta, kkt_tol)) to kkt < tol"}


def secondary(idx, seed, dev, steps):
    """Value + solve of a smaller config in the same process (N = 1)."""
    import torch

    res = Resident(idx, seed, dev, None, 1, 0)
    ms, launches, rep, _ = timed_steps(res, steps, 3, 1, dev, dev.index)
    roof = roofline(res, idx, steps)
    out = {"config": config_dict(idx, res.pts), "value": steps / (ms / 1e3), "ms_per_step": ms / steps,
           "cg_iters_per_step": rep.cg_iters[-1] if rep.cg_iters else 0,
           "roofline": {k: roof[k] for k in ("kernel", "achieved", "frac", "traffic")},
           "solve": solve_measure(res.prob, res.pts, None, 1, warm=True)}
    res.s.close()
    del res
    torch.cuda.empty_cache()
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    # OTB_NCCL_SELFTEST=1 (under torchrun --nproc-per-node 1): the multi-rank set-up and the NCCL
    # all-reduce call sites with a one-rank communicator, for a one-GPU box
    if world > 1 or os.environ.get("OTB_NCCL_SELFTEST") == "1":
        dist.init_process_group("nccl", device_id=dev)
        from paper_2603_07156_b200.distributed import RowComm

        comm = RowComm()

    res = Resident(args.config, args.seed, dev, comm, world, rank)
    m, n = res.m, res.n
    shard = [res.r0, res.r1]
    ms, launches, rep, clocks = timed_steps(res, args.steps, args.warmup, world, dev, local)
    value = args.steps / (ms / 1e3)
    geometry = res.s.info()
    nnz = rep.nnz[-1] if rep.nnz else 0
    cg_its = rep.cg_iters[-1] if rep.cg_iters else 0
    roof = roofline(res, args.config, args.steps)

    solve = None
    if not args.no_solve:
        solve = solve_measure(res.prob, res.pts, comm, world, warm=True)
    e2e = e2e_measure(res, args.e2e_steps, world, dev, comm) if args.e2e_steps > 0 else None

    sec = {}
    sec_list = args.secondary if args.secondary is not None else ("2,3" if args.config == DEFAULT_CONFIG else "")
    if world == 1 and sec_list:
        del res
        torch.cuda.empty_cache()
        for s_idx in [int(x) for x in sec_list.split(",") if x.strip()]:
            sec[f"config{s_idx}"] = secondary(s_idx, args.seed, dev, 10)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import cpu_step
        from paper_2603_07156_b200 import instances

        pts = instances.config_points(args.config, args.seed)
        v, sample, kind = cpu_measure(args.config, pts, 1, 0, args.cpu_sample)
        cpu = {"value": v, "unit": UNIT, "cores": cpu_step.blas_threads(), "kind": kind,
               "sample": sample + " (BLAS threads as stated; numpy ufuncs and scipy sparse products are "
                                  "single-threaded)"}

    if rank == 0:
        from paper_2603_07156_b200.instances import config_points

        pts = config_points(args.config, args.seed)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.config, pts),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
            "solve": solve,
            "details": {"nnz": nnz, "density": nnz / (m * n), "cg_iters_per_step": cg_its, "geometry": geometry,
                        "row_shard": shard if world > 1 else None},
            "secondary": sec or None,
        }
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
