#!/usr/bin/env python
"""Benchmark of the IBSN inner loop on B200 (driver contract: one JSON line).

Metric: Newton inner iterations per second.  One *step* is one inner
iteration of ``inner_solve`` on BASELINE config 2 (64x64 grid histograms,
m = n = 4096, eta = 1e-2; ``--config`` selects another), started from the
same state every step — the product plan X^0 = a b^T after the outer-0
warm start — through the public API ``inner_solve(..., max_inner=1,
mu_k=1e3)``: eval of the current dual, sparsify, device CG, Armijo line
search, candidate recovery, rounding, Bregman inexact test and KKT metrics.

Lines reported:
  value      steps/s with inputs resident in HBM, CUDA events, max over ranks
  e2e        the same call with pinned HOST inputs (C, log X, marginals,
             dual copied in, dual + candidate plan copied out, every step)
  roofline   the dominant kernel (by time share, from a profiled pass of the
             same steps): algorithmic bytes / event-timed duration vs the
             measured HBM copy peak of MEASURED_PEAKS.json
  cpu_baseline  the CPU oracle (numpy port of the reference) on a bounded
             sample of the same step, rank 0 at N=1
  solve      OT solve time to tol (full ibsn_solve, device-resident inputs)

``--impl reference`` times the reference's CPU algorithm (the oracle port;
the reference is pure Python/numpy) on the same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
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
E2E_DEFAULT = 30


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--config", type=int, default=2)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--e2e-steps", type=int, default=E2E_DEFAULT)
    p.add_argument("--cpu-sample", type=float, default=15.0, help="seconds of CPU oracle work (cpu_baseline)")
    p.add_argument("--no-solve", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured", d
    except Exception:
        return HBM_FALLBACK_GBS, "fallback", {}


def workload_name(idx, inst):
    m, n = len(inst.a), len(inst.b)
    return f"{inst.name}: m={m} n={n} eta={inst.eta} tol={inst.kkt_tol}"


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


# ------------------------------------------------------------- CPU oracle
def oracle_state(inst):
    from oracle import otb_oracle as O

    a, b, C = inst.a, inst.b, inst.cost
    lx = O.product_log_plan(a, b)
    g0, _, _ = O.warm_start(lx, C, a, b, inst.eta, 1e-3)
    return lx, g0


def oracle_step(inst, lx, g0):
    """The bench step on the CPU oracle: inner_solve(max_inner=1, mu_k=1e3)."""
    from oracle import otb_oracle as O

    m, n = inst.cost.shape
    r = O.inner(lx, inst.cost, inst.a, inst.b, g0, inst.eta, 1e3, float(min(m, n)), max_inner=1)
    # inner() rounds and tests; the bench step also reports the KKT metrics
    O.kkt(r.rounded, r.gamma, inst.cost, inst.a, inst.b)
    return r


def cpu_baseline(inst, budget_s):
    lx, g0 = oracle_state(inst)
    t0 = time.perf_counter()
    done = 0
    while True:
        oracle_step(inst, lx, g0)
        done += 1
        el = time.perf_counter() - t0
        if el >= budget_s or done >= 50:
            break
    cores = int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1))
    return {"value": done / el, "unit": "newton_it/s", "cores": cores, "kind": "port",
            "sample": f"{done} bench steps (one inner Newton iteration + inexact test each) of {inst.name} "
                      f"in {el:.1f} s; numpy restatement of the reference (oracle/otb_oracle.py), "
                      f"BLAS threads={cores}, elementwise numpy single-threaded"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2603_07156_b200 import instances

    inst = instances.config(args.config, args.seed)
    lx, g0 = oracle_state(inst)
    for _ in range(args.warmup):
        oracle_step(inst, lx, g0)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_step(inst, lx, g0)
    el = time.perf_counter() - t0
    v = args.steps / el
    cores = int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1))
    line = {
        "impl": "reference", "metric": "newton_inner_iterations_per_s", "value": v, "unit": "newton_it/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config, inst), "step": "inner_solve(max_inner=1, mu_k=1e3)"},
        "cpu_baseline": {"value": v, "unit": "newton_it/s", "cores": cores, "kind": "port",
                         "sample": f"{args.steps} timed steps after {args.warmup} warm-up steps"},
        "e2e": {"value": v, "unit": "newton_it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2603_07156_b200 import instances
    from paper_2603_07156_b200.core import LogPlan, OtProblem, SolverConfig
    from paper_2603_07156_b200.inner_newton import inner_solve
    from paper_2603_07156_b200.semidual import DualState
    from paper_2603_07156_b200.session import session_for
    from paper_2603_07156_b200.sinkhorn import warm_start

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        from paper_2603_07156_b200.distributed import RowComm

        comm = RowComm()

    pts = instances.config_points(args.config, args.seed)
    m, n = len(pts.a), len(pts.b)
    # configs 4-5 (C is 8.6 / 20 GB): C built on the GPU, bit-identical to the
    # host recipe (instances.device_cost), no m x n host array; those runs
    # skip the CPU arm, the e2e line (unless --e2e-steps is given) and the solve
    big = m * n >= 5e8
    if big:
        inst = instances.Instance(pts.name, None, pts.a, pts.b, pts.eta, pts.kkt_tol)
        cost_dev = instances.device_cost(pts, dev, rows=None, ld=(n + 31) // 32 * 32)
    else:
        inst = pts.build()
        cost_dev = torch.from_numpy(inst.cost).to(dev)
    cfg = SolverConfig(eta=inst.eta, kkt_tol=inst.kkt_tol, max_inner=1)
    prob = OtProblem(cost_dev, inst.a, inst.b)
    s = session_for(prob, inst.eta, comm)
    X0 = s.new_plan()
    s.ops.init_plan(X0)
    lp0 = LogPlan.from_padded(X0, n)
    gst, _ = warm_start(lp0, prob, inst.eta, cfg.warm_tol, gamma0=torch.zeros(n, dtype=torch.float64, device=dev),
                        comm=comm)
    g0 = gst.gamma.clone()
    out_plan = s.new_plan()
    bufs = (s.new_vec(), s.new_vec())

    def step():
        return inner_solve(lp0, DualState(g0), prob, cfg, mu_k=1e3, outer_k=0, session=s, out_plan=out_plan,
                           gamma_bufs=bufs)

    def barrier():
        if world > 1:
            dist.barrier()

    nwarm = max(args.warmup, 3)
    for _ in range(nwarm):
        _, _, rep = step()
    torch.cuda.synchronize()
    l0 = s.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(args.steps):
            _, _, rep = step()
        ev1.record()
        torch.cuda.synchronize()
        barrier()
    ms = ev0.elapsed_time(ev1)
    launches = s.launches() - l0
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = args.steps / (ms / 1e3)
    nnz = rep.nnz[-1] if rep.nnz else 0
    cg_its = rep.cg_iters[-1] if rep.cg_iters else 0

    # profiled pass (same steps) -> per-kernel durations for the roofline
    s.prof_enable(True)
    for _ in range(max(3, min(args.steps, 10))):
        step()
    prof = s.prof_read(reset=True)
    s.prof_enable(False)
    hbm, peak_kind, _ = peaks()
    dom = max(prof, key=lambda k: prof[k]["ms"])
    d = prof[dom]
    per_launch_bytes = d["bytes"] / max(d["launches"], 1)
    per_launch_ms = d["ms"] / max(d["launches"], 1)
    achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9 if per_launch_ms > 0 else 0.0
    total_ms = sum(v["ms"] for v in prof.values())
    roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "peak_kind": peak_kind, "traffic": None,
            "bytes_per_launch": per_launch_bytes, "us_per_launch": per_launch_ms * 1e3,
            "time_share": d["ms"] / total_ms if total_ms else None,
            "per_kernel": {k: {"us_per_launch": 1e3 * v["ms"] / max(v["launches"], 1),
                               "launches": v["launches"],
                               "GB/s": (v["bytes"] / (v["ms"] * 1e-3) / 1e9) if v["ms"] else 0.0,
                               "share": v["ms"] / total_ms if total_ms else 0.0}
                           for k, v in prof.items() if v["launches"]}}
    traffic_file = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic_file):
        try:
            tr = json.load(open(traffic_file)).get(f"cfg{args.config}", {}).get(dom)
            roof["traffic"] = tr
        except Exception:
            pass

    # end to end through the public API with pinned host buffers
    m_loc = s.m_loc
    e2e = None
    if big and args.e2e_steps == E2E_DEFAULT:
        args.e2e_steps = 0
    host_cost = (inst.cost if inst.cost is not None else cost_dev.cpu().numpy()) if args.e2e_steps > 0 else None
    C_pin = torch.from_numpy(np.ascontiguousarray(host_cost)).pin_memory() if host_cost is not None else None
    e2e_steps = args.e2e_steps
    if e2e_steps > 0:
        lx_host = np.log(inst.a)[s.row_begin:s.row_end, None] + np.log(inst.b)[None, :]
        lx_pin = torch.from_numpy(np.maximum(lx_host, -1e6)).pin_memory()
        g_pin = g0[:n].cpu().pin_memory()
    torch.cuda.synchronize()

    if e2e_steps > 0:
        def e2e_step():
            # inputs from pinned host memory every step; the step's result read back
            # to the host: the dual (n doubles) and the report's objective / kkt.
            # The candidate plan stays in HBM, as ibsn_solve keeps it.
            hprob = OtProblem(C_pin, inst.a, inst.b)
            gs, cand, rep = inner_solve(LogPlan(lx_pin), DualState(g_pin), hprob, cfg, mu_k=1e3, outer_k=0, comm=comm)
            return np.asarray(gs.gamma).sum() + rep.objective + rep.kkt

        for _ in range(nwarm):      # first call pays context creation and pinned-buffer allocation
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": e2e_steps / e2e_s, "unit": "newton_it/s",
               "h2d_bytes_per_step": int(8 * m_loc * n * 2 + 8 * (m + 2 * n)),
               "d2h_bytes_per_step": int(8 * n + 8 * 16),
               "path": "inner_solve(LogPlan(pinned host), DualState(pinned host), OtProblem(pinned host C), "
                       "max_inner=1): H2D of C, log X, marginals, dual; D2H of the dual and the report scalars "
                       "(the candidate plan stays in HBM, as in ibsn_solve)"}

    solve = None
    if not args.no_solve and not big:
        from paper_2603_07156_b200.bregman_outer import ibsn_solve

        sprob = OtProblem(torch.from_numpy(inst.cost).to(dev), inst.a, inst.b)
        full = SolverConfig(eta=inst.eta, kkt_tol=inst.kkt_tol)
        ibsn_solve(sprob, full, comm=comm)   # warm (session + capacity growth)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = ibsn_solve(sprob, full, comm=comm)
        e1.record()
        torch.cuda.synchronize()
        solve = {"time_s": e0.elapsed_time(e1) / 1e3, "outer": res.outer_iters, "newton": res.newton_iters,
                 "cg": res.cg_iters, "warm_sweeps": res.warm_sweeps, "objective": res.objective, "kkt": res.kkt,
                 "newton_it_per_s": res.newton_iters / (e0.elapsed_time(e1) / 1e3)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not big:
        cpu = cpu_baseline(inst, args.cpu_sample)

    if rank == 0:
        line = {
            "metric": "newton_inner_iterations_per_s", "value": value, "unit": "newton_it/s", "n_gpus": world,
            "steps": args.steps, "warmup": nwarm, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(args.config, inst),
                       "step": "inner_solve(max_inner=1, mu_k=1e3) from the outer-0 warm-started state",
                       "l2": f"inputs larger than L2 (C + log X = {2 * 8 * m * n / 1e6:.0f} MB > 126 MB)",
                       "nnz": nnz, "density": nnz / (m * n), "cg_iters_per_step": cg_its,
                       "geometry": s.info()},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks.summary(), "solve": solve,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
