"""The row-sharded (multi-rank) path on ONE GPU, through a libotb local group.

``distributed.LocalGroup(world)`` runs ``world`` ranks as host threads of one
process, one libotb context and one CUDA stream each, with disjoint row
shards (``row_range``).  Their all-reduces — the same call sites as the NCCL
path: gradient column sums (semidual.py:98-100), d and every CG iteration's
H v (sparsify.py:143-153, krylov.py:68-84), the rounding column sums
(feasibility.py:56-66), the warm-start gamma sweep max/sum (sinkhorn.py:54-58)
— are a fixed-order device sum over the ranks.  The sharded result must match
the one-rank result to the BASELINE tolerance: |d<C,X>|/<C,X> <= 1e-8, equal
outer and Newton counts, CG totals within 5% (reduction orders differ, so CG
can move by a few iterations, as between 1 and 8 BLAS threads in the
reference).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _api():
    import paper_2603_07156_b200 as P

    return P


def _solve_sharded(inst, world, cfg):
    import torch

    P = _api()
    from paper_2603_07156_b200.distributed import LocalGroup

    grp = LocalGroup(world)
    try:
        def body(r, comm):
            prob = P.OtProblem(inst.cost, inst.a, inst.b)
            res = P.ibsn_solve(prob, cfg, comm=comm)
            info = res._session.info()
            rounded = res.rounded_plan            # local rows of the rounded plan
            gam = np.asarray(res.gamma)
            return res, info, rounded, gam

        out = grp.run(body)
        torch.cuda.synchronize()
        return out
    finally:
        grp.close()


@pytest.mark.parametrize("world", [2, 4])
def test_config1_solve_sharded_matches_one_rank(cuda, world):
    P = _api()
    from paper_2603_07156_b200 import instances
    inst = instances.config(1, 0)
    cfg = P.SolverConfig(eta=inst.eta, kkt_tol=inst.kkt_tol)
    one = P.ibsn_solve(P.OtProblem(inst.cost, inst.a, inst.b), cfg)
    outs = _solve_sharded(inst, world, cfg)
    for r, (res, info, rounded, gam) in enumerate(outs):
        assert info["nranks"] == world and info["rank"] == r
        assert info["cg_fused"] == 0            # the persistent CG is single-rank
        assert res.outer_iters == one.outer_iters
        assert res.newton_iters == one.newton_iters
        assert abs(res.cg_iters - one.cg_iters) <= 0.05 * one.cg_iters
        assert abs(res.objective - one.objective) <= 1e-8 * abs(one.objective)
        assert res.kkt < cfg.kkt_tol
        # the replicated dual is bitwise identical on every rank
        assert np.array_equal(gam, np.asarray(outs[0][3]))
    # the shards of the rounded plan form an exactly feasible plan
    X = np.concatenate([o[2] for o in outs], axis=0)
    assert X.shape == inst.cost.shape
    assert np.max(np.abs(X.sum(axis=1) - inst.a)) <= 1e-12
    assert np.max(np.abs(X.sum(axis=0) - inst.b)) <= 1e-12
    assert abs(float((inst.cost * X).sum()) - one.objective) <= 1e-8 * abs(one.objective)


def test_config2_solve_two_ranks(cuda):
    P = _api()
    from paper_2603_07156_b200 import instances
    inst = instances.config(2, 0)
    cfg = P.SolverConfig(eta=inst.eta, kkt_tol=inst.kkt_tol)
    one = P.ibsn_solve(P.OtProblem(inst.cost, inst.a, inst.b), cfg)
    outs = _solve_sharded(inst, 2, cfg)
    for res, info, _, _ in outs:
        assert info["cg_fused"] == 0
        assert (res.outer_iters, res.newton_iters) == (one.outer_iters, one.newton_iters)
        assert abs(res.cg_iters - one.cg_iters) <= 0.05 * one.cg_iters
        assert abs(res.objective - one.objective) <= 1e-8 * abs(one.objective)


def _inner_sharded(C, a, b, lx, g0, eta, world, max_inner=1):
    """inner_solve(max_inner) with the rows of (C, log X) sharded."""
    P = _api()
    from paper_2603_07156_b200.distributed import LocalGroup

    grp = LocalGroup(world)
    try:
        def body(r, comm):
            r0, r1 = comm.row_range(C.shape[0])
            prob = P.OtProblem(C, a, b)
            cfg = P.SolverConfig(eta=eta, kkt_tol=1e-9, max_inner=max_inner)
            st, cand, rep = P.inner_solve(P.LogPlan(lx[r0:r1]), P.DualState(g0), prob, cfg, mu_k=1e3,
                                          outer_k=0, comm=comm)
            return np.asarray(st.gamma)[: C.shape[1]].copy(), rep
        return grp.run(body)
    finally:
        grp.close()


def _inner_one(C, a, b, lx, g0, eta, max_inner=1):
    P = _api()
    cfg = P.SolverConfig(eta=eta, kkt_tol=1e-9, max_inner=max_inner)
    st, cand, rep = P.inner_solve(P.LogPlan(lx), P.DualState(g0), P.OtProblem(C, a, b), cfg, mu_k=1e3, outer_k=0)
    return np.asarray(st.gamma)[: C.shape[1]], rep


def test_newton_step_window_cluster_geometry_two_ranks(cuda):
    """n = 16384 (config 4's column count): the window-cluster hess_apply
    (hv_mode 3) and the cluster-split dense passes, rows sharded over 2."""
    from oracle import otb_oracle as O
    P = _api()
    rng = np.random.default_rng(11)
    m, n, eta = 96, 16384, 1e-2
    x = rng.random((m, 3))
    y = rng.random((n, 3))
    C = ((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)
    C /= C.max()
    a = np.full(m, 1.0 / m)
    b = np.full(n, 1.0 / n)
    lx = O.product_log_plan(a, b)
    g0, _, _ = O.warm_start(lx, C, a, b, eta, 1e-3)
    g1, r1 = _inner_one(C, a, b, lx, g0, eta, max_inner=2)
    outs = _inner_sharded(C, a, b, lx, g0, eta, 2, max_inner=2)
    for g2, r2 in outs:
        assert r2.newton_iters == r1.newton_iters
        assert all(abs(x - y) <= 1 for x, y in zip(r2.cg_iters, r1.cg_iters))
        assert r2.nnz == r1.nnz                 # global kept count, all-reduced
        assert np.max(np.abs(g2 - g1)) <= 1e-9 * max(1.0, np.abs(g1).max())
        assert r2.objective == pytest.approx(r1.objective, rel=1e-10)
    assert np.array_equal(outs[0][0], outs[1][0])


def test_csr_overflow_on_one_rank_only(cuda, monkeypatch):
    """Rank 0's rows keep (almost) every entry, rank 1's few: only rank 0
    outgrows the initial CSR capacity.  The overflow flag rides with the d
    all-reduce, so both ranks redo the pass and the collectives stay matched
    (a rank-local redo would deadlock the group / NCCL)."""
    from oracle import otb_oracle as O
    P = _api()
    rng = np.random.default_rng(5)
    m, n, eta = 64, 512, 1e-2
    C = np.empty((m, n))
    C[: m // 2] = 0.5 + 1e-4 * rng.random((m // 2, n))   # flat rows: P ~ uniform, all kept
    C[m // 2:] = rng.random((m - m // 2, n))              # varied rows: sparse P
    a = rng.random(m) + 0.1
    a /= a.sum()
    b = rng.random(n) + 0.1
    b /= b.sum()
    lx = O.product_log_plan(a, b)
    g0, _, _ = O.warm_start(lx, C, a, b, eta, 1e-3)
    g1, r1 = _inner_one(C, a, b, lx, g0, eta)
    # contexts created from here on start with a tiny CSR (entries)
    monkeypatch.setenv("OTB_CSR_CAP0", str(m * n // 4))
    outs = _inner_sharded(C, a, b, lx, g0, eta, 2)
    for g2, r2 in outs:
        assert r2.nnz == r1.nnz
        assert abs(r2.cg_iters[0] - r1.cg_iters[0]) <= 1
        assert np.max(np.abs(g2 - g1)) <= 1e-9 * max(1.0, np.abs(g1).max())


def test_group_mismatch_fails_loudly(cuda):
    """A rank that raises breaks the group: the others leave their barrier
    with an error instead of hanging."""
    P = _api()
    from paper_2603_07156_b200.distributed import LocalGroup

    from paper_2603_07156_b200 import instances
    inst = instances.config(1, 0)
    grp = LocalGroup(2)
    try:
        def body(r, comm):
            if r == 1:
                raise RuntimeError("rank 1 gives up")
            prob = P.OtProblem(inst.cost, inst.a, inst.b)
            return P.ibsn_solve(prob, P.SolverConfig(eta=inst.eta, kkt_tol=inst.kkt_tol), comm=comm)

        with pytest.raises(RuntimeError, match="rank 1 gives up"):
            grp.run(body, timeout=120)
    finally:
        grp.close()


def test_row_shard_cost_bench_step_two_ranks(cuda):
    """bench.py's sharded set-up on a local group: each rank builds ONLY its
    rows of C on the GPU (instances.device_cost with a row range, the peak
    max-reduced over the ranks), wraps them in RowShardCost (the session uses
    them in place), warm-starts and runs the bench step.  The result equals
    the one-rank step on the full C."""
    import torch

    P = _api()
    from paper_2603_07156_b200 import instances
    from paper_2603_07156_b200.core import LogPlan, RowShardCost
    from paper_2603_07156_b200.distributed import LocalGroup
    from paper_2603_07156_b200.session import session_for
    from paper_2603_07156_b200.sinkhorn import warm_start

    pts = instances.uniform2d_points(1500, 1300, 3)
    m, n = 1500, 1300
    ld = (n + 31) // 32 * 32
    dev = torch.device("cuda", 0)

    def step(cost, comm, r0=0, r1=m):
        prob = P.OtProblem(cost, pts.a, pts.b)
        cfg = P.SolverConfig(eta=pts.eta, kkt_tol=pts.kkt_tol, max_inner=1)
        s = session_for(prob, pts.eta, comm)
        X = s.new_plan()
        s.ops.init_plan(X)
        lp = LogPlan.from_padded(X, n)
        g, _ = warm_start(lp, prob, pts.eta, cfg.warm_tol, gamma0=torch.zeros(n, dtype=torch.float64, device=dev),
                          comm=comm)
        st, cand, rep = P.inner_solve(lp, g, prob, cfg, mu_k=1e3, outer_k=0, comm=comm)
        return st.gamma[:n].cpu().numpy(), rep

    g1, r1 = step(instances.device_cost(pts, dev, ld=ld), None)
    grp = LocalGroup(2)
    try:
        def body(r, comm):
            a0, a1 = comm.row_range(m)
            local = instances.device_cost(pts, dev, rows=(a0, a1), ld=ld, comm=comm)
            return step(RowShardCost(local, a0, m), comm, a0, a1)

        outs = grp.run(body)
    finally:
        grp.close()
    for g2, r2 in outs:
        assert r2.newton_iters == r1.newton_iters == 1
        assert abs(r2.cg_iters[0] - r1.cg_iters[0]) <= 1
        assert np.max(np.abs(g2 - g1)) <= 1e-9 * max(1.0, np.abs(g1).max())
        assert r2.objective == pytest.approx(r1.objective, rel=1e-10)
        assert r2.kkt == pytest.approx(r1.kkt, rel=1e-6)


def _host(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


def _free_device_memory():
    """Destroy the pooled libotb contexts and return torch's cached blocks (the full-size tests
    hold tens of GB each)."""
    import gc

    import torch

    from paper_2603_07156_b200 import _lib, session

    gc.collect()
    for pool in session._CTX_POOL.values():
        while pool:
            _lib.lib.otb_destroy(pool.pop())
    torch.cuda.empty_cache()


@pytest.mark.parametrize("idx,world", [(4, 2), (4, 4), (5, 2)])
def test_full_size_solve_sharded(cuda, idx, world):
    """BASELINE configs 4 and 5 at FULL size (65536 x 16384 and 50000^2, the configurations BASELINE
    shards over 1/2/4/8 GPUs), rows sharded over a local group: each rank builds only its rows of C on the
    device, the window-cluster hess_apply and the cluster-split dense passes run on the shards,
    every length-n all-reduce goes through the group.  ibsn_solve to tol must match the one-rank
    solve: <C,X> to 1e-8, equal outer and Newton counts, CG within 5%, the same dual on every
    rank."""
    import torch

    P = _api()
    from paper_2603_07156_b200 import instances
    from paper_2603_07156_b200.core import RowShardCost
    from paper_2603_07156_b200.distributed import LocalGroup

    pts = instances.config_points(idx, 0)
    m, n = len(pts.a), len(pts.b)
    ld = (n + 31) // 32 * 32
    dev = torch.device("cuda", 0)
    cfg = P.SolverConfig(eta=pts.eta, kkt_tol=pts.kkt_tol)
    _free_device_memory()
    one = P.ibsn_solve(P.OtProblem(instances.device_cost(pts, dev, ld=ld), pts.a, pts.b), cfg)
    ref = (one.outer_iters, one.newton_iters, one.cg_iters, one.objective, one.kkt)
    g1 = _host(one.gamma)[:n].copy()
    one._session.close()
    del one
    _free_device_memory()
    grp = LocalGroup(world)
    try:
        def body(r, comm):
            r0, r1 = comm.row_range(m)
            local = instances.device_cost(pts, dev, rows=(r0, r1), ld=ld, comm=comm)
            res = P.ibsn_solve(P.OtProblem(RowShardCost(local, r0, m), pts.a, pts.b), cfg, comm=comm)
            info = res._session.info()
            out = (res.outer_iters, res.newton_iters, res.cg_iters, res.objective, res.kkt,
                   _host(res.gamma)[:n].copy(), info["nranks"], info["m_loc"], info["hv_mode"])
            res._session.close()
            return out

        outs = grp.run(body, timeout=900)
    finally:
        grp.close()
        _free_device_memory()
    for r, o in enumerate(outs):
        assert o[6] == world and o[7] in (m // world, m // world + 1) and o[8] == 3
        assert (o[0], o[1]) == ref[:2]
        assert abs(o[2] - ref[2]) <= 0.05 * ref[2]
        assert abs(o[3] - ref[3]) <= 1e-8 * abs(ref[3])
        assert o[4] < pts.kkt_tol
        assert np.array_equal(o[5], outs[0][5])
        assert np.max(np.abs(o[5] - g1)) <= 1e-8 * max(1.0, np.abs(g1).max())


_NCCL_SELFTEST = r"""
import json, os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.environ["OTB_REPO"])
import paper_2603_07156_b200 as P
from paper_2603_07156_b200 import instances
from paper_2603_07156_b200.distributed import RowComm

torch.cuda.set_device(0)
inst = instances.config(int(os.environ["OTB_TEST_CONFIG"]), 0)
cfg = P.SolverConfig(eta=inst.eta, kkt_tol=inst.kkt_tol)
one = P.ibsn_solve(P.OtProblem(inst.cost, inst.a, inst.b), cfg)
dist.init_process_group("gloo", rank=0, world_size=1)
os.environ["OTB_NCCL_SELFTEST"] = "1"
res = P.ibsn_solve(P.OtProblem(inst.cost, inst.a, inst.b), cfg, comm=RowComm())
info = res._session.info()
torch.cuda.synchronize()
print(json.dumps({"one": [one.outer_iters, one.newton_iters, one.cg_iters, one.objective, one.kkt],
                  "nccl": [res.outer_iters, res.newton_iters, res.cg_iters, res.objective, res.kkt],
                  "nranks": info["nranks"], "cg_fused": info["cg_fused"],
                  "dgamma": float(np.max(np.abs(np.asarray(res.gamma) - np.asarray(one.gamma))))}))
dist.destroy_process_group()
"""


@pytest.mark.parametrize("config", [1, 2])
def test_nccl_binding_one_rank_selftest(cuda, config):
    """The NCCL transport on a one-GPU box: OTB_NCCL_SELFTEST=1 attaches a
    ONE-rank NCCL communicator (dlopen of the torch-bundled libnccl, unique
    id, ncclCommInitRank) and runs the context through every multi-rank code
    path — per-iteration CG, fallback reductions, every ncclAllReduce call
    site and their CUDA-graph capture.  The solve must equal the one-rank
    solve (same reduction order on one rank: counts equal, objective 1e-8)."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, OTB_REPO=root, OTB_TEST_CONFIG=str(config), MASTER_ADDR="127.0.0.1",
               MASTER_PORT=str(29600 + config))
    env.pop("OTB_NCCL_SELFTEST", None)
    out = subprocess.run([sys.executable, "-c", _NCCL_SELFTEST], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["nranks"] == 2 and r["cg_fused"] == 0      # the context took the multi-rank paths
    assert r["nccl"][0] == r["one"][0] and r["nccl"][1] == r["one"][1]
    assert abs(r["nccl"][2] - r["one"][2]) <= 0.05 * r["one"][2]
    assert abs(r["nccl"][3] - r["one"][3]) <= 1e-8 * abs(r["one"][3])
    assert r["nccl"][4] < (1e-6 if config < 3 else 1e-7)
