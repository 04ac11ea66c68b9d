"""Multi-rank host logic on the CPU (gloo, world_size 2).

The multi-GPU path shards rows of C and X and all-reduces length-n partials
(SURVEY §8(e)).  These tests run two processes with the gloo backend and
check, with the CPU oracle standing in for the per-shard kernels, that:

  * the 128-byte NCCL id broadcast of distributed.RowComm delivers rank 0's
    bytes to every rank;
  * the decomposition libotb implements is exact: every quantity the kernels
    all-reduce (gradient column sums and a.lse; d = P_rho^T a; the H v
    partial of each CG iteration; the rounding column sums and deficit;
    the warm-start column (max, sum) pairs) summed over the two row shards
    reproduces the unsharded Newton step, inexact test and warm start.
"""

import os
import socket

import numpy as np
import pytest

from oracle import otb_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _allreduce(x, op="sum"):
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64).reshape(-1)).clone()
    dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX)
    out = t.numpy()
    return out if np.ndim(x) else float(out[0])


def _sharded_newton_and_test(rank, world, C, a, b, eta, gamma):
    """One Newton step + inexact test with row shards, mirroring the
    all-reduce points of csrc/otb.cu (eval, sparsify, CG, rounding)."""
    from paper_2603_07156_b200.distributed import row_range

    m, n = C.shape
    lo, hi = row_range(m, rank, world)
    Cl, al = C[lo:hi], a[lo:hi]
    lx = O.product_log_plan(a, b)[lo:hi]
    anchor = O.anchor_index(a)

    def evaluate(g):
        P, lse = O.softmax_rows(lx, Cl, g, eta)
        buf = np.concatenate([P.T @ al, [al @ lse]])      # k_eval partials
        buf = _allreduce(buf)
        grad = buf[:n] - b
        value = float(-b @ g + eta * buf[n])
        return P, lse, grad, value

    P, lse, grad, value = evaluate(gamma)
    gnorm = float(np.linalg.norm(grad))
    rho = O.threshold(eta, m, n, gnorm)                   # global m, n
    # local sparsification; the anchor row lives on its owner only
    keep = (P >= rho) & (P > 0.0)
    loc_anchor = anchor - lo if lo <= anchor < hi else -1
    rows = []
    for i in range(hi - lo):
        if i == loc_anchor:
            rows.append((np.arange(n), P[i].copy()))
            continue
        k = keep[i]
        if not k.any():
            j = int(np.argmax(P[i]))
            rows.append((np.array([j]), np.array([1.0])))
            continue
        cols = np.flatnonzero(k)
        rows.append((cols, P[i, cols] / P[i, cols].sum()))
    d = np.zeros(n)
    for i, (c, v) in enumerate(rows):
        np.add.at(d, c, al[i] * v)
    d = _allreduce(d)                                     # sparsify all-reduce

    def hv(v):
        y = np.zeros(n)
        for i, (c, w) in enumerate(rows):
            s = float(w @ v[c])
            np.add.at(y, c, w * (al[i] * s))
        y = _allreduce(y)                                 # per-CG-iteration all-reduce
        return (d * v - y) / eta

    x, its, _ = O.conjugate_gradient(hv, gnorm, -grad, 1e-10)
    slope = float(grad @ x)
    t = 1.0
    while True:
        g2 = gamma + t * x
        P2, lse2, grad2, v2 = evaluate(g2)
        if v2 <= value + 1e-4 * t * slope:
            break
        t *= 0.8
    # inexact test on the local rows
    cand = O.candidate_log(lx, Cl, g2, lse2, al, eta)
    X = np.exp(cand)
    rs = X.sum(axis=1)
    z = np.where(rs > 0, np.minimum(al / rs, 1.0), 1.0)
    F = X * z[:, None]
    col = _allreduce(F.sum(axis=0))
    y = np.where(col > 0, np.minimum(b / col, 1.0), 1.0)
    F = F * y[None, :]
    er = al - F.sum(axis=1)
    buf = _allreduce(np.concatenate([F.sum(axis=0), [np.abs(er).sum()]]))
    ec, deficit = b - buf[:n], buf[n]
    if deficit > 0:
        F = F + np.outer(er, ec) / deficit
    pos = F > 0
    terms = np.where(pos, F * (np.log(np.where(pos, F, 1.0)) - cand), 0.0)
    D = _allreduce(np.array([terms.sum() - F.sum() + X.sum()]))[0]
    return g2, t, its, float(D)


def _sharded_warm(rank, world, C, a, b, eta):
    from paper_2603_07156_b200.distributed import row_range

    m, n = C.shape
    lo, hi = row_range(m, rank, world)
    Cl, al = C[lo:hi], a[lo:hi]
    lx = O.product_log_plan(a, b)[lo:hi]
    gamma = np.zeros(n)
    for sweep in range(1, 1000):
        zeta = O.zeta_sweep(lx, Cl, al, gamma, eta)
        s = lx + (zeta[:, None] + gamma[None, :] - Cl) / eta
        err = float(np.linalg.norm(_allreduce(np.exp(s).sum(axis=0)) - b))
        if err < 1e-3:
            break
        t = lx + (zeta[:, None] - Cl) / eta
        mloc = t.max(axis=0)
        mglob = _allreduce(mloc, "max")                   # all-reduce(max) then (sum)
        sloc = np.exp(t - mglob[None, :]).sum(axis=0)
        sg = _allreduce(sloc)
        gamma = eta * (np.log(b) - (mglob + np.log(sg)))
    drift = gamma.sum() / n
    return gamma - drift, sweep


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_07156_b200.distributed import broadcast_id
        from paper_2603_07156_b200 import instances

        payload = bytes(range(128)) if rank == 0 else None
        got = broadcast_id(payload)
        C, a, b = instances.small_uniform(21, 13, 4)
        res = _sharded_newton_and_test(rank, world, C, a, b, 1e-2, np.zeros(13))
        warm = _sharded_warm(rank, world, C, a, b, 1e-2)
        q.put((rank, got, res, warm))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_match_unsharded():
    import torch.multiprocessing as mp

    from paper_2603_07156_b200 import instances

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    results.sort(key=lambda r: r[0])
    for rank, got, (g2, t, its, D), (wg, sweeps) in results:
        assert got == bytes(range(128))
    # replicated state identical on both ranks
    assert np.array_equal(results[0][2][0], results[1][2][0])
    C, a, b = instances.small_uniform(21, 13, 4)
    lx = O.product_log_plan(a, b)
    gr, tr, itr = O.newton_step(lx, C, a, b, np.zeros(13), 1e-2)
    g2, t, its, D = results[0][2]
    assert t == tr and its == itr
    np.testing.assert_allclose(g2, gr, rtol=1e-10, atol=1e-14)
    r = O.inner(lx, C, a, b, np.zeros(13), 1e-2, mu_k=1e3, scale=13.0, max_inner=1)
    Dref = O.bregman(O.round_plan(np.exp(r.candidate), a, b), r.candidate)
    assert D == pytest.approx(Dref, rel=1e-9, abs=1e-15)
    wg_ref, _, sweeps_ref = O.warm_start(lx, C, a, b, 1e-2, 1e-3)
    np.testing.assert_allclose(results[0][3][0], wg_ref, rtol=1e-10, atol=1e-14)
    assert results[0][3][1] == sweeps_ref
