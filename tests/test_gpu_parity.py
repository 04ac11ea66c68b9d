"""Parity of the CUDA path (libotb via the drop-in Python API) with the
reference, on the golden fixtures made by running the reference
(tests/golden/make_golden.py) and on seeded inputs checked against the CPU
oracle.

Tolerances (stated per test): elementwise quantities agree to a few ulp
(the device uses CUDA's exp/log and other reduction orders than numpy);
iteration counts must agree exactly except CG totals (+-1 per solve, the
reference itself moves by 1 between 1 and 8 BLAS threads);
objectives to the BASELINE gate |d<C,X>|/<C,X> <= 1e-8.
"""

import json

import numpy as np
import pytest

from conftest import GOLDEN, golden, golden_names
from oracle import otb_oracle as O

pytestmark = pytest.mark.gpu


def _api():
    import paper_2603_07156_b200 as P

    return P


def rel(x, y):
    x, y = np.asarray(x, dtype=np.float64), np.asarray(y, dtype=np.float64)
    return float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-300))


def problem_of(g):
    P = _api()
    return P.OtProblem(g["C"], g["a"], g["b"])


# ------------------------------------------------------------------- K1 eval
@pytest.mark.parametrize("name", golden_names("eval"))
def test_eval_matches_reference(cuda, name):
    P = _api()
    g = golden(name)
    prob = problem_of(g)
    eta = float(g["eta"])
    cache = P.compute_p(P.LogPlan(g["logX"]), P.DualState(g["gamma"]), prob, eta)
    assert rel(cache.row_logsumexp, g["lse"]) <= 1e-14
    assert P.semidual_value(cache, None, prob, eta) == pytest.approx(float(g["value"]), rel=1e-14, abs=1e-16)
    grad = P.semidual_gradient(cache, prob)
    assert np.max(np.abs(grad - g["grad"])) <= 1e-14 * max(1.0, np.abs(g["b"]).max())
    assert rel(cache.p, g["P"]) <= 1e-14
    # semidual.py property: 1^T g = 0 up to rounding
    assert abs(grad.sum()) <= 1e-12


# --------------------------------------------------------- K2-K5 sparsify/CG
@pytest.mark.parametrize("name", golden_names("sparsify"))
def test_sparsify_hessian_cg_match_reference(cuda, name):
    P = _api()
    g = golden(name)
    prob = problem_of(g)
    eta = float(g["eta"])
    cache = P.compute_p(P.LogPlan(g["logX"]), P.DualState(g["gamma"]), prob, eta)
    sp = P.sparsify_p(cache, float(g["rho"]), int(g["anchor"]))
    # structure: identical CSR (threshold ties at exactly rho never occur on these inputs)
    assert np.array_equal(sp.row_offsets, g["row_offsets"])
    assert np.array_equal(sp.col_indices, g["col_indices"])
    assert rel(sp.values, g["values"]) <= 1e-14
    assert rel(sp.anchor_row, g["anchor_row"]) <= 1e-14
    op = P.SparseHessianOp(sp)
    assert rel(op.diag_cache, g["d"]) <= 1e-14
    assert rel(op.matvec(g["v"]), g["hv"]) <= 1e-13
    # H 1 = 0 (Theorem 3.2)
    assert np.max(np.abs(op.matvec(np.ones(prob.shape[1])))) <= 1e-12 / eta
    x, it, res = P.cg_solve(op, float(g["grad_norm"]), -cache.grad_t[: prob.shape[1]].cpu().numpy(), 1e-10)
    assert abs(it - int(g["cg_iters"])) <= 1
    assert rel(x, g["cg_x"]) <= 1e-8


def test_sparsify_empty_row_fallback(cuda):
    """rho=0.5 on gen_uniform(6,4,0) at eta=10 sends every
    off-anchor row to the fallback (first argmax kept with value 1)."""
    P = _api()
    g = golden("sparsify_3")
    prob = problem_of(g)
    cache = P.compute_p(P.LogPlan(g["logX"]), P.DualState(g["gamma"]), prob, float(g["eta"]))
    sp = P.sparsify_p(cache, 0.5, int(g["anchor"]))
    assert np.array_equal(sp.row_offsets, g["row_offsets"])
    assert np.array_equal(sp.col_indices, g["col_indices"])
    assert np.all(sp.values == 1.0) and np.array_equal(sp.values, g["values"])


# ------------------------------------------------------------- Newton step
@pytest.mark.parametrize("name", golden_names("newton"))
def test_newton_step_matches_reference(cuda, name):
    P = _api()
    g = golden(name)
    prob = problem_of(g)
    new, t, its = P.newton_step(P.LogPlan(g["logX"]), P.DualState(g["gamma"]), prob, float(g["eta"]))
    assert t == float(g["t"])                       # includes the 0.8^9 backtracking case
    assert abs(its - int(g["cg_iters"])) <= 1
    assert rel(new.gamma, g["gamma_new"]) <= 1e-8


# ---------------------------------------------- K7-K9 candidate / rounding
@pytest.mark.parametrize("name", golden_names("round"))
def test_rounding_divergence_kkt_match_reference(cuda, name):
    P = _api()
    g = golden(name)
    prob = problem_of(g)
    f = P.round_log_plan(P.LogPlan(g["logX"]), prob, gamma=g["gamma"], metrics=True)
    assert rel(f.entries, g["rounded"]) <= 1e-13
    # exact marginals of the rounded plan (SPEC acceptance #9)
    R = f.entries
    assert np.max(np.abs(R.sum(axis=1) - g["a"])) <= 1e-15 * 10
    assert np.max(np.abs(R.sum(axis=0) - g["b"])) <= 1e-15 * 10
    assert f.bregman == pytest.approx(float(g["bregman"]), rel=1e-9, abs=1e-14)
    assert f.objective == pytest.approx(float(g["objective"]), rel=1e-13)
    for key in ("delta_p", "delta_d", "delta_c", "delta_kkt"):
        assert getattr(f, key) == pytest.approx(float(g[key]), rel=1e-6, abs=1e-15)


@pytest.mark.parametrize("name", golden_names("candidate"))
def test_candidate_matches_reference(cuda, name):
    P = _api()
    g = golden(name)
    prob = problem_of(g)
    eta = float(g["eta"])
    st = P.DualState(g["gamma"])
    cache = P.compute_p(P.LogPlan(g["logX"]), st, prob, eta)
    cand = P.plan_candidate_log(P.LogPlan(g["logX"]), cache, st, prob, eta)
    ref = g["candidate"]
    # equal up to the ulp of the row log-normaliser
    assert np.max(np.abs(cand.log_entries - ref)) <= 4e-16 * max(1.0, np.abs(ref).max())


# --------------------------------------------------------------- warm start
@pytest.mark.parametrize("name", golden_names("warm"))
def test_warm_start_matches_reference(cuda, name):
    P = _api()
    g = golden(name)
    prob = problem_of(g)
    st, zeta = P.warm_start(P.LogPlan(g["logX"]), prob, float(g["eta"]), 1e-3)
    assert rel(st.gamma, g["gamma"]) <= 1e-12
    assert rel(zeta, g["zeta"]) <= 1e-12
    assert abs(st.gamma.sum()) <= 1e-15 * max(1.0, np.abs(st.gamma).sum())


# ------------------------------------------------------------- inner solve
@pytest.mark.parametrize("name", golden_names("inner"))
def test_inner_solve_matches_reference(cuda, name):
    P = _api()
    g = golden(name)
    prob = problem_of(g)
    cfg = P.SolverConfig(eta=float(g["eta"]), kkt_tol=1e-9)
    st, cand, rep = P.inner_solve(P.LogPlan(g["logX"]), P.DualState(g["gamma0"]), prob, cfg, mu_k=1e-4, outer_k=0)
    assert rep.newton_iters == int(g["newton_iters"])
    assert rep.stop_reason.value == str(g["stop"])
    assert abs(rep.cg_iters_total - int(g["cg_iters_total"])) <= rep.newton_iters
    assert list(rep.step_sizes) == list(g["steps"])
    assert rel(st.gamma, g["gamma"]) <= 1e-8
    assert np.max(np.abs(cand.log_entries - g["candidate"])) <= 1e-7


# --------------------------------------------------------------- full solve
@pytest.mark.parametrize("name", golden_names("solve"))
def test_ibsn_solve_matches_reference(cuda, name):
    P = _api()
    g = golden(name)
    prob = problem_of(g)
    res = P.ibsn_solve(prob, P.SolverConfig(eta=float(g["eta"]), kkt_tol=float(g["kkt_tol"])))
    assert res.outer_iters == int(g["outer_iters"])
    assert res.objective == pytest.approx(float(g["objective"]), rel=1e-8)
    assert res.kkt < float(g["kkt_tol"])
    # Newton counts: equal while the Armijo comparison L(trial) <= L0 + sigma t
    # slope is decided above rounding.  Deep in these tiny solves (mu_k ~ 5e-8,
    # slope ~ 1e-19) L changes by less than ulp(L) and the accept/reject
    # decision is set by summation-order noise in L — in the reference too
    # (tools/trace_solve.py shows identical L to 17 digits).  Compare counts
    # over the outers whose steps stay above that floor.
    ref_inner = list(g["inner_total"])
    ours = [r.inner_total for r in res.trajectory.records]
    agree = 0
    while agree < len(ref_inner) and ours[agree] == ref_inner[agree]:
        agree += 1
    assert agree >= min(len(ref_inner), 10), (ours, ref_inner)
    # CG counts at ||g|| ~ 1e-13 also move with summation order; the 5% CG gate
    # of BASELINE.md is enforced on the BASELINE configs below, 10% here.
    cg_ref = int(g["cg_total"][agree - 1])
    assert abs(res.trajectory.records[agree - 1].cg_total - cg_ref) <= max(2, 0.10 * cg_ref)
    R = res.rounded_plan
    assert rel(R, g["rounded"]) <= 1e-6
    assert np.max(np.abs(R.sum(axis=1) - g["a"])) <= 1e-12
    assert np.max(np.abs(R.sum(axis=0) - g["b"])) <= 1e-12
    assert abs(res.gamma.sum()) <= 1e-8 * max(1.0, np.linalg.norm(res.gamma))


@pytest.mark.parametrize("idx", [1, 2])
def test_baseline_config_end_to_end(cuda, idx):
    """BASELINE configs 1 and 2 (seed 0) against the reference's own run:
    <C,X> to 1e-8 relative, outer and Newton counts equal, CG within 5%."""
    P = _api()
    from paper_2603_07156_b200 import instances

    ref = json.loads((GOLDEN / "config_scalars.json").read_text())[f"cfg{idx}"]
    inst = instances.config(idx, 0)
    res = P.ibsn_solve(P.OtProblem(inst.cost, inst.a, inst.b), P.SolverConfig(eta=inst.eta, kkt_tol=inst.kkt_tol))
    assert res.objective == pytest.approx(ref["objective"], rel=1e-8)
    assert res.outer_iters == ref["outer_iters"]
    assert res.newton_iters == ref["newton_total"]
    assert abs(res.cg_iters - ref["cg_total"]) <= 0.05 * ref["cg_total"]
    assert res.kkt < inst.kkt_tol
    objs = [r.objective for r in res.trajectory.records]
    np.testing.assert_allclose(objs, ref["objectives"], rtol=1e-8)


# ------------------------------------------------- oracle-checked seeded cases
@pytest.mark.parametrize("m,n,eta", [(1, 5, 1e-2), (7, 1, 1e-2), (37, 29, 5e-2), (257, 131, 1e-2),
                                     (64, 9000, 1e-2), (40, 16400, 1e-2), (9, 50001, 1e-2), (24, 60000, 1e-2),
                                     (12, 70000, 1e-2), (6, 131072, 1e-2)])
def test_step_pipeline_vs_oracle(cuda, m, n, eta):
    """Ragged / odd / cluster-split (n > 10240; 60000 columns = clusters of 8)
    / window-cluster geometries: eval, one Newton step and the inexact test
    vs the oracle.  n > 65536 (up to 131072 = 16 windows of 8192 columns) runs
    on the window-cluster formats, which store no 16-bit column indices."""
    P = _api()
    from paper_2603_07156_b200 import instances

    C, a, b = instances.small_uniform(m, n, 11 + m)
    prob = P.OtProblem(C, a, b)
    lx = O.product_log_plan(a, b)
    gam0 = np.zeros(n)
    cache = P.compute_p(P.LogPlan(lx), P.DualState(gam0), prob, eta)
    Pm, lse = O.softmax_rows(lx, C, gam0, eta)
    assert rel(cache.row_logsumexp, lse) <= 1e-14
    assert np.max(np.abs(P.semidual_gradient(cache, prob) - O.gradient(Pm, a, b))) <= 1e-15
    if n > 1:
        new, t, its = P.newton_step(P.LogPlan(lx), P.DualState(gam0), prob, eta)
        gr, tr, itr = O.newton_step(lx, C, a, b, gam0, eta)
        assert t == tr and abs(its - itr) <= 1
        assert rel(new.gamma, gr) <= 1e-8
    f = P.round_log_plan(P.LogPlan(lx + 0.1), prob, gamma=gam0)
    R = O.round_plan(np.exp(O.clamp_log_plan(lx + 0.1)), a, b)
    assert f.bregman == pytest.approx(O.bregman(R, O.clamp_log_plan(lx + 0.1)), rel=1e-9, abs=1e-15)
    assert f.objective == pytest.approx(float((C * R).sum()), rel=1e-12)


def test_underflow_zeros_excluded(cuda):
    """Exact-zero P entries (exp underflow) are never stored (sparsify.py:99-100)."""
    P = _api()
    from paper_2603_07156_b200 import instances

    C, a, b = instances.small_uniform(30, 40, 3)
    prob = P.OtProblem(C, a, b)
    eta = 1e-4                       # logits span ~1e4 -> many exact zeros
    lx = O.product_log_plan(a, b)
    cache = P.compute_p(P.LogPlan(lx), P.DualState(np.zeros(40)), prob, eta)
    Pm, _ = O.softmax_rows(lx, C, np.zeros(40), eta)
    assert (Pm == 0).any()
    sp = P.sparsify_p(cache, 0.0, int(np.argmax(a)))
    ref = O.threshold_rows(Pm, 0.0, int(np.argmax(a)))
    assert np.array_equal(sp.row_offsets, ref.row_ptr)
    assert np.array_equal(sp.col_indices, ref.cols)
    assert np.array_equal(sp.anchor_row == 0, ref.anchor_row == 0)


def test_error_mapping(cuda):
    """Reference exception classes come back through the status codes."""
    P = _api()
    from paper_2603_07156_b200 import errors, instances

    C, a, b = instances.small_uniform(10, 8, 0)
    with pytest.raises(errors.InvalidCost):
        P.LogPlan(np.full((2, 2), np.nan))
    bad = C.copy()
    bad[0, 0] = np.nan
    with pytest.raises(errors.InvalidCost):
        P.ibsn_solve(P.OtProblem(bad, a, b), P.SolverConfig(eta=1e-2))
    prob = P.OtProblem(C, a, b)
    cache = P.compute_p(P.initial_plan(prob), P.DualState(np.zeros(8)), prob, 1e-2)
    op = P.SparseHessianOp(P.sparsify_p(cache, 0.0, int(np.argmax(a))))
    with pytest.raises(errors.InconsistentSystem):
        P.cg_solve(op, 0.0, np.ones(8))
    # rhs = 0 -> 0 iterations
    x, it, res = P.cg_solve(op, 1.0, np.zeros(8))
    assert it == 0 and res == 0.0 and not x.any()


# ------------------------------------------------ fixed-divisor fast division
@pytest.mark.parametrize("y", [1e-2, 5e-3, 1e-3, 0.7310585786300049, 3.0, 1e-17, 2.5e-290, 1e300, 1.0, 2.0 ** 600,
                               2.0 ** -1020, -3.7, 5e-320, 0.0, np.inf])
def test_fast_division_is_correctly_rounded(cuda, y):
    """The kernels divide by eta / row sums / the rounding deficit through a
    reciprocal + one FMA residual step (csrc/common.cuh Divider); it must give
    numpy's x / y bit for bit, including zeros, signs, infinities and NaN."""
    import torch

    from paper_2603_07156_b200 import _lib

    rng = np.random.default_rng(11)
    with np.errstate(all="ignore"):   # y = inf: inf * 0 in the multiples of y
        parts = [
            rng.standard_normal(200_000) * 10.0 ** rng.uniform(-30, 30, 200_000),
            rng.uniform(-1.0, 1.0, 100_000),
            np.exp(rng.uniform(-745, 709, 50_000)),
            np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 1.7e308, 2.2250738585072014e-308]),
            y * np.arange(-1000, 1000, dtype=np.float64),
            np.nextafter(y * np.arange(1, 1000, dtype=np.float64), np.inf),
            # every power of two and its neighbours: the edges of the fast path's range
            2.0 ** np.arange(-1074, 1024, dtype=np.float64),
            np.nextafter(2.0 ** np.arange(-1074, 1024, dtype=np.float64), np.inf),
            -np.nextafter(2.0 ** np.arange(-1074, 1024, dtype=np.float64), 0.0),
        ]
    x = np.concatenate(parts)
    xd = torch.from_numpy(x).cuda()
    out = torch.empty_like(xd)
    _lib.check(_lib.lib.otb_selftest_div(xd.data_ptr(), x.size, float(y), out.data_ptr()))
    got = out.cpu().numpy()
    with np.errstate(all="ignore"):
        want = x / y
    bad = got.view(np.uint64) != want.view(np.uint64)
    bad &= ~(np.isnan(got) & np.isnan(want))
    assert not bad.any(), (x[bad][:5], got[bad][:5], want[bad][:5])


@pytest.mark.parametrize("m,n,env", [(300, 4100, None), (200, 9000, None), (120, 16400, None),
                                     (310, 4000, "OTB_HV_STAGED"), (190, 9000, "OTB_HV_WC"),
                                     (70, 50001, None), (20, 70000, None)])
def test_hess_apply_deterministic_and_matches_oracle(cuda, monkeypatch, m, n, env):
    """hess_apply (cp.async bitmap, TMA-staged bitmap, warp-group and
    window-cluster variants) is bitwise reproducible run to run and matches
    the oracle's H v (sparsify.py:151-153).  `env` opts into a variant the
    library would not pick for this shape (read when the context is made)."""
    if env:
        monkeypatch.setenv(env, "1")
    P = _api()
    from paper_2603_07156_b200 import instances

    C, a, b = instances.small_uniform(m, n, 5 + n)
    prob = P.OtProblem(C, a, b)
    eta = 1e-2
    lx = O.product_log_plan(a, b)
    rng = np.random.default_rng(n)
    gam = rng.standard_normal(n) * 1e-3
    cache = P.compute_p(P.LogPlan(lx), P.DualState(gam), prob, eta)
    rho = eta * float(np.linalg.norm(P.semidual_gradient(cache, prob))) / (m * n)
    op = P.SparseHessianOp(P.sparsify_p(cache, rho, int(np.argmax(a))))
    v = rng.standard_normal(n)
    h1, h2 = op.matvec(v), op.matvec(v)
    assert np.array_equal(h1.view(np.uint64), h2.view(np.uint64))
    Pm, _ = O.softmax_rows(lx, C, gam, eta)
    ref = O.SparseHessian(O.threshold_rows(Pm, rho, int(np.argmax(a))), a, eta).matvec(v)
    assert rel(h1, ref) <= 1e-12


@pytest.mark.parametrize("m,n", [(97, 1203), (41, 9100)])
def test_sparsify_from_stored_p_equals_recomputed(cuda, monkeypatch, m, n):
    """sparsify streams the P stored by the eval of the same gamma; with
    OTB_STORE_P=0 it recomputes P from C and log X.  Both give the same CSR
    bit for bit (the stored P is the reference's shifted / row_sum)."""
    P = _api()
    from paper_2603_07156_b200 import instances

    C, a, b = instances.small_uniform(m, n, 3 + n)
    lx = O.product_log_plan(a, b)
    gam = np.random.default_rng(m).standard_normal(n) * 1e-3
    outs = []
    for store in ("1", "0"):
        monkeypatch.setenv("OTB_STORE_P", store)
        prob = P.OtProblem(C.copy(), a, b)          # fresh problem -> fresh context (env read at creation)
        cache = P.compute_p(P.LogPlan(lx), P.DualState(gam), prob, 1e-2)
        rho = 1e-2 * float(np.linalg.norm(P.semidual_gradient(cache, prob))) / (m * n)
        sp = P.sparsify_p(cache, rho, int(np.argmax(a)))
        outs.append((sp.row_offsets, sp.col_indices, sp.values, sp.anchor_row))
    for x, y in zip(*outs):
        assert np.array_equal(np.asarray(x).view(np.uint64) if np.asarray(x).dtype == np.float64 else x,
                              np.asarray(y).view(np.uint64) if np.asarray(y).dtype == np.float64 else y)


def test_fast_log_accuracy(cuda):
    """The device log of the Bregman sum (common.cuh log_fast) is within 2
    ulp of numpy's log over the positive doubles, and defers to CUDA's log
    for zero, subnormals, negatives, inf and NaN."""
    import torch

    from paper_2603_07156_b200 import _lib

    rng = np.random.default_rng(5)
    x = np.concatenate([np.exp(rng.uniform(-744, 709, 400_000)), rng.uniform(0.5, 2.0, 200_000),
                        1.0 + rng.standard_normal(50_000) * 1e-9,
                        # |s| largest at m = sqrt(2)^-+, the series' truncation edge, at many exponents
                        np.sqrt(2.0) * (1.0 + rng.uniform(-1e-3, 1e-3, 50_000)) * 2.0 ** rng.integers(-1000, 1000, 50_000),
                        np.array([1.0, 2.0, 0.5, np.sqrt(2.0), 1e-310,
                                                                               0.0, -1.0, np.inf, np.nan])])
    xd = torch.from_numpy(x).cuda()
    out = torch.empty_like(xd)
    _lib.check(_lib.lib.otb_selftest_log(xd.data_ptr(), x.size, out.data_ptr()))
    got = out.cpu().numpy()
    with np.errstate(all="ignore"):
        want = np.log(x)
    fin = np.isfinite(want) & (want != 0)
    ulp = np.abs(got[fin] - want[fin]) / np.spacing(np.abs(want[fin]))
    assert ulp.max() <= 2.0, (ulp.max(), x[fin][np.argmax(ulp)])
    assert got[x == 1.0][0] == 0.0
    assert np.isneginf(got[x == 0.0]).all() and np.isnan(got[x == -1.0]).all() and np.isposinf(got[x == np.inf]).all()


@pytest.mark.parametrize("name", golden_names("eot"))
def test_eot_single_solve_matches_reference(cuda, name):
    """eot_single_solve on the device against the reference's run."""
    P = _api()
    g = golden(name)
    res = P.eot_single_solve(problem_of(g), P.SolverConfig(eta=float(g["eta"]), kkt_tol=float(g["kkt_tol"])))
    rec = res.trajectory.records[-1]
    # Armijo at the rounding floor: when sigma * slope of a reference step is
    # below one ulp of the objective, its accept/backtrack decision is set by
    # the last bit of a 576-term sum (eot_1: slope -2e-19 on f = 2.9e-2), so
    # the step counts may differ; the gradient target and objective may not.
    m, n = g["C"].shape
    lx = np.zeros((m, n))
    gam, _, _ = O.warm_start(lx, g["C"], g["a"], g["b"], float(g["eta"]), 1e-3)
    ref = O.inner(lx, g["C"], g["a"], g["b"], gam, float(g["eta"]), 0.0, float(min(m, n)),
                  grad_target=float(g["kkt_tol"]))
    assert ref.newton_iters == int(g["newton_iters"])
    floor = any(1e-4 * abs(st.slope) < np.spacing(v) for st, v in zip(ref.steps, ref.values))
    if floor:
        assert int(g["newton_iters"]) <= rec.inner_total <= int(g["newton_iters"]) + 4
    else:
        assert rec.inner_total == int(g["newton_iters"])
        assert abs(rec.cg_total - int(g["cg_total"])) <= max(1, rec.inner_total)
    assert res.objective == pytest.approx(float(g["objective"]), rel=1e-8)      # the BASELINE gate
    assert res.kkt == pytest.approx(float(g["kkt"]), rel=1e-6)
    assert rel(res.rounded_plan, g["rounded"]) <= 1e-7
    assert rec.grad_norm <= float(g["kkt_tol"])


@pytest.mark.parametrize("name", golden_names("ibsink"))
def test_ibsink_solve_matches_reference(cuda, name):
    """ibsink_solve (Sinkhorn sweeps as the inner solver) on the device
    against the reference's run: same outers, same sweep counts per outer,
    objectives within the BASELINE gate."""
    P = _api()
    g = golden(name)
    cfg = P.SolverConfig(eta=float(g["eta"]), kkt_tol=float(g["kkt_tol"]), max_outer=int(g["max_outer"]))
    res = P.ibsink_solve(problem_of(g), cfg)
    assert res.outer_iters == int(g["outer_iters"])
    assert [r.inner_total for r in res.trajectory.records] == list(g["inner_total"])
    np.testing.assert_allclose([r.objective for r in res.trajectory.records], g["traj_objective"], rtol=1e-8)
    assert rel(res.rounded_plan, g["rounded"]) <= 1e-8


@pytest.mark.parametrize("kind", ["uniform2d", "gmm", "colour", "grid"])
def test_device_cost_construction_is_bitwise_numpy(cuda, kind):
    """instances.device_cost (otb_sq_dist + otb_scale_cost) builds the cost
    matrix on the GPU bit-identically to the host numpy recipe, including a
    row sub-range into a padded buffer (one rank's shard)."""
    import torch

    from paper_2603_07156_b200 import instances as I

    pts = {"uniform2d": lambda: I.uniform2d_points(300, 211, 4), "gmm": lambda: I.gmm_points(150, 170, 5),
           "colour": lambda: I.colour_points(200, 97, 6), "grid": lambda: I.grid_points(16, 7)}[kind]()
    host = pts.build().cost
    dev = I.device_cost(pts, torch.device("cuda", 0)).cpu().numpy()
    assert np.array_equal(dev.view(np.uint64), host.view(np.uint64))
    m, n = host.shape
    r0, r1 = m // 3, m // 3 + 17
    part = I.device_cost(pts, torch.device("cuda", 0), rows=(r0, r1), ld=(n + 31) // 32 * 32)
    if pts.normalised:   # without a comm a shard normalises by its own peak
        want = I.normalise(I.sq_dist(pts.x[r0:r1], pts.y))
    else:
        want = host[r0:r1]
    assert np.array_equal(part.cpu().numpy().view(np.uint64), want.view(np.uint64))


def test_config3_first_newton_step_vs_oracle(cuda):
    """BASELINE config 3 (10000^2, cluster-split rows, warp-group hess_apply):
    the first Newton step from X0 = a b^T, gamma = 0 against the CPU oracle
    (~30 s on the host), plus size-independent properties at full size:
    1^T g = 0, H_rho 1 = 0, determinism of eval and hess_apply."""
    import torch

    P = _api()
    from paper_2603_07156_b200 import instances
    from paper_2603_07156_b200.session import session_for

    inst = instances.config(3, 0)
    m, n = inst.cost.shape
    dev = torch.device("cuda", 0)
    prob = P.OtProblem(torch.from_numpy(inst.cost).to(dev), inst.a, inst.b)
    s = session_for(prob, inst.eta)
    X0 = s.new_plan()
    s.ops.init_plan(X0)
    g = s.new_vec()
    v1, gn1 = s.ops.eval(X0, g)
    grad = s.new_vec()
    v2, gn2 = s.ops.eval(X0, g, grad_out=grad)
    assert (v1, gn1) == (v2, gn2)                                       # deterministic
    assert abs(float(grad[:n].sum())) <= 1e-13                          # 1^T g = 0
    rho = inst.eta * gn1 / (m * n)
    s.ops.sparsify(X0, g, rho)
    ones = s._vec(np.ones(n))
    out = s.new_vec()
    s.ops.hess_apply(ones, 0.0, out)
    assert float(out[:n].abs().max()) <= 1e-10 / inst.eta                # H_rho 1 = 0
    h1 = s.new_vec()
    s.ops.hess_apply(ones, 0.0, h1)
    assert torch.equal(out, h1)
    g2 = s.new_vec()
    s.ops.eval(X0, g)
    r = s.ops.newton_step(X0, g, g2, 1e-4, 0.8, 1e-10, None)
    lx = np.log(inst.a)[:, None] + np.log(inst.b)[None, :]
    gr, tr, itr = O.newton_step(lx, inst.cost, inst.a, inst.b, np.zeros(n), inst.eta)
    assert float(r.t) == tr and abs(int(r.cg_iters) - itr) <= 1
    assert rel(g2[:n].cpu().numpy(), gr) <= 1e-8


def test_config2_solve_rounded_marginals_and_determinism(cuda):
    """BASELINE config 2 at full size: the rounded plan meets both marginals
    to 1e-12 (SPEC acceptance #9) and two solves give identical bits."""
    P = _api()
    from paper_2603_07156_b200 import instances

    inst = instances.config(2, 0)
    cfg = P.SolverConfig(eta=inst.eta, kkt_tol=inst.kkt_tol)
    r1 = P.ibsn_solve(P.OtProblem(inst.cost, inst.a, inst.b), cfg)
    r2 = P.ibsn_solve(P.OtProblem(inst.cost, inst.a, inst.b), cfg)
    assert r1.objective == r2.objective and r1.cg_iters == r2.cg_iters
    R = r1.rounded_plan
    assert np.max(np.abs(R.sum(axis=1) - inst.a)) <= 1e-12
    assert np.max(np.abs(R.sum(axis=0) - inst.b)) <= 1e-12
    assert R.min() >= -1e-18        # e_r e_c^T / deficit can carry rounding-level negatives, in the reference too


def test_newton_step_csr_overflow_retry_is_identical(cuda, monkeypatch):
    """The single-synchronisation Newton step (sparsify, CG, slope and the
    t = 1 trial launched back to back) detects a CSR capacity overflow only
    after the trial: it grows the CSR, re-evaluates at gamma_in and repeats.
    Starting from a tiny capacity must give bit-identical results to a
    context whose capacity suffices from the start."""
    import torch

    P = _api()
    from paper_2603_07156_b200 import instances

    inst = instances.uniform2d_points(701, 899, seed=3, eta=2e-2).build()
    X = np.log(np.outer(inst.a, inst.b))
    outs = []
    for cap0 in ("4096", None):            # fresh contexts (shape used nowhere else)
        if cap0 is None:
            monkeypatch.delenv("OTB_CSR_CAP0", raising=False)
        else:
            monkeypatch.setenv("OTB_CSR_CAP0", cap0)
        prob = P.OtProblem(torch.from_numpy(inst.cost.copy()).cuda(), inst.a, inst.b)
        gam, _ = P.warm_start(P.LogPlan(X), prob, inst.eta, 1e-3, gamma0=np.zeros(899))
        new, t, its = P.newton_step(P.LogPlan(X), gam, prob, inst.eta)
        g = new.gamma.cpu().numpy() if hasattr(new.gamma, "cpu") else np.asarray(new.gamma)
        outs.append((g, t, its, prob))     # keep the problem (and its context) alive
    monkeypatch.delenv("OTB_CSR_CAP0", raising=False)
    assert outs[0][1] == outs[1][1] and outs[0][2] == outs[1][2]
    assert np.array_equal(outs[0][0], outs[1][0])


@pytest.mark.parametrize("m,n", [(48, 6000), (40, 10240), (32, 16400)])
def test_rounding_metrics_wide_rows_match_oracle(cuda, m, n):
    """Pass C's KKT metrics on rows of more than 6 slices take the row
    c-transform from pass A (k_test_c kZetaFromA), and above 10240 columns
    the row is split over a cluster (cl = 2 at 16400): rounded plan,
    Bregman divergence, objective and KKT residuals against the oracle."""
    P = _api()
    rng = np.random.default_rng(n)
    x = rng.random((m, 2))
    y = rng.random((n, 2))
    C = ((x[:, None, :] - y[None, :, :]) ** 2).sum(axis=2)
    C /= C.max()
    a = rng.random(m) + 0.1
    a /= a.sum()
    b = rng.random(n) + 0.1
    b /= b.sum()
    gamma = rng.standard_normal(n) * 1e-3
    logX = np.log(np.outer(a, b)) + rng.standard_normal((m, n)) * 0.3
    prob = P.OtProblem(C, a, b)
    f = P.round_log_plan(P.LogPlan(logX), prob, gamma=gamma, metrics=True)
    R = O.round_plan(np.exp(logX), a, b)
    assert rel(f.entries, R) <= 1e-13
    assert f.bregman == pytest.approx(O.bregman(R, logX), rel=1e-9, abs=1e-14)
    assert f.objective == pytest.approx(float((C * R).sum()), rel=1e-12)
    k = O.kkt(R, gamma, C, a, b)
    for key in ("delta_p", "delta_d", "delta_c", "delta_kkt"):
        assert getattr(f, key) == pytest.approx(float(k[key]), rel=1e-6, abs=1e-15)


def test_fast_exp_is_cuda_exp(cuda):
    """The dense passes' branch-free exp (common.cuh exp_fast, with exp() for
    |x| >= 708.4) returns CUDA exp()'s bits on every input, including the
    range edges, subnormal results, infinities and NaN."""
    import torch

    from paper_2603_07156_b200 import _lib

    rng = np.random.default_rng(17)
    x = np.concatenate([rng.uniform(-750, 710, 500_000), rng.standard_normal(200_000) * 30,
                        rng.uniform(-1e-3, 1e-3, 100_000), np.linspace(-709.0, -707.0, 20_001),
                        np.linspace(707.0, 709.9, 20_001), -(2.0 ** np.arange(-1074, 11, dtype=np.float64)),
                        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 709.782712893384, -745.1332191019412])])
    xd = torch.from_numpy(x).cuda()
    out = torch.empty(2 * x.size, dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib.otb_selftest_exp(xd.data_ptr(), x.size, out.data_ptr()))
    got = out.cpu().numpy()
    fast, ref = got[: x.size], got[x.size:]
    same = (fast.view(np.uint64) == ref.view(np.uint64)) | (np.isnan(fast) & np.isnan(ref))
    assert same.all(), (x[~same][:5], fast[~same][:5], ref[~same][:5])
    with np.errstate(all="ignore"):
        fin = np.isfinite(ref) & (ref > 1e-300)
        assert np.max(np.abs(ref[fin] - np.exp(x[fin])) / np.spacing(np.exp(x[fin]))) <= 2.0


def test_table_exp_log_accuracy(cuda):
    """The streaming passes' table-driven exp (<= 0.51 ulp by construction)
    and log (<= 1.5 ulp) with their fallbacks (exp() for |x| >= 707 and NaN,
    log_fast near 1 and for special inputs), against numpy on the range
    edges, subnormal results, special values and the near-1 switch."""
    import torch

    from paper_2603_07156_b200 import _lib

    rng = np.random.default_rng(23)
    x = np.concatenate([rng.uniform(-750, 710, 400_000), rng.standard_normal(200_000) * 30,
                        rng.uniform(-1e-3, 1e-3, 100_000), np.linspace(-708.0, -706.0, 20_001),
                        np.linspace(706.0, 708.0, 20_001), -(2.0 ** np.arange(-1074, 11, dtype=np.float64)),
                        np.exp(rng.uniform(-700, 700, 200_000)), 1.0 + rng.uniform(-0.05, 0.05, 100_000),
                        2.0 ** rng.integers(-1070, 1020, 20_000) * rng.uniform(1, 2, 20_000),
                        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 1.0, 0.984375, 1.015625,
                                  709.782712893384, -745.1332191019412, -1e6])])
    xd = torch.from_numpy(x).cuda()
    out = torch.empty(2 * x.size, dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib.otb_selftest_tab(xd.data_ptr(), x.size, out.data_ptr()))
    got = out.cpu().numpy()
    e, lg = got[: x.size], got[x.size:]
    with np.errstate(all="ignore"):
        we, wl = np.exp(x), np.log(x)
    fin = np.isfinite(we) & (we > 0)
    ulp_e = np.abs(e[fin] - we[fin]) / np.spacing(we[fin])
    assert ulp_e.max() <= 1.0, (ulp_e.max(), x[fin][np.argmax(ulp_e)])
    assert np.array_equal(np.isnan(e), np.isnan(we)) and np.array_equal(e[~fin & ~np.isnan(we)], we[~fin & ~np.isnan(we)])
    finl = np.isfinite(wl) & (wl != 0)
    ulp_l = np.abs(lg[finl] - wl[finl]) / np.spacing(np.abs(wl[finl]))
    assert ulp_l.max() <= 2.0, (ulp_l.max(), x[finl][np.argmax(ulp_l)])
    assert lg[x == 1.0][0] == 0.0
    assert np.isneginf(lg[x == 0.0]).all() and np.isnan(lg[x == -1.0]).all() and np.isposinf(lg[x == np.inf]).all()


def test_host_tensor_log_plan_check_and_clamp_on_device(cuda):
    """A LogPlan given as a host torch tensor is checked and clamped on the
    device in one pass (otb_check_clamp_plan, core.py:141-145): NaN or +inf
    raise InvalidCost; entries below LOG_FLOOR (and -inf) become LOG_FLOOR."""
    import torch

    P = _api()
    from paper_2603_07156_b200 import errors
    from paper_2603_07156_b200.core import LOG_FLOOR

    rng = np.random.default_rng(3)
    for bad_val in (np.nan, np.inf):
        x = rng.standard_normal((37, 45))
        x[5, 7] = bad_val
        with pytest.raises(errors.InvalidCost):
            P.LogPlan(torch.from_numpy(x).pin_memory()).device_padded(64, torch.device("cuda", 0))
    x = rng.standard_normal((37, 45))
    x[0, 0], x[3, 44], x[36, 1] = -np.inf, -3e6, LOG_FLOOR
    t = P.LogPlan(torch.from_numpy(x).pin_memory()).device_padded(64, torch.device("cuda", 0))
    got = t[:, :45].cpu().numpy()
    want = np.maximum(x, LOG_FLOOR)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("mu_k,grad_target,max_inner", [(1e-3, None, 6), (1e-9, None, 3), (0.0, 1e-9, 8),
                                                         (0.0, 1.0, 4)])
def test_native_inner_iteration_equals_python_loop(cuda, mu_k, grad_target, max_inner):
    """inner_solve's loop body runs natively (otb_inner_iteration: the first
    step launched without waiting for the first eval, decisions in C) unless
    an observer is given; both paths must give the same bits: dual,
    candidate, Newton/CG counts, stop reason, objective — including the
    inexact-test stop, max_inner, and the gradient-floor stop before any
    step (grad_target = 1: the speculative step is discarded)."""
    import torch

    P = _api()
    from paper_2603_07156_b200 import instances
    from paper_2603_07156_b200.inner_newton import inner_solve
    from paper_2603_07156_b200.sinkhorn import warm_start

    C, a, b = instances.small_uniform(300, 257, 5)
    eta = 1e-2
    outs = []
    for observe in (False, True):
        prob = P.OtProblem(torch.from_numpy(C).cuda(), a, b)
        cfg = P.SolverConfig(eta=eta, kkt_tol=1e-9, max_inner=max_inner)
        X = P.LogPlan(O.product_log_plan(a, b))
        gam, _ = warm_start(X, prob, eta, 1e-3, gamma0=np.zeros(257))
        seen = []
        gs, cand, rep = inner_solve(X, gam, prob, cfg, mu_k=mu_k, outer_k=0, grad_target=grad_target,
                                    observer=(seen.append if observe else None))
        g = gs.gamma.cpu().numpy() if hasattr(gs.gamma, "cpu") else np.asarray(gs.gamma)
        outs.append((g.copy(), np.asarray(cand.log_entries).copy(), rep))
    (g0, c0, r0), (g1, c1, r1) = outs
    assert r0.newton_iters == r1.newton_iters and r0.cg_iters_total == r1.cg_iters_total
    assert r0.stop_reason == r1.stop_reason
    assert np.array_equal(g0.view(np.uint64), g1.view(np.uint64))
    assert np.array_equal(c0.view(np.uint64), c1.view(np.uint64))
    assert r0.objective == r1.objective and r0.kkt == r1.kkt and r0.bregman == r1.bregman
    assert r0.values == r1.values and r0.step_sizes == r1.step_sizes
    if grad_target == 1.0:
        assert r0.newton_iters == 0


@pytest.mark.parametrize("m,n", [(64, 16400), (24, 60000)])
def test_cluster_paths_are_deterministic(cuda, m, n):
    """Rows split over thread-block clusters (DSMEM exchanges, replicated
    CSR chunk state) and window-cluster hess_apply: two runs of a Newton
    step + inexact test give identical bits."""
    P = _api()
    from paper_2603_07156_b200 import instances
    from paper_2603_07156_b200.inner_newton import inner_solve

    C, a, b = instances.small_uniform(m, n, 2)
    res = []
    for _ in range(2):
        prob = P.OtProblem(C, a, b)
        cfg = P.SolverConfig(eta=1e-2, kkt_tol=1e-9, max_inner=2)
        gs, cand, rep = inner_solve(P.LogPlan(O.product_log_plan(a, b)), P.DualState(np.zeros(n)), prob, cfg,
                                    mu_k=1e-3, outer_k=0)
        res.append((np.asarray(gs.gamma).copy(), rep.cg_iters_total, rep.objective, rep.bregman))
    assert np.array_equal(res[0][0].view(np.uint64), res[1][0].view(np.uint64))
    assert res[0][1:] == res[1][1:]


@pytest.mark.parametrize("m,n", [(120, 16400), (70, 50001), (33, 9000)])
def test_dense_rho_equals_bitmap_rho(cuda, monkeypatch, m, n):
    """Window-cluster hess_apply over a DENSE P_rho (sparsify's dense mode,
    OTB_HV_DENSE=1) and over the bitmap-indexed pair runs (OTB_HV_DENSE=0):
    the same CSR, H v bitwise equal (dropped entries are 0.0 and every thread
    sums the same columns in the same order), and a 2-step inner solve gives
    the same bits.  (9000 columns forces the window clusters with OTB_HV_WC.)"""
    P = _api()
    from paper_2603_07156_b200 import instances
    from paper_2603_07156_b200.inner_newton import inner_solve

    monkeypatch.setenv("OTB_HV_WC", "1")
    C, a, b = instances.small_uniform(m, n, 9 + n)
    lx = O.product_log_plan(a, b)
    rng = np.random.default_rng(n)
    gam = rng.standard_normal(n) * 1e-3
    v = rng.standard_normal(n)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("OTB_HV_DENSE", mode)
        prob = P.OtProblem(C, a, b)
        eta = 1e-2
        cache = P.compute_p(P.LogPlan(lx), P.DualState(gam), prob, eta)
        rho = eta * float(np.linalg.norm(P.semidual_gradient(cache, prob))) / (m * n)
        sp = P.sparsify_p(cache, rho, int(np.argmax(a)))
        op = P.SparseHessianOp(sp)
        hv = op.matvec(v)
        info = cache.session.info()
        cfg = P.SolverConfig(eta=eta, kkt_tol=1e-9, max_inner=2)
        gs, cand, rep = inner_solve(P.LogPlan(lx), P.DualState(np.zeros(n)), P.OtProblem(C, a, b), cfg,
                                    mu_k=1e-3, outer_k=0)
        out[mode] = (sp, hv, np.asarray(gs.gamma).copy(), rep.cg_iters_total, rep.objective, info)
    assert out["0"][5]["hv_mode"] == 3 and out["1"][5]["hv_mode"] == 3
    s0, s1 = out["0"][0], out["1"][0]
    assert np.array_equal(s0.row_offsets, s1.row_offsets) and np.array_equal(s0.col_indices, s1.col_indices)
    assert np.array_equal(s0.values, s1.values) and np.array_equal(s0.anchor_row, s1.anchor_row)
    assert np.array_equal(out["0"][1].view(np.uint64), out["1"][1].view(np.uint64))
    assert np.array_equal(out["0"][2].view(np.uint64), out["1"][2].view(np.uint64))
    assert out["0"][3:5] == out["1"][3:5]


def _drop_pooled_contexts():
    """Destroy the idle libotb contexts (geometry knobs are read at creation)."""
    from paper_2603_07156_b200 import _lib, session

    for pool in session._CTX_POOL.values():
        while pool:
            _lib.lib.otb_destroy(pool.pop())


@pytest.mark.parametrize("m,n", [(150, 9000), (80, 10000)])
def test_dense_overlay_equals_group_kernel(cuda, monkeypatch, m, n):
    """8192 < n with shared-memory accumulators (the CSR group kernel, config
    3's geometry): while a quarter or more of P is kept, sparsify writes P_rho
    dense and hess_apply is the dense window-cluster kernel (the overlay);
    OTB_HV_OVERLAY=0 keeps the CSR group kernel.  The same CSR (bitwise), H v
    to reduction-order accuracy, the same CG counts and objective in a 2-step
    inner solve, and below the density threshold the overlay context goes back
    to the group kernel."""
    P = _api()
    from paper_2603_07156_b200 import instances
    from paper_2603_07156_b200.inner_newton import inner_solve

    C, a, b = instances.small_uniform(m, n, 5 + n)
    lx = O.product_log_plan(a, b)
    rng = np.random.default_rng(n)
    gam = rng.standard_normal(n) * 1e-3
    v = rng.standard_normal(n)
    eta = 1e-2
    out = {}
    for mode in ("0", "1"):
        _drop_pooled_contexts()
        monkeypatch.setenv("OTB_HV_OVERLAY", mode)
        monkeypatch.setenv("OTB_HV_DENSE", "1")   # dense wherever the context can (whatever the kept density)
        prob = P.OtProblem(C, a, b)
        cache = P.compute_p(P.LogPlan(lx), P.DualState(gam), prob, eta)
        rho = eta * float(np.linalg.norm(P.semidual_gradient(cache, prob))) / (m * n)
        sp = P.sparsify_p(cache, rho, int(np.argmax(a)))
        info = cache.session.info()
        hv = P.SparseHessianOp(sp).matvec(v)
        # by density (the default policy) with a threshold that keeps almost nothing: the overlay
        # context takes the group kernel again
        monkeypatch.delenv("OTB_HV_DENSE")
        cache2 = P.compute_p(P.LogPlan(lx), P.DualState(gam), prob, eta)
        sp2 = P.sparsify_p(cache2, 0.05, int(np.argmax(a)))
        info2 = cache2.session.info()
        hv2 = P.SparseHessianOp(sp2).matvec(v)
        monkeypatch.setenv("OTB_HV_DENSE", "1")
        cfg = P.SolverConfig(eta=eta, kkt_tol=1e-9, max_inner=2)
        gs, cand, rep = inner_solve(P.LogPlan(lx), P.DualState(np.zeros(n)), P.OtProblem(C, a, b), cfg,
                                    mu_k=1e-3, outer_k=0)
        out[mode] = (sp, hv, np.asarray(gs.gamma).copy(), rep.cg_iters_total, rep.objective, info, info2, sp2, hv2)
    i0, i1 = out["0"][5], out["1"][5]
    assert i0["hv_mode"] == 0 and i1["hv_mode"] == 0
    assert i0["rho_dense"] == 0 and i1["rho_dense"] == 1 and i1["wc_win"] >= 2     # the overlay ran
    assert out["1"][6]["rho_dense"] == 0                                            # ... and was left
    s0, s1 = out["0"][0], out["1"][0]
    assert np.array_equal(s0.row_offsets, s1.row_offsets) and np.array_equal(s0.col_indices, s1.col_indices)
    assert np.array_equal(s0.values, s1.values) and np.array_equal(s0.anchor_row, s1.anchor_row)
    assert np.max(np.abs(out["0"][1] - out["1"][1])) <= 1e-13 * np.max(np.abs(out["0"][1]))
    assert np.array_equal(out["0"][7].values, out["1"][7].values)
    assert np.array_equal(out["0"][8].view(np.uint64), out["1"][8].view(np.uint64))   # both: the group kernel
    assert np.max(np.abs(out["0"][2] - out["1"][2])) <= 1e-9 * max(1.0, np.max(np.abs(out["0"][2])))
    assert abs(out["0"][3] - out["1"][3]) <= 1
    assert abs(out["0"][4] - out["1"][4]) <= 1e-10 * abs(out["0"][4])
    monkeypatch.delenv("OTB_HV_DENSE")
    _drop_pooled_contexts()


@pytest.mark.parametrize("m,n", [(90, 70), (300, 4100), (64, 16400)])
def test_jacobi_pcg_matches_oracle(cuda, m, n):
    """cg_solve(preconditioner="jacobi") (extension; the reference's CG is
    plain): the device PCG direction and iteration count match the oracle's
    Jacobi PCG (diag(H_rho) = (d - (P_rho o P_rho)^T a)/eta accumulated by
    sparsify), it solves the same system as plain CG, and needs fewer
    iterations."""
    P = _api()
    from paper_2603_07156_b200 import instances

    C, a, b = instances.small_uniform(m, n, 3 + n)
    prob = P.OtProblem(C, a, b)
    eta = 1e-2
    lx = O.product_log_plan(a, b)
    rng = np.random.default_rng(m)
    gam = rng.standard_normal(n) * 1e-3
    cache = P.compute_p(P.LogPlan(lx), P.DualState(gam), prob, eta)
    grad = P.semidual_gradient(cache, prob)
    gn = float(np.linalg.norm(grad))
    rho = eta * gn / (m * n)
    op = P.SparseHessianOp(P.sparsify_p(cache, rho, int(np.argmax(a))))
    x0, it0, _ = P.cg_solve(op, gn, -grad, 1e-10)
    x1, it1, res1 = P.cg_solve(op, gn, -grad, 1e-10, preconditioner="jacobi")
    Pm, _ = O.softmax_rows(lx, C, gam, eta)
    H = O.SparseHessian(O.threshold_rows(Pm, rho, int(np.argmax(a))), a, eta)
    xr, itr, _ = O.preconditioned_cg(H.matvec, gn, -grad, O.jacobi_inverse(H, gn), 1e-10)
    assert abs(it1 - itr) <= 1
    assert rel(x1, xr) <= 1e-8
    assert rel(x1, x0) <= 1e-7            # the same Newton direction
    assert it1 <= it0
    x2, it2, _ = P.cg_solve(op, gn, -grad, 1e-10)   # back to plain: the reference's iterates
    assert it2 == it0 and np.array_equal(x2, x0)


def test_jacobi_pcg_solve_same_answer(cuda):
    """ibsn_solve with SolverConfig(cg_preconditioner="jacobi") on BASELINE
    config 1: the same outer / Newton counts and objective (<= 1e-8) as the
    plain-CG solve (the parity default), with fewer CG iterations in total."""
    P = _api()
    from paper_2603_07156_b200 import instances

    inst = instances.config(1, 0)
    plain = P.ibsn_solve(P.OtProblem(inst.cost, inst.a, inst.b), P.SolverConfig(eta=inst.eta, kkt_tol=inst.kkt_tol))
    pcg = P.ibsn_solve(P.OtProblem(inst.cost, inst.a, inst.b),
                       P.SolverConfig(eta=inst.eta, kkt_tol=inst.kkt_tol, cg_preconditioner="jacobi"))
    assert (pcg.outer_iters, pcg.newton_iters) == (plain.outer_iters, plain.newton_iters)
    assert abs(pcg.objective - plain.objective) <= 1e-8 * abs(plain.objective)
    assert pcg.cg_iters < plain.cg_iters


def test_speculative_step_with_eval_post_fallback(cuda, monkeypatch):
    """OTB_FORCE_EVAL_POST=1 makes a single rank finish its evals with the
    multi-rank kernels (k_colreduce + k_eval_post, and for the speculative
    first step of the native inner iteration the ev0 scalars copied by
    cudaMemcpyAsync).  Same bits as the fused single-rank finish, and the
    native loop equals the Python loop on that path too."""
    import torch

    P = _api()
    from paper_2603_07156_b200 import instances
    from paper_2603_07156_b200.inner_newton import inner_solve
    from paper_2603_07156_b200.sinkhorn import warm_start

    C, a, b = instances.small_uniform(301, 259, 6)   # a shape no pooled context has
    eta = 1e-2
    outs = []
    for force, observe in (("0", False), ("1", False), ("1", True)):
        monkeypatch.setenv("OTB_FORCE_EVAL_POST", force)
        from paper_2603_07156_b200 import session as S
        S._CTX_POOL.clear()                              # contexts read the knob when created
        prob = P.OtProblem(torch.from_numpy(C).cuda(), a, b)
        cfg = P.SolverConfig(eta=eta, kkt_tol=1e-9, max_inner=4)
        X = P.LogPlan(O.product_log_plan(a, b))
        gam, _ = warm_start(X, prob, eta, 1e-3, gamma0=np.zeros(259))
        seen = []
        gs, cand, rep = inner_solve(X, gam, prob, cfg, mu_k=1e-3, outer_k=0,
                                    observer=(seen.append if observe else None))
        g = gs.gamma.cpu().numpy() if hasattr(gs.gamma, "cpu") else np.asarray(gs.gamma)
        outs.append((g.copy(), rep.newton_iters, rep.cg_iters_total, rep.objective, rep.values))
    for o in outs[1:]:
        assert np.array_equal(o[0].view(np.uint64), outs[0][0].view(np.uint64))
        assert o[1:] == outs[0][1:]


@pytest.mark.parametrize("m,n,env", [(130, 16400, None), (97, 3000, "OTB_CG_FUSED")])
def test_cg_graph_batches_equal_eager_launches(cuda, monkeypatch, m, n, env):
    """The per-iteration CG path (multi-rank, window clusters, PCG, or the
    persistent CG switched off) replays each 16-iteration batch from a CUDA
    graph (OTB_CG_GRAPH, default on); eager launches (OTB_CG_GRAPH=0) give
    the same bits: Newton direction, CG iteration count, residual."""
    P = _api()
    from paper_2603_07156_b200 import instances
    from paper_2603_07156_b200 import session as S

    if env:
        monkeypatch.setenv(env, "0")
    C, a, b = instances.small_uniform(m, n, 21 + n)
    lx = O.product_log_plan(a, b)
    gam = np.random.default_rng(m).standard_normal(n) * 1e-3
    out = []
    for graph in ("1", "0"):
        monkeypatch.setenv("OTB_CG_GRAPH", graph)
        S._CTX_POOL.clear()                               # contexts read the knobs when created
        prob = P.OtProblem(C, a, b)
        eta = 1e-2
        cache = P.compute_p(P.LogPlan(lx), P.DualState(gam), prob, eta)
        grad = P.semidual_gradient(cache, prob)
        gn = float(np.linalg.norm(grad))
        op = P.SparseHessianOp(P.sparsify_p(cache, eta * gn / (m * n), int(np.argmax(a))))
        x, it, res = P.cg_solve(op, gn, -grad, 1e-10)
        assert cache.session.info()["cg_fused"] == 0
        out.append((x, it, res))
    assert out[0][1] == out[1][1] and out[0][1] > 16          # more than one batch
    assert np.array_equal(out[0][0].view(np.uint64), out[1][0].view(np.uint64))
    assert out[0][2] == out[1][2]
