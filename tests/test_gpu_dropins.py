"""Kernel-level drop-ins with the reference's signatures, on dense LINEAR
matrices (csrc/dense_api.cuh), against goldens produced by the reference
itself (tests/golden/make_golden.py ``dense``):

- round_to_feasible -> FeasiblePlan (feasibility.py:44-69)
- bregman_div(x, LogPlan) (72-85)
- c_transform, kkt_residual on x AS GIVEN (negative entries, infeasible
  marginals: the ||min(x,0)|| term and zeta_used) (88-122)
- gap (125-127)
- hessian_matvec_exact (semidual.py:103-114)
- zeta_update, gamma_update, scaled_plan_log (sinkhorn.py:41-58)

Tolerances: elementwise numpy expressions in numpy's order, sums in a fixed
device order -> agreement to a few ulp of the summed magnitudes.
"""

import numpy as np
import pytest

from conftest import golden, golden_names

pytestmark = pytest.mark.gpu


def _api():
    import paper_2603_07156_b200 as P

    return P


def rel(x, y):
    x, y = np.asarray(x, dtype=np.float64), np.asarray(y, dtype=np.float64)
    return float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-300))


@pytest.mark.parametrize("name", golden_names("dense"))
def test_round_to_feasible_returns_feasible_plan(cuda, name):
    P = _api()
    g = golden(name)
    f = P.round_to_feasible(g["x"], g["a"], g["b"])
    assert isinstance(f, P.FeasiblePlan)
    assert f.shape == g["x"].shape
    assert rel(f.entries, g["rounded"]) <= 1e-13
    assert np.max(np.abs(f.entries.sum(axis=1) - g["a"])) <= 1e-15
    assert np.max(np.abs(f.entries.sum(axis=0) - g["b"])) <= 1e-15
    # an already feasible input passes through (up to the last bits of the sums)
    f2 = P.round_to_feasible(f.entries, g["a"], g["b"])
    assert rel(f2.entries, f.entries) <= 1e-14


@pytest.mark.parametrize("name", golden_names("dense"))
def test_bregman_div_matches_reference(cuda, name):
    P = _api()
    g = golden(name)
    d = P.bregman_div(g["x"], P.LogPlan(g["logY"]))
    assert d == pytest.approx(float(g["bregman"]), rel=1e-12, abs=1e-15)
    # FeasiblePlan input (the reference passes .entries)
    f = P.FeasiblePlan(g["x"])
    assert P.bregman_div(f, P.LogPlan(g["logY"])) == d


@pytest.mark.parametrize("name", golden_names("dense"))
def test_kkt_residual_certifies_x_as_given(cuda, name):
    P = _api()
    g = golden(name)
    rep = P.kkt_residual(g["xneg"], g["gamma"], g["C"], g["a"], g["b"])
    ref = g["kkt"]
    for got, want in zip((rep.delta_p, rep.delta_d, rep.delta_c, rep.delta_kkt), ref):
        assert got == pytest.approx(float(want), rel=1e-10, abs=1e-17)
    assert rep.delta_p > 1e-6                       # the infeasibility is visible (not rounded away)
    assert np.array_equal(rep.zeta_used, g["zeta_used"])   # min of exact differences: bitwise
    assert np.array_equal(P.c_transform(g["gamma"], g["C"]), g["c_transform"])


@pytest.mark.parametrize("name", golden_names("dense"))
def test_gap_matches_reference(cuda, name):
    P = _api()
    g = golden(name)
    f = P.FeasiblePlan(g["rounded"])
    assert P.gap(f, g["C"], 0.01) == pytest.approx(float(g["gap"]), rel=1e-12)


@pytest.mark.parametrize("name", golden_names("dense"))
def test_hessian_matvec_exact_matches_reference(cuda, name):
    P = _api()
    g = golden(name)
    prob = P.OtProblem(g["C"], g["a"], g["b"])
    eta = float(g["eta"])
    cache = P.compute_p(P.LogPlan(g["logY"]), P.DualState(g["gamma"]), prob, eta)
    hv = P.hessian_matvec_exact(cache, prob, eta, g["v"])
    assert rel(hv, g["hv"]) <= 1e-12
    # H 1 = 0
    h1 = P.hessian_matvec_exact(cache, prob, eta, np.ones(prob.shape[1]))
    assert np.max(np.abs(h1)) <= 1e-12 / eta


@pytest.mark.parametrize("name", golden_names("dense"))
def test_single_sinkhorn_updates_match_reference(cuda, name):
    P = _api()
    g = golden(name)
    prob = P.OtProblem(g["C"], g["a"], g["b"])
    eta = float(g["eta"])
    lp = P.LogPlan(g["logY"])
    st = P.TwoDualState(g["gamma"], g["zeta0"])
    zu = P.zeta_update(lp, st, prob, eta)
    assert rel(zu.zeta, g["zeta_upd"]) <= 1e-13
    assert np.array_equal(zu.gamma, g["gamma"])
    gu = P.gamma_update(lp, st, prob, eta)
    assert rel(gu.gamma, g["gamma_upd"]) <= 1e-13
    spl = P.scaled_plan_log(lp, st, prob, eta)
    assert rel(spl, g["scaled_log"]) <= 1e-15
