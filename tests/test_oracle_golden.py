"""Pin the CPU oracle (oracle/otb_oracle.py) to the reference's own outputs.

The golden .npz files were produced by running the reference package
(tests/golden/make_golden.py).  The oracle restates the reference with the
same numpy expressions, so elementwise stages must match bit for bit; where
only a reduction order could differ the tolerance is a few ulp.  Also checks
the SPEC.md known-answer examples that pin the hot path.
"""

import math

import numpy as np
import pytest

from conftest import golden, golden_names
from oracle import otb_oracle as O


@pytest.mark.parametrize("name", golden_names("eval"))
def test_eval_bitwise(name):
    g = golden(name)
    P, lse = O.softmax_rows(g["logX"], g["C"], g["gamma"], float(g["eta"]))
    assert np.array_equal(P, g["P"])
    assert np.array_equal(lse, g["lse"])
    assert O.objective(lse, g["gamma"], g["a"], g["b"], float(g["eta"])) == float(g["value"])
    assert np.array_equal(O.gradient(P, g["a"], g["b"]), g["grad"])


@pytest.mark.parametrize("name", golden_names("sparsify"))
def test_sparsify_hv_cg(name):
    g = golden(name)
    eta = float(g["eta"])
    P, _ = O.softmax_rows(g["logX"], g["C"], g["gamma"], eta)
    rows = O.threshold_rows(P, float(g["rho"]), int(g["anchor"]))
    assert np.array_equal(rows.row_ptr, g["row_offsets"])
    assert np.array_equal(rows.cols, g["col_indices"])
    assert np.array_equal(rows.vals, g["values"])
    assert np.array_equal(rows.anchor_row, g["anchor_row"])
    h = O.SparseHessian(rows, g["a"], eta)
    assert np.array_equal(h.d, g["d"])
    assert np.array_equal(h.matvec(g["v"]), g["hv"])
    grad = O.gradient(P, g["a"], g["b"])
    x, it, res = O.conjugate_gradient(h.matvec, float(g["grad_norm"]), -grad, 1e-10)
    assert it == int(g["cg_iters"])
    np.testing.assert_allclose(x, g["cg_x"], rtol=0, atol=1e-13 * np.abs(g["cg_x"]).max())


@pytest.mark.parametrize("name", golden_names("newton"))
def test_newton_step(name):
    g = golden(name)
    gam, t, its = O.newton_step(g["logX"], g["C"], g["a"], g["b"], g["gamma"], float(g["eta"]))
    assert t == float(g["t"])
    assert its == int(g["cg_iters"])
    np.testing.assert_allclose(gam, g["gamma_new"], rtol=1e-12, atol=1e-15)


def test_newton_backtracks_in_golden():
    """SURVEY §4 rare branch: gen_uniform(24,16,1) at eta=1e-3 backtracks to 0.8^9."""
    g = golden("newton_0")
    assert float(g["t"]) == pytest.approx(0.8 ** 9)


@pytest.mark.parametrize("name", golden_names("round"))
def test_rounding_divergence_kkt(name):
    g = golden(name)
    L = O.clamp_log_plan(g["logX"])
    R = O.round_plan(np.exp(L), g["a"], g["b"])
    assert np.array_equal(R, g["rounded"])
    assert O.bregman(R, L) == float(g["bregman"])
    k = O.kkt(R, g["gamma"], g["C"], g["a"], g["b"])
    for key in ("delta_p", "delta_d", "delta_c", "delta_kkt"):
        assert k[key] == float(g[key])


@pytest.mark.parametrize("name", golden_names("candidate"))
def test_candidate(name):
    g = golden(name)
    _, lse = O.softmax_rows(g["logX"], g["C"], g["gamma"], float(g["eta"]))
    cand = O.candidate_log(g["logX"], g["C"], g["gamma"], lse, g["a"], float(g["eta"]))
    assert np.array_equal(cand, g["candidate"])


@pytest.mark.parametrize("name", golden_names("warm"))
def test_warm_start(name):
    g = golden(name)
    gam, zeta, _ = O.warm_start(g["logX"], g["C"], g["a"], g["b"], float(g["eta"]), 1e-3)
    assert np.array_equal(gam, g["gamma"])
    assert np.array_equal(zeta, g["zeta"])


@pytest.mark.parametrize("name", golden_names("inner"))
def test_inner_solve(name):
    g = golden(name)
    m, n = g["C"].shape
    r = O.inner(g["logX"], g["C"], g["a"], g["b"], g["gamma0"], float(g["eta"]), 1e-4, float(min(m, n)))
    assert r.newton_iters == int(g["newton_iters"])
    assert r.cg_total == int(g["cg_iters_total"])
    assert r.stop == str(g["stop"])
    np.testing.assert_array_equal(np.asarray([s.t for s in r.steps]), g["steps"])
    np.testing.assert_allclose(r.gamma, g["gamma"], rtol=1e-12, atol=1e-16)
    np.testing.assert_allclose(r.candidate, g["candidate"], rtol=1e-12, atol=1e-9)


@pytest.mark.slow
@pytest.mark.parametrize("name", golden_names("solve"))
def test_solve(name):
    g = golden(name)
    res = O.solve(g["C"], g["a"], g["b"], float(g["eta"]), kkt_tol=float(g["kkt_tol"]))
    assert res.outer_iters == int(g["outer_iters"])
    assert res.objective == pytest.approx(float(g["objective"]), rel=1e-12)
    assert [r["inner_total"] for r in res.records] == list(g["inner_total"])
    assert [r["cg_total"] for r in res.records] == list(g["cg_total"])


# ---------------------------------------------------------------- SPEC KATs

def test_spec_compute_p_two_term():
    """m=1, n=2, X=[[.5,.5]], gamma=0, C=[[0, eta ln 2]] -> [2/3, 1/3]."""
    eta = 0.1
    P, _ = O.softmax_rows(np.log([[0.5, 0.5]]), np.array([[0.0, eta * math.log(2)]]), np.zeros(2), eta)
    np.testing.assert_allclose(P, [[2 / 3, 1 / 3]], rtol=1e-14)


def test_spec_sparsify_row():
    """(0.6,0.3,0.1) rho=0.2 -> (2/3,1/3); (0.4,0.3,0.3) rho=0.5 -> (1.0) at 0."""
    P = np.array([[0.5, 0.25, 0.25], [0.6, 0.3, 0.1], [0.4, 0.3, 0.3]])
    rows = O.threshold_rows(P, 0.2, 0)
    c, v = rows.row(1)
    assert list(c) == [0, 1] and np.allclose(v, [2 / 3, 1 / 3])
    rows = O.threshold_rows(P, 0.5, 0)
    c, v = rows.row(2)
    assert list(c) == [0] and list(v) == [1.0]


def test_spec_threshold_and_anchor():
    """SPEC.md:191-202."""
    assert O.anchor_index(np.array([0.2, 0.5, 0.3])) == 1
    assert O.anchor_index(np.array([0.5, 0.5])) == 0
    assert O.threshold(1e-4, 100, 100, 0.5) == pytest.approx(5e-9)
    assert O.threshold(1.0, 1, 1, 2.0) == 2.0


def test_spec_bregman_and_rounding():
    """SPEC.md:497-508."""
    d = O.bregman(np.array([[0.5, 0.5]]), np.log([[0.25, 0.75]]))
    assert d == pytest.approx(0.5 * math.log(2) + 0.5 * math.log(2 / 3), abs=1e-12)
    r = O.round_plan(np.array([[0.6, 0.0], [0.0, 0.6]]), np.array([0.5, 0.5]), np.array([0.5, 0.5]))
    np.testing.assert_allclose(r, [[0.5, 0.0], [0.0, 0.5]], atol=1e-15)
    r0 = O.round_plan(np.zeros((2, 3)), np.array([0.5, 0.5]), np.array([0.2, 0.3, 0.5]))
    np.testing.assert_allclose(r0, np.outer([0.5, 0.5], [0.2, 0.3, 0.5]), atol=1e-15)


def test_spec_mu_schedule():
    """SPEC.md:425-427, acceptance #10."""
    assert O.mu(0) == 1e-4
    assert O.mu(9) == pytest.approx(1e-6)
    assert O.mu(10**6) == 1e-11


def test_spec_cg_trivial():
    """rhs = 0 -> x = 0 in 0 iterations; zero operator + shift 1 -> x = rhs."""
    x, it, res = O.conjugate_gradient(lambda v: np.zeros_like(v), 1.0, np.zeros(4))
    assert it == 0 and not x.any() and res == 0.0
    rhs = np.array([1.0, -2.0, 0.5])
    x, it, _ = O.conjugate_gradient(lambda v: np.zeros_like(v), 1.0, rhs)
    np.testing.assert_allclose(x, rhs)


@pytest.mark.parametrize("name", golden_names("eot"))
def test_oracle_eot_matches_reference(name):
    """eot_single_solve (bregman_outer.py:284-327) restated by the oracle."""
    g = golden(name)
    cand, rounded, obj, kkt, newton, cg, gamma, gn = O.eot_solve(g["C"], g["a"], g["b"], float(g["eta"]),
                                                                 float(g["kkt_tol"]))
    assert newton == int(g["newton_iters"])
    assert abs(cg - int(g["cg_total"])) <= 1
    assert obj == pytest.approx(float(g["objective"]), rel=1e-12)
    assert kkt == pytest.approx(float(g["kkt"]), rel=1e-9)
    assert np.max(np.abs(rounded - g["rounded"])) <= 1e-12


@pytest.mark.parametrize("name", golden_names("ibsink"))
def test_oracle_ibsink_matches_reference(name):
    """ibsink_solve (bregman_outer.py:191-281) restated by the oracle."""
    g = golden(name)
    log_x, rounded, obj, kkt, outer, sweeps, recs = O.ibsink_solve(g["C"], g["a"], g["b"], float(g["eta"]),
                                                                   float(g["kkt_tol"]), max_outer=int(g["max_outer"]))
    assert outer == int(g["outer_iters"])
    assert [r["inner_total"] for r in recs] == list(g["inner_total"])
    assert obj == pytest.approx(float(g["objective"]), rel=1e-12)
    assert np.max(np.abs(rounded - g["rounded"])) <= 1e-12


def test_oracle_jacobi_pcg_solves_the_system():
    """The oracle's Jacobi PCG (extension) reaches the same solution as the
    oracle's plain CG (pinned to the reference's krylov.py) on a golden
    sparsify case, in no more iterations."""
    g = golden("sparsify_1")
    C, a, b, lx, gam, eta = g["C"], g["a"], g["b"], g["logX"], g["gamma"], float(g["eta"])
    P, _ = O.softmax_rows(lx, C, gam, eta)
    H = O.SparseHessian(O.threshold_rows(P, float(g["rho"]), int(g["anchor"])), a, eta)
    grad = O.gradient(P, a, b)
    gn = float(np.linalg.norm(grad))
    x0, k0, _ = O.conjugate_gradient(H.matvec, gn, -grad, 1e-10)
    x1, k1, _ = O.preconditioned_cg(H.matvec, gn, -grad, O.jacobi_inverse(H, gn), 1e-10)
    assert np.max(np.abs(x1 - x0)) <= 1e-8 * np.max(np.abs(x0))
    assert k1 <= k0
