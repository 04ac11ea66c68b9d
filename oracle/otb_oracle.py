"""CPU oracle for the IBSN inner loop — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference algorithm on the hot
path (pkg/src/otibsn/*.py under /root/reference).  It exists so that the
CUDA path can be checked on machines where the reference is absent (the GPU
box) and so that ``bench.py --impl reference`` can time the reference's CPU
algorithm on the box's host cores.

Rules:
  * only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
    baseline / reference arm may import this module;
  * the product package ``paper_2603_07156_b200`` never imports it;
  * every function cites the reference file:line it restates.

Pinning: ``tests/golden/make_golden.py`` runs the live reference in the
build container and stores its outputs as ``tests/golden/*.npz``;
``tests/test_oracle_golden.py`` checks this module against them (bitwise for
the elementwise stages, within a few ulp where numpy reduction order is the
only difference).  Parity is therefore pinned, not assumed.

Elementwise arithmetic follows numpy's evaluation order in the reference
expression by expression (e.g. ``(gamma - C) / eta`` is a subtraction then a
true division, never a multiplication by 1/eta), because those are the
values the CUDA kernels are compared against.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# Constants restated from the reference.
LOG_FLOOR = -1e6                 # core.py:24
MARGINAL_SUM_TOL = 1e-12         # core.py:27
LINE_SEARCH_CAP = 200            # inner_newton.py:35
GRAD_HARD_FLOOR = 1e-15          # inner_newton.py:39
DEFAULT_SWEEP_CAP = 100_000      # sinkhorn.py:21


class OracleError(Exception):
    """Raised where the reference raises; ``kind`` names the reference class."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# --------------------------------------------------------------------------
# semi-dual evaluation  (semidual.py)
# --------------------------------------------------------------------------

def row_logits(log_x: np.ndarray, cost: np.ndarray, gamma: np.ndarray, eta: float) -> np.ndarray:
    """semidual.py:51-52 — logX + (gamma - C) / eta."""
    return log_x + (gamma[None, :] - cost) / eta


def softmax_rows(log_x, cost, gamma, eta):
    """semidual.py:55-87 — stabilised row softmax P and per-row log-normaliser.

    Returns (P, lse).  Raises OracleError('NumericalOverflow') on non-finite
    output like semidual.py:85-86.
    """
    z = row_logits(log_x, cost, gamma, eta)
    top = z.max(axis=1, keepdims=True)
    e = np.exp(z - top)
    tot = e.sum(axis=1, keepdims=True)
    p = e / tot
    lse = top[:, 0] + np.log(tot[:, 0])
    if not (np.isfinite(p).all() and np.isfinite(lse).all()):
        raise OracleError("NumericalOverflow", "non-finite softmax")
    return p, lse


def objective(lse, gamma, a, b, eta) -> float:
    """semidual.py:90-95 — L = -b.gamma + eta * (a.lse)."""
    return float(-b @ gamma + eta * (a @ lse))


def gradient(p, a, b) -> np.ndarray:
    """semidual.py:98-100 — g = P^T a - b."""
    return p.T @ a - b


def hessian_exact_apply(p, a, eta, v):
    """semidual.py:103-114 — (diag(P^T a) v - P^T (a * (P v))) / eta."""
    w = p.T @ a
    return (w * v - p.T @ (a * (p @ v))) / eta


# --------------------------------------------------------------------------
# sparsification  (sparsify.py)
# --------------------------------------------------------------------------

def anchor_index(a) -> int:
    """sparsify.py:25-27 — first index of max(a)."""
    return int(np.argmax(a))


def threshold(eta, m, n, grad_norm) -> float:
    """sparsify.py:30-32 — rho = eta * ||g|| / (m n)."""
    return eta * grad_norm / (m * n)


@dataclass
class ThresholdedRows:
    """The output of sparsify.py:90-127 in plain arrays.

    ``row_ptr``/``cols``/``vals`` are the CSR of the m-1 off-anchor rows in
    original order (anchor skipped, columns ascending); ``anchor_row`` is the
    unnormalised dense copy of P[anchor].
    """

    row_ptr: np.ndarray
    cols: np.ndarray
    vals: np.ndarray
    anchor: int
    anchor_row: np.ndarray
    n: int

    @property
    def m(self) -> int:
        return self.row_ptr.size  # (m-1) + 1

    def row(self, i: int):
        """(cols, vals) of original row i (anchor: all n columns)."""
        if i == self.anchor:
            return np.arange(self.n), self.anchor_row
        k = i if i < self.anchor else i - 1
        s, e = self.row_ptr[k], self.row_ptr[k + 1]
        return self.cols[s:e], self.vals[s:e]

    def dense(self) -> np.ndarray:
        """sparsify.py:80-87."""
        out = np.zeros((self.m, self.n))
        for i in range(self.m):
            c, v = self.row(i)
            out[i, c] = v
        return out

    def apply(self, v):
        """sparsify.py:64-72 — P_rho v (length m)."""
        r = np.repeat(np.arange(self.row_ptr.size - 1), np.diff(self.row_ptr))
        off = np.zeros(self.row_ptr.size - 1)
        np.add.at(off, r, self.vals * v[self.cols])
        i = self.anchor
        return np.concatenate((off[:i], [self.anchor_row @ v], off[i:]))

    def apply_t(self, w):
        """sparsify.py:74-78 — P_rho^T w (length n)."""
        i = self.anchor
        w_off = np.concatenate((w[:i], w[i + 1:]))
        r = np.repeat(np.arange(self.row_ptr.size - 1), np.diff(self.row_ptr))
        out = np.zeros(self.n)
        np.add.at(out, self.cols, self.vals * w_off[r])
        return out + self.anchor_row * w[i]


def threshold_rows(p, rho, anchor) -> ThresholdedRows:
    """sparsify.py:90-127 — keep P >= rho (and P > 0), renormalise rows.

    Rows with nothing kept keep their first argmax with value 1; the anchor
    row is copied unnormalised and stored apart.
    """
    m, n = p.shape
    mask = (p >= rho) & (p > 0.0)
    mask[anchor, :] = False
    has = mask.any(axis=1)
    has[anchor] = True
    empty = np.flatnonzero(~has)
    if empty.size:
        mask[empty, np.argmax(p[empty], axis=1)] = True
    sums = np.where(mask, p, 0.0).sum(axis=1)
    sums[anchor] = 1.0
    order = np.array([i for i in range(m) if i != anchor], dtype=np.int64)
    sub = mask[order]
    row_ptr = np.zeros(m, dtype=np.int64)
    np.cumsum(sub.sum(axis=1), out=row_ptr[1:])
    rr, cc = np.nonzero(sub)
    vals = p[order[rr], cc] / sums[order[rr]]
    return ThresholdedRows(row_ptr, cc.astype(np.int64), vals, anchor, p[anchor].copy(), n)


@dataclass
class SparseHessian:
    """sparsify.py:130-159 — (diag(P_rho^T a) - P_rho^T diag(a) P_rho)/eta."""

    rows: ThresholdedRows
    a: np.ndarray
    eta: float
    d: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.d is None:
            self.d = self.rows.apply_t(self.a)   # sparsify.py:143-145

    def matvec(self, v):
        """sparsify.py:151-153."""
        return (self.d * v - self.rows.apply_t(self.a * self.rows.apply(v))) / self.eta

    def dense(self):
        """sparsify.py:155-159."""
        p = self.rows.dense()
        w = p.T @ self.a
        return (np.diag(w) - p.T @ (self.a[:, None] * p)) / self.eta


# --------------------------------------------------------------------------
# conjugate gradients  (krylov.py)
# --------------------------------------------------------------------------

def conjugate_gradient(apply_h, shift, rhs, rel_tol=1e-10, max_iters=None):
    """krylov.py:17-85 — CG on (H + shift I) x = rhs from x0 = 0.

    Returns (x, iterations, final residual norm).
    """
    rhs = np.asarray(rhs, dtype=np.float64)
    n = rhs.size
    cap = 2 * n if max_iters is None else max_iters
    bnorm = float(np.linalg.norm(rhs))
    if shift == 0.0 and abs(rhs.sum()) > 1e-12 * max(1.0, bnorm):
        raise OracleError("InconsistentSystem", "rhs outside range")
    x = np.zeros(n)
    if bnorm == 0.0:
        return x, 0, 0.0
    r = rhs.copy()
    d = rhs.copy()
    rr = float(r @ r)
    goal = rel_tol * bnorm
    k = 0
    for _ in range(cap):
        hd = apply_h(d) + shift * d
        curv = float(d @ hd)
        if curv <= 0.0:
            if math.sqrt(rr) <= goal:
                break
            raise OracleError("NotPositiveDefinite", f"curvature {curv:.3g}")
        alpha = rr / curv
        x += alpha * d
        r -= alpha * hd
        k += 1
        rr_new = float(r @ r)
        if math.sqrt(rr_new) <= goal:
            rr = rr_new
            break
        d = r + (rr_new / rr) * d
        rr = rr_new
    return x, k, float(np.sqrt(rr))


def jacobi_inverse(h: SparseHessian, shift):
    """Extension (no reference counterpart; the reference's CG is plain):
    1 / diag(H_rho + shift I), diag(H_rho)_j = (d_j - sum_i a_i P_rho[i,j]^2)/eta."""
    p = h.rows.dense()
    q = (p * p).T @ h.a
    dj = (h.d - q) / h.eta + shift
    return np.where(dj > 0.0, 1.0 / np.where(dj > 0.0, dj, 1.0), 1.0)


def preconditioned_cg(apply_h, shift, rhs, minv, rel_tol=1e-10, max_iters=None):
    """Jacobi PCG on (H + shift I) x = rhs from x0 = 0: z = minv r, the
    same stopping test on ||r|| as krylov.py:79-82 (extension)."""
    rhs = np.asarray(rhs, dtype=np.float64)
    n = rhs.size
    cap = 2 * n if max_iters is None else max_iters
    bnorm = float(np.linalg.norm(rhs))
    x = np.zeros(n)
    if bnorm == 0.0:
        return x, 0, 0.0
    r = rhs.copy()
    z = minv * r
    d = z.copy()
    rz = float(r @ z)
    rr = float(r @ r)
    goal = rel_tol * bnorm
    k = 0
    for _ in range(cap):
        hd = apply_h(d) + shift * d
        curv = float(d @ hd)
        if curv <= 0.0:
            if math.sqrt(rr) <= goal:
                break
            raise OracleError("NotPositiveDefinite", f"curvature {curv:.3g}")
        alpha = rz / curv
        x += alpha * d
        r -= alpha * hd
        k += 1
        rr = float(r @ r)
        if math.sqrt(rr) <= goal:
            break
        z = minv * r
        rz_new = float(r @ z)
        d = z + (rz_new / rz) * d
        rz = rz_new
    return x, k, float(np.sqrt(rr))


# --------------------------------------------------------------------------
# feasibility  (feasibility.py)
# --------------------------------------------------------------------------

def round_plan(x, a, b) -> np.ndarray:
    """feasibility.py:44-69 — Altschuler rounding onto the transport polytope."""
    x = np.asarray(x, dtype=np.float64)
    rs = x.sum(axis=1)
    with np.errstate(divide="ignore", invalid="ignore"):
        z = np.where(rs > 0.0, np.minimum(a / rs, 1.0), 1.0)
    f = x * z[:, None]
    cs = f.sum(axis=0)
    with np.errstate(divide="ignore", invalid="ignore"):
        y = np.where(cs > 0.0, np.minimum(b / cs, 1.0), 1.0)
    f = f * y[None, :]
    er = a - f.sum(axis=1)
    ec = b - f.sum(axis=0)
    deficit = float(np.abs(er).sum())
    if deficit > 0.0:
        f = f + np.outer(er, ec) / deficit
    return f


def bregman(x, log_y) -> float:
    """feasibility.py:72-85 — sum x(log x - log y) - sum x + sum exp(log y)."""
    x = np.asarray(x, dtype=np.float64)
    pos = x > 0.0
    t = np.where(pos, x * (np.log(np.where(pos, x, 1.0)) - log_y), 0.0)
    return float(t.sum() - x.sum() + np.exp(log_y).sum())


def kkt(x, gamma, cost, a, b):
    """feasibility.py:93-122 — relative KKT residual with c-transform.

    Returns dict(delta_p, delta_d, delta_c, delta_kkt, zeta).
    """
    sh = cost - gamma[None, :]
    zeta = sh.min(axis=1)
    slack = sh - zeta[:, None]
    cscale = 1.0 + float(np.linalg.norm(cost))
    dp = max(
        float(np.linalg.norm(x.sum(axis=1) - a)) / (1.0 + float(np.linalg.norm(a))),
        float(np.linalg.norm(x.sum(axis=0) - b)) / (1.0 + float(np.linalg.norm(b))),
        float(np.linalg.norm(np.minimum(x, 0.0))) / (1.0 + float(np.linalg.norm(x))),
    )
    dd = float(np.linalg.norm(np.minimum(slack, 0.0))) / cscale
    dc = abs(float((x * slack).sum())) / cscale
    return dict(delta_p=dp, delta_d=dd, delta_c=dc, delta_kkt=max(dp, dd, dc), zeta=zeta)


# --------------------------------------------------------------------------
# log plan helpers  (core.py)
# --------------------------------------------------------------------------

def clamp_log_plan(arr) -> np.ndarray:
    """core.py:141-145 — reject NaN/+inf, clamp at LOG_FLOOR."""
    arr = np.ascontiguousarray(np.asarray(arr, dtype=np.float64))
    if np.isnan(arr).any() or (arr == np.inf).any():
        raise OracleError("InvalidCost", "log plan contains NaN or +inf")
    return np.maximum(arr, LOG_FLOOR)


def product_log_plan(a, b) -> np.ndarray:
    """bregman_outer.py:91-93 / core.py:208-212 — log a_i + log b_j."""
    return clamp_log_plan(np.log(a)[:, None] + np.log(b)[None, :])


def candidate_log(log_x, cost, gamma, lse, a, eta) -> np.ndarray:
    """inner_newton.py:151-167 — log(diag(a) P) assembled left to right."""
    raw = np.log(a)[:, None] + log_x + (gamma[None, :] - cost) / eta - lse[:, None]
    return clamp_log_plan(raw)


def mu(k, mu0=1e-4, floor=1e-11) -> float:
    """bregman_outer.py:34-36."""
    return max(mu0 / (k + 1) ** 2, floor)


# --------------------------------------------------------------------------
# Newton step and inner loop  (inner_newton.py)
# --------------------------------------------------------------------------

@dataclass
class Evaluation:
    gamma: np.ndarray
    p: np.ndarray
    lse: np.ndarray
    value: float


def evaluate(log_x, cost, a, b, gamma, eta) -> Evaluation:
    p, lse = softmax_rows(log_x, cost, gamma, eta)
    return Evaluation(gamma, p, lse, objective(lse, gamma, a, b, eta))


def line_search(log_x, cost, a, b, gamma, step_dir, value0, slope, eta, sigma, beta):
    """inner_newton.py:74-94 — Armijo backtracking from t = 1."""
    t = 1.0
    for _ in range(LINE_SEARCH_CAP):
        ev = evaluate(log_x, cost, a, b, gamma + t * step_dir, eta)
        if ev.value <= value0 + sigma * t * slope:
            return ev, t
        t *= beta
    raise OracleError("LineSearchStalled", f"{LINE_SEARCH_CAP} trials")


@dataclass
class StepInfo:
    t: float
    cg_iters: int
    slope: float
    rho: float
    nnz: int


def step_from(log_x, cost, a, b, ev: Evaluation, grad, eta, sigma=1e-4, beta=0.8,
              cg_rel_tol=1e-10, cg_max_iters=None, rho=None):
    """inner_newton.py:97-122 — one sparsified Newton step from a cached eval.

    Returns (new Evaluation, StepInfo).  ``rho`` may be forced (test hook).
    """
    m, n = cost.shape
    gnorm = float(np.linalg.norm(grad))
    if rho is None:
        rho = threshold(eta, m, n, gnorm)
    rows = threshold_rows(ev.p, rho, anchor_index(a))
    h = SparseHessian(rows, a, eta)
    direction, its, _ = conjugate_gradient(h.matvec, gnorm, -grad, cg_rel_tol, cg_max_iters)
    slope = float(grad @ direction)
    new_ev, t = line_search(log_x, cost, a, b, ev.gamma, direction, ev.value, slope, eta, sigma, beta)
    return new_ev, StepInfo(t, its, slope, rho, int(rows.vals.size + rows.anchor_row.size))


def newton_step(log_x, cost, a, b, gamma, eta, sigma=1e-4, beta=0.8, cg_rel_tol=1e-10,
                cg_max_iters=None):
    """inner_newton.py:125-148 — returns (gamma', t, cg_iters)."""
    ev = evaluate(log_x, cost, a, b, gamma, eta)
    g = gradient(ev.p, a, b)
    if float(np.linalg.norm(g)) == 0.0:
        return gamma, 0.0, 0
    new_ev, info = step_from(log_x, cost, a, b, ev, g, eta, sigma, beta, cg_rel_tol, cg_max_iters)
    return new_ev.gamma, info.t, info.cg_iters


@dataclass
class InnerResult:
    gamma: np.ndarray
    candidate: np.ndarray        # clamped log plan
    lse: np.ndarray
    newton_iters: int
    cg_total: int
    grad_norm: float
    stop: str                    # inexact_criterion | grad_floor | max_inner
    steps: list
    values: list
    rounded: np.ndarray | None   # rounding of the accepted candidate when tested


def inner(log_x, cost, a, b, gamma0, eta, mu_k, scale, max_inner=500, sigma=1e-4, beta=0.8,
          cg_rel_tol=1e-10, cg_max_iters=None, grad_target=None) -> InnerResult:
    """inner_newton.py:170-258 — Newton steps until the inexact test passes."""
    floor = GRAD_HARD_FLOOR if grad_target is None else max(grad_target, GRAD_HARD_FLOOR)
    ev = evaluate(log_x, cost, a, b, gamma0, eta)
    g = gradient(ev.p, a, b)
    gn = float(np.linalg.norm(g))
    steps, values, cg_total = [], [ev.value], 0
    stop = "max_inner"
    cand = None
    rounded = None
    for _ in range(max_inner):
        if gn <= floor:
            stop = "grad_floor"
            break
        ev, info = step_from(log_x, cost, a, b, ev, g, eta, sigma, beta, cg_rel_tol, cg_max_iters)
        steps.append(info)
        values.append(ev.value)
        cg_total += info.cg_iters
        g = gradient(ev.p, a, b)
        gn = float(np.linalg.norm(g))
        if grad_target is None and gn < mu_k:
            cand = candidate_log(log_x, cost, ev.gamma, ev.lse, a, eta)
            rounded = round_plan(np.exp(cand), a, b)
            if bregman(rounded, cand) <= scale * mu_k:
                stop = "inexact_criterion"
                break
        cand = None
        rounded = None
    if cand is None:
        cand = candidate_log(log_x, cost, ev.gamma, ev.lse, a, eta)
    return InnerResult(ev.gamma, cand, ev.lse, len(steps), cg_total, gn, stop, steps, values, rounded)


# --------------------------------------------------------------------------
# warm start  (sinkhorn.py)
# --------------------------------------------------------------------------

def _lse(values, axis):
    """sinkhorn.py:36-39."""
    peak = values.max(axis=axis, keepdims=True)
    out = peak[:, 0] if axis == 1 else peak[0, :]
    return out + np.log(np.exp(values - peak).sum(axis=axis))


def zeta_sweep(log_x, cost, a, gamma, eta):
    """sinkhorn.py:47-51."""
    return eta * (np.log(a) - _lse(log_x + (gamma[None, :] - cost) / eta, axis=1))


def gamma_sweep(log_x, cost, b, zeta, eta):
    """sinkhorn.py:54-58."""
    return eta * (np.log(b) - _lse(log_x + (zeta[:, None] - cost) / eta, axis=0))


def column_error(log_x, cost, b, zeta, gamma, eta) -> float:
    """sinkhorn.py:42-44 + 61-65."""
    s = log_x + (zeta[:, None] + gamma[None, :] - cost) / eta
    return float(np.linalg.norm(np.exp(s).sum(axis=0) - b))


def warm_start(log_x, cost, a, b, eta, warm_tol, gamma0=None, zeta0=None, max_sweeps=DEFAULT_SWEEP_CAP):
    """sinkhorn.py:68-103 — returns (gamma recentred, zeta shifted, sweeps)."""
    m, n = cost.shape
    gamma = np.zeros(n) if gamma0 is None else np.asarray(gamma0, dtype=np.float64)
    zeta = np.zeros(m) if zeta0 is None else np.asarray(zeta0, dtype=np.float64)
    sweeps = 0
    for _ in range(max_sweeps):
        zeta = zeta_sweep(log_x, cost, a, gamma, eta)
        sweeps += 1
        if column_error(log_x, cost, b, zeta, gamma, eta) < warm_tol:
            break
        gamma = gamma_sweep(log_x, cost, b, zeta, eta)
    else:
        raise OracleError("WarmStartStalled", f"{max_sweeps} sweeps")
    drift = gamma.sum() / n
    return gamma - drift, zeta + drift, sweeps


# --------------------------------------------------------------------------
# outer loop  (bregman_outer.py)
# --------------------------------------------------------------------------

@dataclass
class SolveResult:
    log_plan: np.ndarray
    rounded: np.ndarray
    objective: float
    kkt: float
    outer_iters: int
    newton_total: int
    cg_total: int
    gamma: np.ndarray
    zeta: np.ndarray
    records: list


def solve(cost, a, b, eta, kkt_tol=1e-11, mu0=1e-4, mu_floor=1e-11, min_dim_scale=True,
          warm_tol=1e-3, max_outer=300, max_inner=500, cg_rel_tol=1e-10, cg_max_iters=None,
          sigma=1e-4, beta=0.8) -> SolveResult:
    """bregman_outer.py:62-159 — the IBSN outer loop (trajectory as dicts)."""
    m, n = cost.shape
    scale = float(min(m, n)) if min_dim_scale else 1.0
    log_x = product_log_plan(a, b)
    gamma = np.zeros(n)
    zeta = np.zeros(m)
    newton_total = cg_total = 0
    records = []
    kkt_value = math.inf
    rounded = None
    obj = math.nan
    outer_iters = 0
    for k in range(max_outer):
        mu_k = mu(k, mu0, mu_floor)
        gamma, zeta, _ = warm_start(log_x, cost, a, b, eta, warm_tol, gamma, zeta)
        res = inner(log_x, cost, a, b, gamma, eta, mu_k, scale, max_inner, sigma, beta,
                    cg_rel_tol, cg_max_iters)
        zeta = zeta_sweep(log_x, cost, a, res.gamma, eta)     # bregman_outer.py:123-126
        gamma = res.gamma
        log_x = res.candidate
        outer_iters = k + 1
        newton_total += res.newton_iters
        cg_total += res.cg_total
        rounded = round_plan(np.exp(log_x), a, b)            # bregman_outer.py:51-59
        obj = float((cost * rounded).sum())
        if not np.isfinite(obj):
            raise OracleError("NumericalFailure", f"objective {obj!r}")
        kkt_value = kkt(rounded, gamma, cost, a, b)["delta_kkt"]
        records.append(dict(outer_k=k, inner_total=newton_total, cg_total=cg_total,
                            objective=obj, kkt=kkt_value, grad_norm=res.grad_norm,
                            stop=res.stop, newton=res.newton_iters, cg=res.cg_total))
        if kkt_value < kkt_tol:
            break
    return SolveResult(log_x, rounded, obj, kkt_value, outer_iters, newton_total, cg_total,
                       gamma, zeta, records)


def eot_solve(cost, a, b, eta, kkt_tol, warm_tol=1e-3, max_inner=500, cg_rel_tol=1e-10, cg_max_iters=None,
              sigma=1e-4, beta=0.8, min_dim_scale=True):
    """bregman_outer.py:284-327 — one entropic subproblem on the all-ones
    reference plan (log X = 0): warm start, Newton to the gradient target
    kkt_tol (pre-check off), metrics of the candidate.  Returns (candidate
    log plan, rounded plan, objective, kkt, newton_iters, cg_total, gamma,
    grad_norm)."""
    m, n = cost.shape
    scale = float(min(m, n)) if min_dim_scale else 1.0
    log_x = np.zeros((m, n))
    gamma, _, _ = warm_start(log_x, cost, a, b, eta, warm_tol)
    res = inner(log_x, cost, a, b, gamma, eta, 0.0, scale, max_inner, sigma, beta, cg_rel_tol, cg_max_iters,
                grad_target=kkt_tol)
    rounded = round_plan(np.exp(res.candidate), a, b)
    obj = float((cost * rounded).sum())
    kkt_value = kkt(rounded, res.gamma, cost, a, b)["delta_kkt"]
    return res.candidate, rounded, obj, kkt_value, res.newton_iters, res.cg_total, res.gamma, res.grad_norm


def ibsink_solve(cost, a, b, eta, kkt_tol=1e-11, mu0=1e-4, mu_floor=1e-11, min_dim_scale=True, max_outer=300,
                 max_inner=500):
    """bregman_outer.py:191-281 — outer loop with alternating dual sweeps as
    the inner solver.  Returns (log plan, rounded, objective, kkt,
    outer_iters, sweep_total, records)."""
    m, n = cost.shape
    scale = float(min(m, n)) if min_dim_scale else 1.0
    log_x = product_log_plan(a, b)
    gamma, zeta = np.zeros(n), np.zeros(m)
    sweep_total = 0
    records = []
    rounded, obj, kkt_value, outer_iters = None, math.nan, math.inf, 0
    for k in range(max_outer):
        mu_k = mu(k, mu0, mu_floor)
        cand = None
        sweeps = 0
        err = math.inf
        for _ in range(max_inner):
            zeta = zeta_sweep(log_x, cost, a, gamma, eta)
            sweeps += 1
            chi = log_x + (zeta[:, None] + gamma[None, :] - cost) / eta          # sinkhorn.py:41-43
            err = float(np.linalg.norm(np.exp(chi).sum(axis=0) - b))
            if err < mu_k:
                cand = clamp_log_plan(chi)
                if bregman(round_plan(np.exp(cand), a, b), cand) <= scale * mu_k:
                    break
                cand = None
            gamma = gamma_sweep(log_x, cost, b, zeta, eta)
        if cand is None:
            zeta = zeta_sweep(log_x, cost, a, gamma, eta)
            sweeps += 1
            chi = log_x + (zeta[:, None] + gamma[None, :] - cost) / eta
            err = float(np.linalg.norm(np.exp(chi).sum(axis=0) - b))
            cand = clamp_log_plan(chi)
        log_x = cand
        outer_iters = k + 1
        sweep_total += sweeps
        rounded = round_plan(np.exp(log_x), a, b)
        obj = float((cost * rounded).sum())
        kkt_value = kkt(rounded, gamma, cost, a, b)["delta_kkt"]
        records.append(dict(outer_k=k, inner_total=sweep_total, objective=obj, kkt=kkt_value, grad_norm=err))
        if kkt_value < kkt_tol:
            break
    return log_x, rounded, obj, kkt_value, outer_iters, sweep_total, records
