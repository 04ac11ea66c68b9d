"""Semi-dual objective, row softmax and gradient on the device (K1).

Drop-in for pkg/src/otibsn/semidual.py.  ``compute_p`` runs the fused
``eval`` kernel (one streaming pass over C and log X): it produces the
per-row log-normalisers, the objective and the gradient P^T a - b without
ever materialising P.  ``RowSoftmaxCache.p`` materialises P on demand for
tests (the reference's dense cache, semidual.py:38-48).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .core import LogPlan, OtProblem, _is_torch, host
from .session import session_for


@dataclass(frozen=True)
class DualState:
    """semidual.py:21-35 — column dual gamma (numpy or CUDA tensor) and its
    outer generation."""

    gamma: object = field(repr=False)
    generation: int = 0

    def __post_init__(self):
        g = self.gamma
        if _is_torch(g):
            import torch

            g = g.detach().to(torch.float64).reshape(-1).contiguous()
        else:
            g = np.ascontiguousarray(np.asarray(g, dtype=np.float64))
        object.__setattr__(self, "gamma", g)


class RowSoftmaxCache:
    """Device-backed replacement of semidual.py:38-48.

    Holds the session, the plan and dual it was evaluated at, the per-row
    log-normalisers, the objective value and the gradient.  ``p`` and
    ``row_logsumexp`` are host (numpy) views produced on first access.
    """

    def __init__(self, session, plan_t, gamma_t, lse_t, grad_t, value, grad_norm):
        self.session = session
        self.plan_t = plan_t
        self.gamma_t = gamma_t
        self.lse_t = lse_t
        self.grad_t = grad_t
        self.value = float(value)
        self.grad_norm = float(grad_norm)
        self._p = None

    @property
    def row_logsumexp(self) -> np.ndarray:
        return self.lse_t[: self.session.m_loc].cpu().numpy()

    @property
    def p(self) -> np.ndarray:
        if self._p is None:
            s = self.session
            s.ops.eval(self.plan_t, self.gamma_t)          # re-arm the row statistics
            self._p = s.ops.materialize_p(self.plan_t, self.gamma_t).cpu().numpy()
        return self._p


def _gamma_tensor(session, gamma):
    g = gamma.gamma if isinstance(gamma, DualState) else gamma
    return session._vec(g)


def compute_p(logplan: LogPlan, gamma: DualState, problem: OtProblem, eta: float) -> RowSoftmaxCache:
    """semidual.py:55-87.  Raises NumericalOverflow like the reference."""
    s = session_for(problem, eta)
    plan_t = s.plan(logplan)
    gam = _gamma_tensor(s, gamma)
    lse = s.new_vec(s.m_loc)
    grad = s.new_vec()
    value, gnorm = s.ops.eval(plan_t, gam, lse, grad)
    return RowSoftmaxCache(s, plan_t, gam, lse, grad, value, gnorm)


def semidual_value(cache: RowSoftmaxCache, gamma: DualState, problem: OtProblem, eta: float) -> float:
    """semidual.py:90-95 — L = -b.gamma + eta a.lse (reduced in the eval kernel)."""
    return cache.value


def semidual_gradient(cache: RowSoftmaxCache, problem: OtProblem) -> np.ndarray:
    """semidual.py:98-100 — g = P^T a - b."""
    return cache.grad_t[: cache.session.n].cpu().numpy()


def zeta_from_cache(cache: RowSoftmaxCache, problem: OtProblem, eta: float) -> np.ndarray:
    """semidual.py:117-119 — eta (log a - lse)."""
    s = cache.session
    s.ops.eval(cache.plan_t, cache.gamma_t)
    z = s.new_vec(s.m_loc)
    s.ops.zeta_from_lse(z)
    return z[: s.m_loc].cpu().numpy()


def hessian_matvec_exact(cache: RowSoftmaxCache, problem: OtProblem, eta: float, v) -> np.ndarray:
    """semidual.py:103-114 — (diag(P^T a) - P^T diag(a) P) v / eta with the
    dense P of ``cache`` (materialised in HBM, then otb_hessian_dense: row
    dots P v, column sums P^T a and P^T (a P v), one output pass)."""
    import ctypes as C

    from . import _lib

    s = cache.session
    s.ops.eval(cache.plan_t, cache.gamma_t)          # re-arm the row statistics
    P = s.ops.materialize_p(cache.plan_t, cache.gamma_t)
    vd = s._vec(v)
    out = s.new_vec()
    m_loc, n = s.m_loc, s.n
    a_loc = s.a[s.row_begin:s.row_end]
    _lib.check(_lib.lib.otb_hessian_dense(P.data_ptr(), n, m_loc, n, a_loc.data_ptr(), vd.data_ptr(), float(eta),
                                          out.data_ptr(), C.c_void_p(s.torch.cuda.current_stream().cuda_stream)))
    return out[:n].cpu().numpy()
