"""Thresholded sparsification and the sparse Hessian operator (K2-K4).

Drop-in for pkg/src/otibsn/sparsify.py.  ``sparsify_p`` runs the fused
``sparsify`` kernel (recompute P from C and log X with the row statistics of
the cached eval, threshold, compact with ballot/prefix scans into a device
CSR, accumulate d = P_rho^T a).  ``SparseRowStochastic`` exposes the result
in the reference's layout (CSR of the m-1 off-anchor rows in original
order, anchor row apart) for tests; ``SparseHessianOp.matvec`` applies
H_rho on the device.
"""

from __future__ import annotations

import numpy as np

from .core import host
from .errors import TestOnlyLimit
from .semidual import RowSoftmaxCache

_SPECTRAL_MAX_DIM = 64


def choose_anchor(a) -> int:
    """sparsify.py:25-27 — smallest index attaining max(a)."""
    return int(np.argmax(host(a)))


def threshold_rho(eta: float, m: int, n: int, grad_norm: float) -> float:
    """sparsify.py:30-32."""
    return eta * grad_norm / (m * n)


class SparseRowStochastic:
    """sparsify.py:35-87 — host view of the device CSR of one sparsify call.

    Attributes follow the reference: ``row_offsets`` (m), ``col_indices``,
    ``values`` for the off-anchor rows in original order, ``anchor_index``
    and ``anchor_row`` (the unnormalised dense anchor row), ``n_cols``.
    """

    def __init__(self, session, nnz: int, anchor: int):
        self.session = session
        self.nnz_total = nnz
        self.anchor_index = anchor
        self.n_cols = session.n
        row_ptr, cols, vals, d = session.ops.csr_export(nnz)
        rp = row_ptr.cpu().numpy()
        cc = cols.cpu().numpy().astype(np.int64)
        vv = vals.cpu().numpy()
        self._d = d.cpu().numpy()
        i = anchor
        s, e = rp[i], rp[i + 1]
        anchor_row = np.zeros(self.n_cols)
        anchor_row[cc[s:e]] = vv[s:e]
        self.anchor_row = anchor_row
        keep = np.ones(cc.size, dtype=bool)
        keep[s:e] = False
        self.col_indices = cc[keep]
        self.values = vv[keep]
        lens = np.diff(rp)
        lens = np.delete(lens, i)
        self.row_offsets = np.zeros(lens.size + 1, dtype=np.int64)
        np.cumsum(lens, out=self.row_offsets[1:])

    @property
    def shape(self) -> tuple[int, int]:
        return (self.row_offsets.size, self.n_cols)

    def nnz(self) -> int:
        """sparsify.py:61-62 — stored values plus the dense anchor row."""
        return int(self.values.size) + int(self.anchor_row.size)

    def dense(self) -> np.ndarray:
        """sparsify.py:80-87 (test helper)."""
        m = self.row_offsets.size
        out = np.zeros((m, self.n_cols))
        i = self.anchor_index
        r = 0
        for row in range(m):
            if row == i:
                out[row] = self.anchor_row
                continue
            s, e = self.row_offsets[r], self.row_offsets[r + 1]
            out[row, self.col_indices[s:e]] = self.values[s:e]
            r += 1
        return out


def sparsify_p(cache: RowSoftmaxCache, rho: float, anchor: int) -> SparseRowStochastic:
    """sparsify.py:90-127 on the device.  ``rho`` and ``anchor`` may be
    forced (the reference's signature); the cache's eval is re-armed."""
    s = cache.session
    s.bind(s.eta, anchor)
    s.ops.eval(cache.plan_t, cache.gamma_t)
    nnz = s.ops.sparsify(cache.plan_t, cache.gamma_t, rho)
    rows = SparseRowStochastic(s, nnz, anchor)
    rows._op_state = (cache.plan_t, cache.gamma_t, rho, anchor)
    s._last_sparsify = rows
    return rows


class SparseHessianOp:
    """sparsify.py:130-159 — (diag(P_rho^T a) - P_rho^T diag(a) P_rho)/eta,
    applied by the ``hess_apply`` kernel on the CSR of ``p_rho``."""

    def __init__(self, p_rho: SparseRowStochastic, weights=None, eta: float | None = None, diag_cache=None):
        self.p_rho = p_rho
        self.session = p_rho.session
        self.eta = self.session.eta if eta is None else float(eta)
        self.diag_cache = p_rho._d if diag_cache is None else np.asarray(diag_cache)

    @property
    def dim(self) -> int:
        return self.p_rho.n_cols

    def _rearm(self):
        """Make the context's CSR the one of this operator (tests may build
        several operators on one session)."""
        s = self.session
        plan_t, gamma_t, rho, anchor = self.p_rho._op_state
        if getattr(s, "_last_sparsify", None) is not self.p_rho:
            s.bind(s.eta, anchor)
            s.ops.eval(plan_t, gamma_t)
            s.ops.sparsify(plan_t, gamma_t, rho)
            s._last_sparsify = self.p_rho

    def matvec(self, v, shift: float = 0.0) -> np.ndarray:
        self._rearm()
        s = self.session
        out = s.ops.hess_apply(s._vec(v), shift)
        return out[: s.n].cpu().numpy()

    def dense(self) -> np.ndarray:
        """sparsify.py:155-159 (test helper, small n)."""
        n = self.dim
        return np.stack([self.matvec(e) for e in np.eye(n)], axis=1)


def hessian_matvec_sparse(op: SparseHessianOp, v) -> np.ndarray:
    """sparsify.py:162-164."""
    return op.matvec(v)


def spectral_bounds_check(op: SparseHessianOp) -> tuple[float, float]:
    """sparsify.py:167-190 (test-only, n <= 64)."""
    n = op.dim
    if n > _SPECTRAL_MAX_DIM:
        raise TestOnlyLimit(f"dense eigendecomposition capped at n <= {_SPECTRAL_MAX_DIM}")
    h = op.dense()
    h = (h + h.T) / 2.0
    lam_max = float(np.linalg.eigvalsh(h)[-1])
    if n == 1:
        return 0.0, lam_max
    q, _ = np.linalg.qr(np.vstack([np.ones(n), np.eye(n)[1:]]).T)
    basis = q[:, 1:]
    lam_min_perp = float(np.linalg.eigvalsh(basis.T @ h @ basis)[0])
    return lam_min_perp, lam_max
