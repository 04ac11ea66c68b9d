"""Conjugate gradients for the shifted Newton system (K5) on the device.

Drop-in for pkg/src/otibsn/krylov.py.  The whole loop runs in HBM: per
iteration one ``hess_apply`` kernel plus two fused vector kernels (curvature
+ alpha, then x/r update + convergence test + beta).  On one rank with
n <= 8192 the whole loop is ONE persistent cooperative kernel (k_cg_fused:
no host round trip until it ends); otherwise the iterations are launched in
batches of 16 and the host reads the solver status once per batch.  The iteration count and stopping
rule are the reference's (krylov.py:63-84): the device stops at exactly the
iteration the reference would.
"""

from __future__ import annotations

import numpy as np

from .sparsify import SparseHessianOp


def cg_solve(op: SparseHessianOp, shift: float, rhs, rel_tol: float = 1e-10, max_iters: int | None = None,
             *, preconditioner: str | None = None):
    """krylov.py:17-85 — solve (H + shift I) x = rhs from x0 = 0.

    ``op`` must be the device operator returned by this package's
    ``SparseHessianOp`` (the product path has no host callback).
    Returns (solution, iters, final_residual); raises InconsistentSystem /
    NotPositiveDefinite like the reference.  ``preconditioner="jacobi"``
    (extension) runs Jacobi PCG with the same stopping test on ||r||.
    """
    if not isinstance(op, SparseHessianOp):
        raise TypeError("cg_solve runs on the device operator (paper_2603_07156_b200.sparsify.SparseHessianOp)")
    op.session.set_precond(preconditioner)   # the Jacobi diagonal is accumulated by sparsify
    op._rearm()
    s = op.session
    n = s.n
    max_iters = 2 * n if max_iters is None else int(max_iters)
    x, iters, res = s.ops.cg(shift, s._vec(np.asarray(rhs, dtype=np.float64)), rel_tol, max_iters)
    return x[:n].cpu().numpy(), iters, res
