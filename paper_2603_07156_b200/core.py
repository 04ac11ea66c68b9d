"""Problem, configuration and log-plan types of the drop-in solver.

Mirrors pkg/src/otibsn/core.py of the reference: same class names, fields,
defaults, validation messages and exception classes, so ``OtProblem`` /
``SolverConfig`` / ``LogPlan`` built for the reference can be rebuilt here
unchanged.  The differences are storage only: arrays may be numpy (host) or
torch CUDA tensors (device), and a ``LogPlan`` produced by the CUDA path
stays in HBM in the padded row layout of libotb (leading dimension
``round_up(n, 32)``) until ``.log_entries`` is read.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np

from .errors import InvalidCost, MarginalNotNormalized, MarginalNotPositive, ShapeMismatch

LOG_FLOOR = -1e6            # core.py:24
MARGINAL_SUM_TOL = 1e-12    # core.py:27


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


class RowShardCost:
    """The rows [row0, row0 + rows.shape[0]) of an m x n cost matrix, held
    on this rank's GPU (multi-GPU runs build only their own rows: config 5's
    C is 20 GB).  ``OtProblem(RowShardCost(...), a, b)`` has the GLOBAL shape
    (m, n); a session created with the matching row range (distributed
    ``row_range``) uses the local tensor in place.  ``rows`` may be a padded
    view (stride (ld, 1))."""

    def __init__(self, rows, row0: int, m: int):
        if not (_is_torch(rows) and rows.dim() == 2):
            raise ShapeMismatch("RowShardCost needs a 2-D torch tensor of local rows")
        if not 0 <= row0 <= row0 + rows.shape[0] <= m:
            raise ShapeMismatch("row shard outside the matrix")
        self.rows = rows
        self.row0 = int(row0)
        self.m = int(m)

    @property
    def shape(self) -> tuple[int, int]:
        return (self.m, int(self.rows.shape[1]))

    @property
    def ndim(self) -> int:
        return 2

    @property
    def is_cuda(self) -> bool:
        return bool(self.rows.is_cuda)


def _as_float_array(x, ndim: int):
    """core.py:30-34; torch tensors are kept (as contiguous float64)."""
    if isinstance(x, RowShardCost):
        return x
    if _is_torch(x):
        import torch

        t = x.detach().to(torch.float64)
        if t.dim() != ndim:
            raise ShapeMismatch(f"expected {ndim}-dimensional array, got shape {tuple(t.shape)}")
        # row-major with padded rows (stride (ld, 1), ld >= n) is kept as is:
        # the device path reads such a matrix in place
        padded_rows = ndim == 2 and t.stride(1) == 1 and t.stride(0) >= t.shape[1]
        return t if padded_rows else t.contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if arr.ndim != ndim:
        raise ShapeMismatch(f"expected {ndim}-dimensional array, got shape {arr.shape}")
    return arr


def host(x) -> np.ndarray:
    """numpy view/copy of an array that may live on the device."""
    if _is_torch(x):
        return x.detach().cpu().numpy()
    return np.asarray(x)


@dataclass(frozen=True, eq=False)
class OtProblem:
    """core.py:37-62 — cost matrix (m, n) and the two marginals."""

    cost: object
    source_marginal: object
    target_marginal: object

    def __post_init__(self):
        object.__setattr__(self, "cost", _as_float_array(self.cost, 2))
        object.__setattr__(self, "source_marginal", _as_float_array(self.source_marginal, 1))
        object.__setattr__(self, "target_marginal", _as_float_array(self.target_marginal, 1))

    @property
    def shape(self) -> tuple[int, int]:
        return tuple(self.cost.shape)


class InnerScale(enum.Enum):
    """core.py:65-69."""

    MIN_DIM = "min_dim"
    ONE = "one"


@dataclass(frozen=True)
class SolverConfig:
    """core.py:72-128 — identical fields, defaults and validation."""

    eta: float
    mu0: float = 1e-4
    mu_floor: float = 1e-11
    inner_scale: InnerScale = InnerScale.MIN_DIM
    warm_tol: float = 1e-3
    kkt_tol: float = 1e-11
    max_outer: int = 300
    max_inner: int = 500
    cg_rel_tol: float = 1e-10
    cg_max_iters: int | None = None
    armijo_sigma: float = 1e-4
    armijo_beta: float = 0.8
    seed: int = 0
    log_inner_kkt: bool = False
    # extension (not in the reference, which runs plain CG): None = plain CG
    # (krylov.py, the parity default) or "jacobi" = Jacobi-preconditioned CG
    # on the same Newton systems with the same stopping test
    cg_preconditioner: str | None = None

    def __post_init__(self):
        for name in ("eta", "mu0", "mu_floor", "warm_tol", "kkt_tol", "cg_rel_tol"):
            if not getattr(self, name) > 0:
                raise ValueError(f"{name} must be positive")
        for name in ("armijo_sigma", "armijo_beta"):
            if not 0.0 < getattr(self, name) < 1.0:
                raise ValueError(f"{name} must lie in (0, 1)")
        for name in ("max_outer", "max_inner"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be at least 1")
        if self.cg_preconditioner not in (None, "jacobi"):
            raise ValueError("cg_preconditioner must be None or 'jacobi'")


class LogPlan:
    """core.py:131-156 — transport plan in the log domain, clamped at LOG_FLOOR.

    Construct from a numpy array or a (m, n) torch tensor exactly like the
    reference (NaN / +inf raise ``InvalidCost``; entries are clamped).  The
    CUDA path produces plans that already live in the padded device layout;
    those are wrapped with :meth:`from_padded` without a round trip.
    """

    __slots__ = ("_host", "_dev", "_shape", "__weakref__")

    def __init__(self, log_entries):
        arr = _as_float_array(log_entries, 2)
        if _is_torch(arr) and not arr.is_cuda:
            # host tensor (e.g. pinned): validated and clamped on the device
            # right after its upload (device_padded), raising the same error
            self._host = None
            self._dev = ("host", arr)
            self._shape = tuple(arr.shape)
        elif _is_torch(arr):
            import torch

            _check_plan_tensor(arr)
            self._host = None
            self._dev = ("dense", torch.clamp_min(arr, LOG_FLOOR))
            self._shape = tuple(arr.shape)
        else:
            if np.isnan(arr).any() or (arr == np.inf).any():
                raise InvalidCost("log plan contains NaN or +inf entries")
            self._host = np.maximum(arr, LOG_FLOOR)
            self._dev = None
            self._shape = arr.shape

    @classmethod
    def from_padded(cls, padded, n: int) -> "LogPlan":
        """Wrap a device buffer (m, ld) whose first n columns are a valid,
        already clamped log plan (written by libotb)."""
        obj = cls.__new__(cls)
        obj._host = None
        obj._dev = ("padded", padded)
        obj._shape = (int(padded.shape[0]), int(n))
        return obj

    @property
    def shape(self) -> tuple[int, int]:
        return tuple(self._shape)

    @property
    def log_entries(self) -> np.ndarray:
        if self._host is None:
            kind, t = self._dev
            if kind == "host":
                arr = t.numpy()
                if np.isnan(arr).any() or (arr == np.inf).any():
                    raise InvalidCost("log plan contains NaN or +inf entries")
                self._host = np.maximum(arr, LOG_FLOOR)
                return self._host
            t = t[:, : self._shape[1]] if kind == "padded" else t
            self._host = _to_host(t)
        return self._host

    def device_padded(self, ld: int, device):
        """(m, ld) float64 CUDA tensor with the plan in columns [0, n)."""
        import torch

        check = False
        if self._dev is not None:
            kind, t = self._dev
            if kind == "padded" and t.shape[1] == ld and t.device == device:
                return t
            src = t[:, : self._shape[1]] if kind == "padded" else t
            check = kind == "host"
        else:
            src = torch.from_numpy(self._host)
        m, n = self._shape
        out = torch.empty((m, ld), dtype=torch.float64, device=device)
        out[:, :n].copy_(src, non_blocking=True)
        if ld > n:
            out[:, n:].zero_()
        if check:   # core.py:141-145 in one native pass (count NaN/+inf, clamp at LOG_FLOOR)
            import ctypes

            from . import _lib

            bad = ctypes.c_int64()
            _lib.check(_lib.lib.otb_check_clamp_plan(out.data_ptr(), m, n, ld, float(LOG_FLOOR),
                                                     ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream),
                                                     ctypes.byref(bad)))
            if bad.value:
                raise InvalidCost("log plan contains NaN or +inf entries")
        self._dev = ("padded", out)
        return out

    def dense(self) -> np.ndarray:
        """core.py:151-153."""
        return np.exp(self.log_entries)

    def total_mass(self) -> float:
        return float(self.dense().sum())


def _check_plan_tensor(t) -> None:
    """core.py:143-144 on a tensor: NaN or +inf -> InvalidCost."""
    import torch

    if bool(torch.logical_or(t != t, t == float("inf")).any()):
        raise InvalidCost("log plan contains NaN or +inf entries")


def _to_host(t) -> np.ndarray:
    """Device -> host copy through (cached) pinned memory."""
    import torch

    if not t.is_cuda:
        return t.detach().numpy()
    out = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    out.copy_(t)
    return out.numpy()


def normalize_cost(raw_cost) -> np.ndarray:
    """core.py:159-175."""
    cost = np.ascontiguousarray(np.asarray(host(raw_cost), dtype=np.float64))
    if cost.ndim != 2:
        raise ShapeMismatch(f"expected 2-dimensional array, got shape {cost.shape}")
    if cost.size == 0:
        raise InvalidCost("cost matrix is empty")
    if np.isnan(cost).any() or np.isinf(cost).any():
        raise InvalidCost("cost matrix contains NaN or infinite entries")
    if (cost < 0).any():
        raise InvalidCost("cost matrix contains negative entries")
    peak = cost.max()
    if peak == 0.0:
        return cost.copy()
    return cost / peak


def validate(problem: OtProblem) -> None:
    """core.py:178-205 — same checks, order and exception classes.

    Device-resident problems are checked with reductions on the device."""
    cost, a, b = problem.cost, problem.source_marginal, problem.target_marginal
    m, n = problem.shape
    if m == 0 or n == 0:
        raise ShapeMismatch("cost matrix must be nonempty")
    if a.shape[0] != m:
        raise ShapeMismatch(f"source marginal has length {a.shape[0]}, cost has {m} rows")
    if b.shape[0] != n:
        raise ShapeMismatch(f"target marginal has length {b.shape[0]}, cost has {n} columns")
    if isinstance(cost, RowShardCost):   # each rank checks its own rows
        cost = cost.rows
    if _is_torch(cost):
        import torch

        if bool((~torch.isfinite(cost)).any()):
            raise InvalidCost("cost matrix contains NaN or infinite entries")
        if bool((cost < 0).any()):
            raise InvalidCost("cost matrix contains negative entries")
    else:
        if np.isnan(cost).any() or np.isinf(cost).any():
            raise InvalidCost("cost matrix contains NaN or infinite entries")
        if (cost < 0).any():
            raise InvalidCost("cost matrix contains negative entries")
    for name, vec in (("source", host(a)), ("target", host(b))):
        if not np.isfinite(vec).all() or (vec <= 0).any():
            raise MarginalNotPositive(f"{name} marginal has nonpositive or non-finite entries")
    for name, vec in (("source", host(a)), ("target", host(b))):
        drift = abs(vec.sum() - 1.0)
        if drift > MARGINAL_SUM_TOL:
            raise MarginalNotNormalized(
                f"{name} marginal sums to {vec.sum():.17g} (|drift| = {drift:.3g} > {MARGINAL_SUM_TOL:g})"
            )


def initial_plan(problem: OtProblem) -> LogPlan:
    """core.py:208-212 — log a_i + log b_j (computed on the host with numpy
    so that the device starts from the reference's exact bits)."""
    log_a = np.log(host(problem.source_marginal))
    log_b = np.log(host(problem.target_marginal))
    return LogPlan(log_a[:, None] + log_b[None, :])
