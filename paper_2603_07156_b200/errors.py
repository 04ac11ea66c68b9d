"""Exception hierarchy of the drop-in solver.

The class names, their base class and their meaning follow the reference
package one for one (pkg/src/otibsn/errors.py:4-65).  When the reference
package ``otibsn`` is importable in the same interpreter, every class here
ALSO subclasses its namesake in ``otibsn.errors``, so existing
``except otibsn.errors.X`` handlers catch this package's errors unchanged;
without it, catch ``paper_2603_07156_b200.errors.X``.  The CUDA library
reports failures as integer status codes (include/otb.h);
``STATUS_TO_ERROR`` maps each code onto the class the reference would raise
at the corresponding site.
"""

from __future__ import annotations

try:  # the reference's hierarchy, when installed alongside (drop-in catching)
    import otibsn.errors as _ref
except Exception:  # pragma: no cover - depends on the environment
    _ref = None


def _also(name: str) -> tuple:
    """The reference's class of the same name (as an extra base), if any."""
    cls = getattr(_ref, name, None) if _ref is not None else None
    return (cls,) if isinstance(cls, type) else ()


class OtibsnError(*(_also("OtibsnError") or (Exception,))):
    """Base class (errors.py:4)."""


class ShapeMismatch(OtibsnError, *_also("ShapeMismatch")):
    """Cost matrix and marginal dimensions disagree (errors.py:8)."""


class InvalidCost(OtibsnError, *_also("InvalidCost")):
    """NaN / infinite / negative cost, or a log plan with NaN/+inf (errors.py:12)."""


class MarginalNotPositive(OtibsnError, *_also("MarginalNotPositive")):
    """A marginal has a nonpositive entry (errors.py:16)."""


class MarginalNotNormalized(OtibsnError, *_also("MarginalNotNormalized")):
    """A marginal does not sum to one within tolerance (errors.py:20)."""


class NumericalOverflow(OtibsnError, *_also("NumericalOverflow")):
    """Stabilised row softmax produced a non-finite value (errors.py:24)."""


class InconsistentSystem(OtibsnError, *_also("InconsistentSystem")):
    """Unshifted singular system whose right-hand side leaves the range (errors.py:28)."""


class NotPositiveDefinite(OtibsnError, *_also("NotPositiveDefinite")):
    """CG met nonpositive curvature before convergence (errors.py:32)."""


class LineSearchStalled(OtibsnError, *_also("LineSearchStalled")):
    """Armijo backtracking exceeded its trial cap (errors.py:36)."""


class WarmStartStalled(OtibsnError, *_also("WarmStartStalled")):
    """Alternating dual sweeps hit the sweep cap (errors.py:40)."""


class NumericalFailure(OtibsnError, *_also("NumericalFailure")):
    """A solver produced a non-finite objective (errors.py:44)."""


class OracleTooLarge(OtibsnError, *_also("OracleTooLarge")):
    """Instance exceeds the exact LP oracle's size cap (errors.py:48)."""


class OracleFailed(OtibsnError, *_also("OracleFailed")):
    """Exact LP oracle failed to certify optimality (errors.py:52)."""


class TestOnlyLimit(OtibsnError, *_also("TestOnlyLimit")):
    """A test-only helper was called outside its supported range (errors.py:56)."""

    __test__ = False  # not a pytest test class


class LoadError(OtibsnError, *_also("LoadError")):
    """An input file could not be read as a valid instance (errors.py:60)."""


class ClockError(OtibsnError, *_also("ClockError")):
    """Recorded wall time went backwards (errors.py:64)."""


class DeviceError(RuntimeError):
    """CUDA / NCCL failure inside libotb (no reference counterpart)."""


# Status codes returned by every libotb entry point (include/otb.h).
OTB_OK = 0
OTB_ERR_NONFINITE = 1
OTB_ERR_NOT_PD = 2
OTB_ERR_INCONSISTENT = 3
OTB_ERR_LINESEARCH = 4
OTB_ERR_BAD_LOGPLAN = 5
OTB_ERR_WARMSTART = 6
OTB_ERR_ARG = 7
OTB_ERR_CUDA = 8
OTB_ERR_NCCL = 9
OTB_ERR_NOMEM = 10
OTB_ERR_OBJECTIVE = 11

STATUS_TO_ERROR = {
    OTB_ERR_NONFINITE: NumericalOverflow,        # semidual.py:85-86
    OTB_ERR_NOT_PD: NotPositiveDefinite,         # krylov.py:70-74
    OTB_ERR_INCONSISTENT: InconsistentSystem,    # krylov.py:57-58
    OTB_ERR_LINESEARCH: LineSearchStalled,       # inner_newton.py:94
    OTB_ERR_BAD_LOGPLAN: InvalidCost,            # core.py:143-144
    OTB_ERR_WARMSTART: WarmStartStalled,         # sinkhorn.py:100-101
    OTB_ERR_ARG: ValueError,
    OTB_ERR_CUDA: DeviceError,
    OTB_ERR_NCCL: DeviceError,
    OTB_ERR_NOMEM: MemoryError,
    OTB_ERR_OBJECTIVE: NumericalFailure,         # bregman_outer.py:54-55
}
