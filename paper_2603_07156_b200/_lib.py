"""ctypes binding of libotb.so (include/otb.h).

The library is the product: there is no CPU fallback.  Importing this
module on a machine where ``libotb.so`` is missing raises immediately, and
every entry point checks its status code and raises the exception class the
reference raises at the corresponding site (errors.STATUS_TO_ERROR).
"""

from __future__ import annotations

import ctypes as C
import glob
import os
from pathlib import Path

from . import errors

# OTB_LIB: an alternative build of the library (experiments: variants compiled
# with different -D knobs side by side)
LIB_PATH = Path(os.environ.get("OTB_LIB") or (Path(__file__).resolve().parent / "libotb.so"))

i64 = C.c_int64
dbl = C.c_double
vp = C.c_void_p


class EvalOut(C.Structure):
    _fields_ = [("value", dbl), ("grad_norm", dbl)]


class CgOut(C.Structure):
    _fields_ = [("iters", i64), ("residual", dbl), ("status", C.c_int), ("pad", C.c_int)]


class NewtonParams(C.Structure):
    _fields_ = [("sigma", dbl), ("beta", dbl), ("cg_rel_tol", dbl), ("cg_max_iters", i64),
                ("rho_override", dbl)]


class NewtonOut(C.Structure):
    _fields_ = [("t", dbl), ("slope", dbl), ("rho", dbl), ("value_before", dbl),
                ("value_after", dbl), ("grad_norm_before", dbl), ("grad_norm_after", dbl),
                ("cg_iters", i64), ("nnz", i64), ("trials", i64), ("cg_residual", dbl)]


class TestOut(C.Structure):
    _fields_ = [("bregman", dbl), ("objective", dbl), ("delta_p", dbl), ("delta_d", dbl),
                ("delta_c", dbl), ("delta_kkt", dbl), ("sum_x", dbl), ("deficit", dbl)]

    __test__ = False


class InnerOut(C.Structure):
    _fields_ = [("value0", dbl), ("grad_norm0", dbl), ("stepped", C.c_int), ("tested", C.c_int),
                ("newton", NewtonOut), ("test", TestOut)]


class WarmOut(C.Structure):
    _fields_ = [("sweeps", i64), ("err", dbl)]


# name -> (restype, argtypes); the export list of include/otb.h
SIGNATURES = {
    "otb_abi_version": (C.c_int, []),
    "otb_last_error": (C.c_char_p, []),
    "otb_create": (C.c_int, [C.POINTER(vp), i64, i64, i64, i64, i64, C.c_int, vp]),
    "otb_destroy": (C.c_int, [vp]),
    "otb_set_stream": (C.c_int, [vp, vp]),
    "otb_nccl_get_unique_id": (C.c_int, [C.c_char_p, vp]),
    "otb_attach_nccl": (C.c_int, [vp, C.c_char_p, vp, C.c_int, C.c_int]),
    "otb_group_create": (C.c_int, [C.POINTER(vp), C.c_int]),
    "otb_group_destroy": (C.c_int, [vp]),
    "otb_group_abort": (C.c_int, [vp]),
    "otb_attach_group": (C.c_int, [vp, vp, C.c_int]),
    "otb_set_cg_precond": (C.c_int, [vp, C.c_int]),
    "otb_bind": (C.c_int, [vp, vp, vp, vp, vp, vp, dbl, i64, dbl, dbl, dbl]),
    "otb_eval": (C.c_int, [vp, vp, vp, vp, vp, C.POINTER(EvalOut)]),
    "otb_sparsify": (C.c_int, [vp, vp, vp, dbl, C.POINTER(i64)]),
    "otb_csr_export": (C.c_int, [vp, vp, vp, vp, vp]),
    "otb_hess_apply": (C.c_int, [vp, vp, dbl, vp]),
    "otb_cg": (C.c_int, [vp, dbl, vp, dbl, i64, vp, C.POINTER(CgOut)]),
    "otb_newton_step": (C.c_int, [vp, vp, vp, vp, C.POINTER(NewtonParams), C.POINTER(NewtonOut)]),
    "otb_recover_round": (C.c_int, [vp, vp, vp, vp, C.c_int, C.c_int, C.POINTER(TestOut)]),
    "otb_materialize_rounded": (C.c_int, [vp, vp, i64]),
    "otb_warm_start": (C.c_int, [vp, vp, vp, vp, dbl, i64, C.POINTER(WarmOut)]),
    "otb_zeta_from_lse": (C.c_int, [vp, vp]),
    "otb_sinkhorn_zeta": (C.c_int, [vp, vp, vp, vp, C.POINTER(dbl)]),
    "otb_sinkhorn_gamma": (C.c_int, [vp, vp, vp, vp]),
    "otb_scaled_plan": (C.c_int, [vp, vp, vp, vp, vp]),
    "otb_init_plan": (C.c_int, [vp, vp]),
    "otb_materialize_p": (C.c_int, [vp, vp, vp, vp, i64]),
    "otb_info": (C.c_int, [vp, C.POINTER(i64)]),
    "otb_launch_count": (C.c_int, [vp, C.POINTER(i64)]),
    "otb_sq_dist": (C.c_int, [vp, vp, i64, i64, C.c_int, i64, vp, i64, C.POINTER(dbl), vp]),
    "otb_scale_cost": (C.c_int, [vp, i64, i64, i64, dbl, vp]),
    "otb_selftest_div": (C.c_int, [vp, i64, dbl, vp]),
    "otb_selftest_log": (C.c_int, [vp, i64, vp]),
    "otb_selftest_exp": (C.c_int, [vp, i64, vp]),
    "otb_selftest_tab": (C.c_int, [vp, i64, vp]),
    "otb_inner_iteration": (C.c_int, [vp, vp, vp, vp, vp, C.c_int, dbl, dbl, vp, vp, vp]),
    "otb_set_cost_norm_sq": (C.c_int, [vp, vp]),
    "otb_check_clamp_plan": (C.c_int, [vp, i64, i64, i64, dbl, vp, vp]),
    "otb_cg_trace": (C.c_int, [vp, vp, i64, C.POINTER(i64)]),
    "otb_round_dense": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, i64, C.POINTER(dbl), vp]),
    "otb_bregman_dense": (C.c_int, [vp, i64, vp, i64, i64, i64, C.POINTER(dbl), vp]),
    "otb_kkt_dense": (C.c_int, [vp, i64, vp, i64, vp, vp, vp, i64, i64, vp, C.POINTER(dbl), vp]),
    "otb_hessian_dense": (C.c_int, [vp, i64, i64, i64, vp, vp, dbl, vp, vp]),
    "otb_prof_enable": (C.c_int, [vp, C.c_int]),
    "otb_prof_read": (C.c_int, [vp, C.POINTER(dbl), C.POINTER(i64), C.POINTER(dbl), C.c_int]),
}


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -m paper_2603_07156_b200.build` "
            "(there is no CPU fallback for the solver path)"
        )
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.otb_abi_version() != 1:
        raise ImportError("libotb ABI version mismatch")
    return lib


lib = _load()


def check(status: int) -> None:
    if status != 0:
        msg = lib.otb_last_error().decode(errors="replace")
        raise errors.STATUS_TO_ERROR.get(status, errors.DeviceError)(msg)


def nccl_path() -> str:
    """The torch-bundled libnccl.so.2 (one NCCL per process)."""
    env = os.environ.get("OTB_NCCL_PATH")
    if env:
        return env
    try:
        import nvidia.nccl  # type: ignore

        for base in nvidia.nccl.__path__:
            hits = glob.glob(os.path.join(base, "lib", "libnccl.so*"))
            if hits:
                return sorted(hits)[0]
    except Exception:  # pragma: no cover - layout differs
        pass
    return "libnccl.so.2"
