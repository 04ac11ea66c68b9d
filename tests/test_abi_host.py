"""CPU tests: the C ABI library loads and exports every symbol of
include/otb.h, the status codes map onto the reference exceptions, and the
host-side logic (config validation, instances, trajectory CSV, row
partition) behaves like the reference."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "otb.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(otb_\w+)\(", text, flags=re.M)))


def test_library_exports_every_header_symbol():
    from paper_2603_07156_b200 import _lib

    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    syms = header_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} not bound in _lib.SIGNATURES"
    assert lib.otb_abi_version() == 1


def test_library_is_sm100a():
    import subprocess

    from paper_2603_07156_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_cpu_compute_without_gpu():
    """Creating a context without a driver fails loudly with a CUDA status
    (there is no CPU fallback)."""
    from paper_2603_07156_b200 import _lib, errors

    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = ctypes.c_void_p()
    st = _lib.lib.otb_create(ctypes.byref(p), 4, 4, 0, 4, 32, 0, None)
    assert st == errors.OTB_ERR_CUDA
    with pytest.raises(errors.DeviceError):
        _lib.check(st)


def test_status_codes_match_header():
    from paper_2603_07156_b200 import errors

    text = (ROOT / "include" / "otb.h").read_text()
    for name, val in re.findall(r"(OTB_ERR_\w+) = (\d+)", text):
        assert getattr(errors, name) == int(val)
    assert errors.STATUS_TO_ERROR[errors.OTB_ERR_NONFINITE] is errors.NumericalOverflow
    assert errors.STATUS_TO_ERROR[errors.OTB_ERR_LINESEARCH] is errors.LineSearchStalled
    assert errors.STATUS_TO_ERROR[errors.OTB_ERR_BAD_LOGPLAN] is errors.InvalidCost


def test_solver_config_validation_matches_reference():
    from paper_2603_07156_b200 import SolverConfig

    SolverConfig(eta=1e-2)
    with pytest.raises(ValueError):
        SolverConfig(eta=0.0)
    with pytest.raises(ValueError):
        SolverConfig(eta=1.0, armijo_beta=1.0)
    with pytest.raises(ValueError):
        SolverConfig(eta=1.0, max_inner=0)


def test_validate_and_logplan_errors():
    from paper_2603_07156_b200 import LogPlan, OtProblem, errors, validate

    a = np.array([0.5, 0.5])
    with pytest.raises(errors.MarginalNotNormalized):
        validate(OtProblem(np.ones((2, 2)), a, np.array([0.5, 0.6])))
    with pytest.raises(errors.MarginalNotPositive):
        validate(OtProblem(np.ones((2, 2)), a, np.array([1.0, 0.0])))
    with pytest.raises(errors.InvalidCost):
        validate(OtProblem(-np.ones((2, 2)), a, a))
    with pytest.raises(errors.ShapeMismatch):
        validate(OtProblem(np.ones((2, 3)), a, a))
    lp = LogPlan(np.array([[-2e6, 0.0]]))
    assert lp.log_entries[0, 0] == -1e6
    with pytest.raises(errors.InvalidCost):
        LogPlan(np.array([[np.inf]]))


def test_instances_reproduce_reference_recipes():
    """Config generators are deterministic and satisfy the reference's
    validation (marginals sum to 1 within 1e-12, cost normalised)."""
    from paper_2603_07156_b200 import OtProblem, instances, validate

    inst = instances.config(1, 0)
    validate(OtProblem(inst.cost, inst.a, inst.b))
    assert inst.cost.max() == 1.0 and inst.cost.shape == (1000, 1000)
    inst2 = instances.config(1, 0)
    assert np.array_equal(inst.cost, inst2.cost) and np.array_equal(inst.a, inst2.a)
    g = instances.grid_histograms(8, 0)
    validate(OtProblem(g.cost, g.a, g.b))
    assert g.cost.max() == pytest.approx(2 * (7 / 8) ** 2)


def test_trajectory_csv_roundtrip_and_clock():
    from paper_2603_07156_b200 import errors
    from paper_2603_07156_b200.trajectory import Trajectory, TrajectoryRecord

    t = Trajectory()
    t.record(TrajectoryRecord(0, 1, 10, 0.5, 0.25, 1e-3, 1e-4))
    t.record(TrajectoryRecord(1, 2, 20, 0.75, 0.125, 1e-7, 1e-8, gap=1e-9))
    again = Trajectory.from_csv(t.to_csv())
    assert again.records == t.records
    with pytest.raises(errors.ClockError):
        t.record(TrajectoryRecord(2, 3, 30, 0.1, 0.1, 0.1, 0.1))


def test_trajectory_csv_bytes_match_reference_text():
    """The CSV text the reference's Trajectory.to_csv wrote for these records
    (generated in the build container from pkg/src/otibsn/trajectory.py)."""
    import math

    from paper_2603_07156_b200.trajectory import Trajectory, TrajectoryRecord

    expected = ("outer_k,inner_total,cg_total,wall_seconds,objective,kkt,grad_norm,gap\n"
                "0,1,5,0.10000000000000001,1.2345678901234567,0.001,2.4999999999999999e-07,\n"
                "1,3,17,0.25,1.2,9.9999999999999995e-07,1.0000000000000001e-09,0.00123\n")
    t = Trajectory()
    t.record(TrajectoryRecord(0, 1, 5, 0.1, 1.2345678901234567, 1e-3, 2.5e-7, None))
    t.record(TrajectoryRecord(1, 3, 17, 0.25, 1.2, 1e-6, 1e-9, 0.00123))
    assert t.to_csv() == expected
    assert Trajectory.from_csv(expected).to_csv() == expected
    for bad, exc, msg in [((2, 3, 17, 0.3, math.nan, 1e-6, 1e-9), ValueError, "non-finite objective"),
                          ((0, 3, 17, 0.3, 1.0, 1e-6, 1e-9), ValueError, "outer iteration index went backwards"),
                          ((2, 3, 17, 0.3, 1.0, 1e-6, 1e-9, math.inf), ValueError, "non-finite gap")]:
        with pytest.raises(exc, match=msg):
            t.record(TrajectoryRecord(*bad))


def test_row_partition():
    from paper_2603_07156_b200.distributed import anchor_owner, row_range

    for m in (1, 7, 4096, 50000, 65536):
        for w in (1, 2, 3, 4, 8):
            spans = [row_range(m, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    assert anchor_owner(4095, 4096, 8) == 7
    assert anchor_owner(0, 4096, 8) == 0


def test_mu_schedule():
    from paper_2603_07156_b200.bregman_outer import MuSchedule, mu

    s = MuSchedule()
    assert mu(s, 0) == 1e-4 and mu(s, 9) == pytest.approx(1e-6) and mu(s, 10**6) == 1e-11
