"""bench.py's JSON contract on the CPU: the reference arm (the oracle port
timed on the host) prints one line with the driver's keys, and our arm
refuses to run without a GPU instead of falling back to the CPU."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=300):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, cwd=ROOT, env=env)


def test_reference_arm_line():
    res = _run(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "0"])
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["metric"] == "newton_inner_iterations_per_s"
    assert line["value"] > 0 and line["higher_is_better"] is True and line["steps"] == 1
    assert line["cpu_baseline"]["kind"] in ("port", "reference") and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["e2e"]["value"] == pytest.approx(line["value"])


def test_our_arm_needs_a_gpu():
    res = _run(["--steps", "1", "--warmup", "0", "--no-cpu", "--no-solve"])
    assert res.returncode != 0
    assert "CUDA" in (res.stderr + res.stdout) or "GPU" in (res.stderr + res.stdout)


def test_cpu_row_sample_step_runs_the_reference():
    """The configs-4/5 CPU baseline: a row sample of one step through the
    reference's own functions (otibsn), K CG products exactly."""
    from oracle import cpu_step
    from paper_2603_07156_b200 import instances as I

    pts = I.uniform2d_points(3000, 2500, 1)

    def rows(k):
        return I.normalise(I.sq_dist(pts.x[:k], pts.y))

    st = cpu_step.RowSampleStep(rows, pts.a, pts.b, pts.eta, 3000, 5, 40)
    st.step()
    assert st.kind in ("reference", "port")
    if os.path.isdir("/root/reference/pkg/src"):
        assert st.kind == "reference"
    assert "rows 0..40 of 3000" in st.describe(1, 1.0)
