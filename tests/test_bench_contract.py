"""The driver's bench.py contract: one JSON line with the required keys (the reference arm runs on
CPU here; the GPU arm is checked on a small config on the GPU box)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def _check_common(line):
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"):
        assert key in line, key
    assert line["config"]["workload"]
    assert line["higher_is_better"] is True and line["unit"] == "points/s"
    assert line["value"] > 0
    for key in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert key in line["e2e"], key


def test_reference_arm_contract():
    line = _run(["--impl", "reference", "--config", "2", "--steps", "2", "--warmup", "1"])
    _check_common(line)
    assert line["impl"] == "reference"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_gpu_arm_contract():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    line = _run(["--config", "3", "--steps", "3", "--warmup", "3"])
    _check_common(line)
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] == 3
    rf = line["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in rf, key
    assert 0 < rf["frac"] < 1
    assert line["gpu_launches"] > 0
    for key in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert key in line["clocks"], key
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] > 0 and cb["cores"] >= 1 and cb["sample"]
    assert line["parity"]["rel_err_vs_oracle"] <= 1e-12
    for leg in ("merged", "collapse", "corner_peak", "frontier_kernel"):
        assert leg in line, leg


def test_reference_arm_loads_only_the_oracle():
    """--impl reference runs the CPU oracle alone: the product library must not be mapped into the
    process (the arm's sample is chosen by oracle/ itself)."""
    code = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--config', '5', "
            "'--steps', '1', '--warmup', '1']; runpy.run_path('bench.py', run_name='__main__'); "
            "maps = open('/proc/self/maps').read(); "
            "assert 'libsg_b200' not in maps, 'product library loaded'; "
            "assert 'liboracle_sg' in maps; print('MAPS_OK')")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "MAPS_OK" in out.stdout
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][0])
    assert line["config"]["points"] == 27521113876
    assert 0.5e7 < line["config"]["sample_points_per_step"] < 2e7
