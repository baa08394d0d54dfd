"""bench.py's output contract on CPU: the reference arm (`--impl reference`,
the reference's own CPU implementation compiled under oracle/_ref, or the
oracle port when that is absent) prints exactly one JSON line on stdout with
the keys the driver reads; everything else goes to stderr."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "cfg1",
                        "--steps", "2", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    if "unavailable" in d:
        pytest.skip(d["unavailable"])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "targets/s" and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["cpu_baseline"]["cores"] >= 1
    # the full workload, timed (no sub-box, no extrapolation), without the product library
    assert d["config"]["N"] == 10_000 and d["config"]["NT"] == 10_000
    assert d["steps"] == 2 and d["warmup"] == 1 and len(d["config"]["seconds_per_call"]) == 2
    assert d["config"]["product_library_loaded"] is False
    assert abs(d["ms_per_step"] - 1e3 * sorted(d["config"]["seconds_per_call"])[0]) <= \
        1e3 * abs(d["config"]["seconds_per_call"][1] - d["config"]["seconds_per_call"][0]) + 1e-6


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--impl", "reference"],
                       cwd=ROOT, capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


@pytest.mark.gpu
def test_gpu_arm_prints_one_json_line_with_driver_keys():
    r = subprocess.run([sys.executable, "bench.py", "--workload", "cfg1", "--steps", "3",
                        "--warmup", "3", "--no-cpu-baseline"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "roofline", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["gpu_launches"] > 0 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    rf = d["roofline"]
    assert rf["bound"] in ("hbm", "fp64") and 0 < rf["frac"] <= 1.0 and rf["peak"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
