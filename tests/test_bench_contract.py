"""bench.py's JSON contract, checked on CPU through the reference arm (the
reference's own CPU engine; the GPU arm needs a B200): one JSON line with the
metric, unit, config and the cpu_baseline / e2e keys the driver reads."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, env=None):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout


def test_reference_arm_json_line():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po

    if not po.has_ref():
        pytest.skip("oracle/_ref not built")
    lines = [l for l in run_bench("--impl", "reference", "--workload", "c1", "--steps", "2", "--warmup", "3").splitlines()
             if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert d["impl"] == "reference" and d["metric"] == base["metric"]
    assert d["unit"] == "TFLOPS" and d["higher_is_better"] is True and d["dtype"] == "f64"
    assert d["steps"] == 2 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["config"]["workload"].startswith("C1")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert "whole graph" in cb["sample"]  # C1 is small enough to run in full
    assert d["e2e"] == {"value": d["value"], "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["gpu_launches"] == 0


def test_reference_arm_other_ranks_exit_quietly():
    """under torchrun only rank 0 runs and prints the reference arm"""
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    assert run_bench("--impl", "reference", "--workload", "c1", "--steps", "1", env=env).strip() == ""


def test_reference_arm_precision_override():
    """--m runs the C3 sweep points (here the reference arm on C1's graph at m=1)"""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po

    if not po.has_ref():
        pytest.skip("oracle/_ref not built")
    d = json.loads(run_bench("--impl", "reference", "--workload", "c1", "--m", "1", "--steps", "1",
                             "--warmup", "3").strip())
    assert d["config"]["workload"].endswith("d=15, double (m=1)")
    assert d["value"] > 0
