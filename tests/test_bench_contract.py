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
    assert "whole graph" in cb["sample"]  # the reference's run_bench over the whole graph, no extrapolation
    assert cb["physical_cores"] >= 1 and "threads per core" in cb["smt"]
    assert d["e2e"] == {"value": d["value"], "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["gpu_launches"] == 0


def test_reference_arm_other_ranks_exit_quietly():
    """under torchrun only rank 0 runs and prints the reference arm"""
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    assert run_bench("--impl", "reference", "--gpus", "2", "--workload", "c1", "--steps", "1", env=env).strip() == ""


def test_gpus_flag_must_match_world_size():
    """a torchrun environment whose WORLD_SIZE differs from --gpus fails loudly"""
    env = dict(os.environ, RANK="0", WORLD_SIZE="2", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "c1",
                        "--steps", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr


def test_gpus_n_relaunches_one_rank_per_gpu():
    """`bench.py --gpus 2` without a torchrun environment starts two ranks
    (torch.distributed.run) and rank 0 prints one line with n_gpus 2 and the
    same config as the other arm would"""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po

    if not po.has_ref():
        pytest.skip("oracle/_ref not built")
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    lines = [l for l in run_bench("--impl", "reference", "--gpus", "2", "--workload", "c1", "--steps", "1",
                                  env=env).splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"
    assert d["config"]["parallelism"].startswith("monomials x2")
    import bench

    class A:
        points = 0
        shard = ""

    assert d["config"] == bench.config_for(A, "c1", 2)


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


def test_reference_arm_never_maps_the_product_library():
    """the reference arm generates inputs and counts flops with the reference
    library itself: libpse_b200.so is never mapped into that process"""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po

    if not po.has_ref():
        pytest.skip("oracle/_ref not built")
    code = ("import sys, json; sys.argv=['bench.py','--impl','reference','--workload','c1','--steps','1'];"
            "import bench; bench.main(); maps=open('/proc/self/maps').read();"
            "print(json.dumps({'pse': 'libpse_b200' in maps, 'ref': 'libpseval_ref' in maps}))")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    flags = json.loads(r.stdout.strip().splitlines()[-1])
    assert flags == {"pse": False, "ref": True}
