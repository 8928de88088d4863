"""Short single-GPU run for ncu captures: stage one workload and execute it
`--reps` times (no timing output is a bench number)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2101_10881_b200 as pe  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--m", type=int, default=0, help="override the precision level")
a = ap.parse_args()
pid, d, m, _, _ = bench.WORKLOADS[a.workload]
m = a.m or m
n, N, nvars, idx, st = bench.make_static(pid, d, m, range(1))
g = pe.build_jobgraph_shape(n, d, nvars, idx)
plan = pe.DevicePlan(g, m, "real", 0, 1)
plan.upload(st, 1)
for _ in range(a.reps):
    r = plan.execute(1, detail=True)
print(f"{a.workload} m={m} ({plan.conv_path(1)}): wall {r.wall_ms:.3f} ms conv {r.conv_ms:.3f} add {r.add_ms:.3f}")
