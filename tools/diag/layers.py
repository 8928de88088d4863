"""Per-layer conv times (phase stamps) of one workload, for the planner's path."""
import os, sys, argparse
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench
import paper_2101_10881_b200 as pe
ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c3")
ap.add_argument("--m", type=int, default=1)
a = ap.parse_args()
pid, d, m, _, _ = bench.WORKLOADS[a.workload]
m = a.m or m
n, N, nvars, idx, st = bench.make_static(pid, d, m, range(1))
g = pe.build_jobgraph_shape(n, d, nvars, idx)
plan = pe.DevicePlan(g, m, "real", 0, 1)
plan.upload(st, 1)
for _ in range(3):
    r = plan.execute(1, detail=True)
cl, al = plan.layer_ms()
print(a.workload, m, plan.conv_path(1), "conv", round(r.conv_ms, 4), "layers", len(cl))
print(" ".join(f"{v*1000:.1f}" for v in cl))
