"""Time one workload's conv stage with a tuning build of the engine
(PSE_LIB_VARIANT=<name> selects libpse_b200_<name>.so; see build.py) and
print a checksum of the value/gradient series so that variants can be
compared for bit-identity. Not a bench number: a quick A/B tool."""
import argparse
import hashlib
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2101_10881_b200 as pe  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--m", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
pid, d, m, _, _ = bench.WORKLOADS[a.workload]
m = a.m or m
n, N, nvars, idx, st = bench.make_static(pid, d, m, range(1))
g = pe.build_jobgraph_shape(n, d, nvars, idx)
plan = pe.DevicePlan(g, m, "real", 0, 1)
plan.upload(st, 1)
plan.execute(1)
conv, dev = [], []
for _ in range(a.reps):
    r = plan.execute(1)
    conv.append(r.conv_ms)
    dev.append(r.device_ms)
vg, _ = plan.download(1)
h = hashlib.sha1(vg.tobytes()).hexdigest()[:12]
print(f"{os.environ.get('PSE_LIB_VARIANT', 'default'):>10} {a.workload} m={m} {plan.conv_path(1):>8}: "
      f"conv {statistics.median(conv):8.3f} ms  device {statistics.median(dev):8.3f} ms  vg {h}", flush=True)
