"""conv time of gen_benchmark(pid, d, m) through the planner's path (PSE_CONV_MODE to force)."""
import os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2101_10881_b200 as pe
for spec in sys.argv[1:]:
    pid, d, m = spec.split(":")
    d, m = int(d), int(m)
    pr = pe.gen_benchmark(pid, d, m, seed=7)
    g = pe.build_jobgraph_shape(pr.n, pr.d, pr.nvars, pr.indices)
    plan = pe.DevicePlan(g, m, "real", 0, 1)
    plan.upload(pr.stat, 1)
    for _ in range(2):
        plan.execute(1)
    ts = [plan.execute(1) for _ in range(5)]
    print(f"{os.environ.get('PSE_CONV_MODE', 'auto'):>6} {pid} d={d} m={m} {plan.conv_path(1):>10}: conv "
          f"{statistics.median(r.conv_ms for r in ts):.4f} ms device {statistics.median(r.device_ms for r in ts):.4f} ms", flush=True)
