"""Complex-mode timing (no bench line: complex is not a BASELINE config):
p1 at d=152 in complex deca double, one point, CUDA-graph replay."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2101_10881_b200 as pe  # noqa: E402

for pid, m in (("p1", 10), ("p3", 10), ("p1", 4)):
    pr = pe.gen_benchmark(pid, 152, m, mode="cplx", seed=7)
    g = pe.build_jobgraph_shape(pr.n, pr.d, pr.nvars, pr.indices)
    plan = pe.DevicePlan(g, m, "cplx", 0, 1)
    plan.upload(pr.stat, 1)
    for _ in range(2):
        plan.execute(1)
    ts = [plan.execute(1).wall_ms for _ in range(3)]
    r = plan.execute(1, detail=True)
    print(f"complex {pid} d=152 m={m} ({plan.conv_path(1)}): {min(ts):.2f} ms, model TFLOPS "
          f"{r.double_op_count / min(ts) / 1e9:.1f}, alg Tops/s {r.alg_op_count / min(ts) / 1e9:.1f}")
