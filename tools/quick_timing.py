import os, sys, time, numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'oracle'))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_10881_b200 as pe
print(pe.device_info())
print('fp64 peak', pe.fp64_peak())
for (pid, d, m) in [('p1', 15, 2), ('p1', 152, 10)]:
    pr = pe.gen_benchmark(pid, d, m, seed=7)
    g = pe.build_jobgraph_shape(pr.n, pr.d, pr.nvars, pr.indices)
    plan = pe.DevicePlan(g, m, 'real', 0, 1)
    plan.upload(pr.stat, 1)
    for it in range(3):
        r = plan.execute(1, detail=True)
        print(pid, d, m, 'wall %.3f conv %.3f add %.3f ms' % (r.wall_ms, r.conv_ms, r.add_ms), 'model TFLOPS %.3f' % (r.double_op_count / r.wall_ms / 1e9), 'alg Tops/s %.3f' % (r.alg_op_count / r.wall_ms / 1e9))
    r = plan.execute(1, detail=False)
    print('graph wall', r.wall_ms)
