"""Device vs oracle on the failing Euler instance (m=4, it=2), per conv mode."""
import os, sys, subprocess
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]
import pyoracle as po
from instances import md_instance
from test_accuracy import single_monomial, dev_eval
rng = np.random.default_rng(513)
for it in range(3):
    p, deg = single_monomial(md_instance(rng, 4, nmax=6, Nmax=2, dmax=5, with_exponents=True))
ref = po.evaluate(p, "port")[0]
dv = dev_eval(p)
print("n", p.n, "d", p.d, "exps", p.exps, "idx", p.idx, "nvars", p.nvars)
diff = np.argwhere(ref.view(np.int64) != dv.view(np.int64))
print("mode", os.environ.get("PSE_CONV_MODE", "auto"), "differing words:", len(diff), diff[:10].tolist())
if len(diff):
    q, s, k = diff[0]
    print("ref", ref[:, s, k], "dev", dv[:, s, k])
