"""Power-iteration estimate of ||J^H W^T W J|| (the Gauss-Newton Hessian without eps) at a
BASELINE config, to calibrate eps ~ 1e-2 ||J^H J|| as for config 1."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200 import problem as pr  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 8
p = {"c1": pr.c1_problem, "c3": pr.c3_problem, "c5": pr.c5_problem}[name]()
if len(sys.argv) > 3:
    p.freq_hz = float(sys.argv[3])
p.d_obs = fw.simulate(p)
p.epsilon = 1e-300  # H v - eps v with eps ~ 0
st = fw.GnState(p, exact=True)
v = np.random.default_rng(0).standard_normal(p.n)
v /= np.linalg.norm(v)
lam = 0.0
t0 = time.perf_counter()
for k in range(its):
    hv = fw.hessian_apply(st, v)
    lam = float(v @ hv)
    v = hv / np.linalg.norm(hv)
    print(f"{name} it {k}: rayleigh {lam:.4e}  ({time.perf_counter() - t0:.1f} s)", flush=True)
print(f"{name}: ||J^H J|| ~ {lam:.3e}; eps = 1e-2 * that = {1e-2 * lam:.3e}")
