"""One exact precond_apply on config 3 with cyclic reduction (ncu launch-list driver)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c3_problem, random_kkt  # noqa: E402

q = c3_problem(freq_hz=3.0)
rng = np.random.default_rng(3)
q.u = rng.standard_normal(q.K * q.n) + 1j * rng.standard_normal(q.K * q.n)
q.r = rng.standard_normal(q.survey.num_data) + 0j
st = fw.GnState(q, exact=True)
v = fw.KktVector.from_host(st, random_kkt(q, 1))
y = fw.KktVector(st)
for _ in range(2):
    fw.precond_apply(st, v, fw.PrecondMode.exact, out=y)
st.synchronize()
print("done")
