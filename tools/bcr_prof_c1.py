"""One exact precond_apply on config 1 with cyclic reduction forced (FWI_EXACT_BCR=1; ncu launch-list driver)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c1_problem, random_kkt  # noqa: E402

q = c1_problem()
rng = np.random.default_rng(3)
q.u = rng.standard_normal(q.K * q.n) + 1j * rng.standard_normal(q.K * q.n)
q.r = rng.standard_normal(q.survey.num_data) + 0j
st = fw.GnState(q, exact=True)
v = fw.KktVector.from_host(st, random_kkt(q, 1))
y = fw.KktVector(st)
for _ in range(3):
    fw.precond_apply(st, v, fw.PrecondMode.exact, out=y)
st.synchronize()
print("done")
