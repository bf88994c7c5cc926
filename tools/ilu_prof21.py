"""ILU(21) preconditioner applies on config 1 (ncu capture of the ILU sweep kernels)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c1_problem, random_kkt  # noqa: E402

lev = int(sys.argv[1]) if len(sys.argv) > 1 else 21
q = c1_problem()
rng = np.random.default_rng(3)
q.u = rng.standard_normal(q.K * q.n) + 1j * rng.standard_normal(q.K * q.n)
q.r = rng.standard_normal(q.survey.num_data) + 0j
st = fw.GnState(q, exact=False, ilu_level=lev)
x = fw.KktVector.from_host(st, random_kkt(q, 1))
for _ in range(2):
    y = fw.precond_apply(st, x, fw.PrecondMode.ilu)
st.synchronize()
print(fw.norm(y))
