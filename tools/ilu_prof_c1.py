"""ILU(4) preconditioner applies on config 1 (ncu capture of the shared-memory ILU sweep)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c1_problem, random_kkt  # noqa: E402

q = c1_problem()
q.d_obs = fw.simulate(q)
st = fw.GnState(q, exact=False, ilu_level=4)
x = fw.KktVector.from_host(st, random_kkt(q, 1))
for _ in range(3):
    y = fw.precond_apply(st, x, fw.PrecondMode.ilu)
print(fw.norm(y))
