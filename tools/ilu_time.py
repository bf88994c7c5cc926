"""ILU(4) preconditioner apply time on config 3 (vector beyond shared memory) and config 1."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c1_problem, c3_problem, random_kkt  # noqa: E402

for name, mk in (("c1", c1_problem), ("c3", c3_problem)):
    q = mk()
    q.d_obs = fw.simulate(q)
    st = fw.GnState(q, exact=False, ilu_level=4)
    x = fw.KktVector.from_host(st, random_kkt(q, 1))
    y = fw.KktVector(st)
    for _ in range(3):
        fw.precond_apply(st, x, fw.PrecondMode.ilu, out=y)
    st.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        fw.precond_apply(st, x, fw.PrecondMode.ilu, out=y)
    st.synchronize()
    print(name, "ILU(4) precond_apply ms", round((time.perf_counter() - t0) / 10 * 1e3, 3), "norm", fw.norm(y))
