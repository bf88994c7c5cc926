"""clock64 trace of one ILU sweep (FWI_ILU_TRACE): per level, stager arrival at the barrier,
barrier exit, warp 0's rows done, stager prefetch issued. Prints the per-level split."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c1_problem, random_kkt  # noqa: E402

lev = int(sys.argv[1]) if len(sys.argv) > 1 else 21
adj = len(sys.argv) > 2 and sys.argv[2] == "adj"
q = c1_problem()
rng = np.random.default_rng(3)
q.u = rng.standard_normal(q.K * q.n) + 1j * rng.standard_normal(q.K * q.n)
q.r = rng.standard_normal(q.survey.num_data) + 0j
st = fw.GnState(q, exact=False, ilu_level=lev)
b = rng.standard_normal(q.n) + 1j * rng.standard_normal(q.n)
st.solve(b, fw.PrecondMode.ilu, adj)
path = "/tmp/ilu_trace.bin"
os.environ["FWI_ILU_TRACE"] = path
st.solve(b, fw.PrecondMode.ilu, adj)
t = np.fromfile(path, dtype=np.int64).reshape(-1, 5).astype(np.float64)
st_, a_, b1, b_, b2 = t[:, 0], t[:, 1], t[:, 2], t[:, 3], t[:, 4]
print(f"levels {len(t)}, cycles/level median {np.median(np.diff(st_)):.0f}")
print(f"  loads+phase A: {np.median(a_ - st_):.0f}  barrier 1: {np.median(b1 - a_):.0f}  "
      f"phase B: {np.median(b_ - b1):.0f}  barrier 2: {np.median(b2 - b_):.0f}  to next: {np.median(st_[1:] - b2[:-1]):.0f}")
