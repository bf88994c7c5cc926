"""Driver for an ncu capture of the fused MGS sweep on config 3 (one exact-preconditioned GMRES
solve; the capture picks a late launch with ~20 basis vectors). Not a benchmark."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c3_problem  # noqa: E402

q = c3_problem(freq_hz=3.0)
q.d_obs = fw.simulate(q)
q.epsilon = 2.8e10
st = fw.GnState(q, exact=True)
ds, log = fw.fsgn_gmres_step(st, fw.FsgnOptions(tol=1e-3, maxit=25, ecg_stride=0))
print("iterations", log.iterations())
