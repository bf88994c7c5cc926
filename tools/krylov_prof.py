"""Kernel timeline of one exact-preconditioned GMRES solve on config 1 (run under
ncu --profile-from-start off; the solve is bracketed by cudaProfilerStart/Stop)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c1_problem, c3_problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
q = c1_problem() if name == "c1" else c3_problem()
if name == "c3":
    q.epsilon = 2.8e10
q.d_obs = fw.simulate(q)
st = fw.GnState(q, exact=True)
for _ in range(2):
    fw.fsgn_gmres_step(st, fw.FsgnOptions(tol=1e-3, maxit=30, ecg_stride=0))
torch.cuda.synchronize()
torch.cuda.profiler.start()
ds, log = fw.fsgn_gmres_step(st, fw.FsgnOptions(tol=1e-3, maxit=30, ecg_stride=0))
torch.cuda.profiler.stop()
print("iterations", log.iterations(), "wall", log.entries[-1].wall_time)
