import os, sys
sys.path.insert(0, "/root/repo")
from paper_2204_06489_b200 import api as fw
from paper_2204_06489_b200.problem import c3_problem
q3 = c3_problem(freq_hz=3.0); q3.d_obs = fw.simulate(q3); q3.epsilon = 2.8e10
s3 = fw.GnState(q3, exact=True)
o = fw.FsgnOptions(mode=fw.PrecondMode.exact, restart=30, tol=1e-3, maxit=60, ecg_stride=0)
fw.fsgn_gmres_step(s3, o)
os.environ["FWI_GMRES_TRACE"] = "1"; os.environ["FWI_GMRES_SYNC"] = "1"
fw.fsgn_gmres_step(s3, o)
