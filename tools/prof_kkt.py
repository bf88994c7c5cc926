"""Small driver for ncu captures of the hot kernels (not a benchmark)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import _abi  # noqa: E402
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c1_problem, c2_problem, random_kkt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--what", default="apply", choices=["apply", "apply32", "precond", "fsgn"])
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
if a.what in ("apply", "apply32"):
    p = c2_problem()
    st = fw.GnState(p, exact=False, c64=(a.what == "apply32"))
    prec = _abi.FWI_C64 if a.what == "apply32" else _abi.FWI_C128
    x0 = random_kkt(p, 1)
    x = fw.KktVector.from_host(st, x0.astype("float32") if prec == _abi.FWI_C64 else x0, prec)
    y = fw.KktVector(st, prec)
    for _ in range(a.reps):
        fw.kkt_apply(st, x, y)
    st.synchronize()
else:
    q = c1_problem()
    q.d_obs = fw.simulate(q)
    st = fw.GnState(q, exact=True, ilu_level=4)
    if a.what == "precond":
        x = fw.KktVector.from_host(st, random_kkt(q, 1))
        for mode in (fw.PrecondMode.exact, fw.PrecondMode.ilu):
            for _ in range(a.reps):
                fw.precond_apply(st, x, mode)
    else:
        fw.fsgn_gmres_step(st, fw.FsgnOptions(tol=1e-3, maxit=30, ecg_stride=0))
    st.synchronize()
print("done")
