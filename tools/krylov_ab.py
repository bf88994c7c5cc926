"""Krylov iterations/s with and without the pipelined GMRES loop (FWI_GMRES_SYNC=1 = the synchronous
loop): C1 exact / ILU(4) and C3 exact, tol 1e-3, restart 30, ecg_stride 0; median of 5 solves
(python tools/krylov_ab.py [c1|c3|all])."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c1_problem, c3_problem  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"


def time_solve(state, mode, label):
    o = fw.FsgnOptions(mode=mode, restart=30, tol=1e-3, maxit=60, ecg_stride=0)
    out = {}
    for sync in ("0", "1"):
        if sync == "1":
            os.environ["FWI_GMRES_SYNC"] = "1"
        else:
            os.environ.pop("FWI_GMRES_SYNC", None)
        for _ in range(2):
            fw.fsgn_gmres_step(state, o)
        runs = []
        for _ in range(5):
            t0 = time.perf_counter()
            ds, log = fw.fsgn_gmres_step(state, o)
            runs.append((log.entries[-1].wall_time, time.perf_counter() - t0, log.iterations()))
        runs.sort()
        wt, tw, it = runs[2]
        out["sync" if sync == "1" else "pipelined"] = {"its": it, "it_per_s": round(it / wt, 1),
                                                       "us_per_it": round(wt / it * 1e6, 1),
                                                       "step_wall_ms": round(tw * 1e3, 3)}
    os.environ.pop("FWI_GMRES_SYNC", None)
    print(json.dumps({"solve": label, "env": {k: v for k, v in os.environ.items() if k.startswith("FWI_")},
                      **out}), flush=True)


if which in ("c1", "all"):
    q = c1_problem()
    q.d_obs = fw.simulate(q)
    s1 = fw.GnState(q, exact=True, ilu_level=4)
    time_solve(s1, fw.PrecondMode.exact, "C1 exact")
    time_solve(s1, fw.PrecondMode.ilu, "C1 ILU(4)")
    s1.close()
if which in ("c3", "all"):
    q3 = c3_problem(freq_hz=3.0)
    q3.d_obs = fw.simulate(q3)
    q3.epsilon = 2.8e10
    s3 = fw.GnState(q3, exact=True)
    time_solve(s3, fw.PrecondMode.exact, "C3 exact")
