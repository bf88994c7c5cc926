"""Per-component device time (CUDA events on the library stream, 200 calls) of the pieces of
one GMRES iteration on config 1: precond_apply (2 batched exact solves), kkt_apply, dot."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c1_problem, c3_problem, random_kkt  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
q = c1_problem() if name == "c1" else c3_problem()
q.d_obs = fw.simulate(q)
st = fw.GnState(q, exact=True)
x = fw.KktVector.from_host(st, random_kkt(q, 1))
y = fw.KktVector(st)
sp = st.stream_ptr()
n = 200
for label, fn in (("precond_apply", lambda i: fw.precond_apply(st, x, out=y)),
                  ("kkt_apply", lambda i: fw.kkt_apply(st, x, y)),
                  ("axpy", lambda i: fw.axpy(0.5, x, y))):
    fn(0)
    t0 = time.perf_counter()
    sec = bench.timed_events(sp, fn, n)
    wall = time.perf_counter() - t0
    print(f"{name} {label:14s} device {sec / n * 1e6:8.1f} us/call   host wall {wall / n * 1e6:8.1f} us/call")
for _ in range(3):
    ds, log = fw.fsgn_gmres_step(st, fw.FsgnOptions(tol=1e-3, maxit=30, ecg_stride=0))
    print(f"{name} fsgn {log.iterations()} its  {log.entries[-1].wall_time / log.iterations() * 1e6:.0f} us/iter")
