"""ILU preconditioner apply time and output hash per sweep schedule (FWI_ILU_SWEEP=sf|level,
FWI_ILU_SF_THREADS), on config 1 (ILU(4), ILU(21)) and config 3 (ILU(4), ILU(21)).

    FWI_ILU_SWEEP=level python tools/ilu_sf_probe.py
    python tools/ilu_sf_probe.py            # sync-free (default)
"""
import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c1_problem, c3_problem, random_kkt  # noqa: E402

mode = os.environ.get("FWI_ILU_SWEEP", "sf") + "/" + os.environ.get("FWI_ILU_SF_THREADS", "512")
cases = [("c1", c1_problem, 4), ("c1", c1_problem, 21), ("c3", lambda: c3_problem(freq_hz=3.0), 4),
         ("c3", lambda: c3_problem(freq_hz=3.0), 21)]
only = sys.argv[1:]
for name, mk, lev in cases:
    if only and f"{name}:{lev}" not in only:
        continue
    q = mk()
    rng = np.random.default_rng(3)
    q.u = (rng.standard_normal(q.K * q.n) + 1j * rng.standard_normal(q.K * q.n))
    q.r = rng.standard_normal(q.survey.num_data) + 0j
    st = fw.GnState(q, exact=False, ilu_level=lev)
    x = fw.KktVector.from_host(st, random_kkt(q, 1))
    y = fw.KktVector(st)
    for _ in range(2):
        fw.precond_apply(st, x, fw.PrecondMode.ilu, out=y)
    st.synchronize()
    reps = 10 if lev < 21 or name == "c1" else 3
    t0 = time.perf_counter()
    for _ in range(reps):
        fw.precond_apply(st, x, fw.PrecondMode.ilu, out=y)
    st.synchronize()
    ms = (time.perf_counter() - t0) / reps * 1e3
    h = hashlib.sha1(y.to_host().tobytes()).hexdigest()[:16]
    print(f"{mode:10s} {name} ILU({lev}) precond_apply {ms:8.3f} ms  out sha1 {h}", flush=True)
    st.close()
