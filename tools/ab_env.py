"""Interleaved in-process A/B of one FWI_* knob on a C1/C3 GMRES solve (the knob must be read per
call): python tools/ab_env.py NAME VAL_A VAL_B [c1|c3] [exact|ilu] [rounds]. Prints the median
it/s per value over `rounds` alternations of 3-solve medians."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c1_problem, c3_problem  # noqa: E402

name, va, vb = sys.argv[1:4]
cfg = sys.argv[4] if len(sys.argv) > 4 else "c1"
mode = sys.argv[5] if len(sys.argv) > 5 else "exact"
rounds = int(sys.argv[6]) if len(sys.argv) > 6 else 8
p = c1_problem() if cfg == "c1" else c3_problem()
p.d_obs = fw.simulate(p)
st = fw.GnState(p, exact=True, ilu_level=4)
o = fw.FsgnOptions(mode=getattr(fw.PrecondMode, mode), restart=30, tol=1e-3, maxit=60, ecg_stride=0)
res = {va: [], vb: []}
ref = None
for r in range(rounds):
    for v in (va, vb) if r % 2 == 0 else (vb, va):
        os.environ[name] = v
        fw.fsgn_gmres_step(st, o)
        ts = []
        for _ in range(3):
            ds, log = fw.fsgn_gmres_step(st, o)
            ts.append(log.iterations() / log.entries[-1].wall_time)
            h = log.residuals()
            ref = h if ref is None else ref
            assert h == ref, "residual history changed with the knob"
        res[v].append(statistics.median(ts))
print(json.dumps({"knob": name, "cfg": cfg, "mode": mode,
                  **{f"{name}={v}": round(statistics.median(x), 1) for v, x in res.items()},
                  "all": {v: [round(t) for t in x] for v, x in res.items()}}))
