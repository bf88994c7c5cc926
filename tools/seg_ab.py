"""Interleaved A/B of the exact factorisation's layout on a C1/C3 exact GMRES solve: one GnState
per FWI_EXACT_SEGMENTS value (read at factorisation time), solves alternated between them.
python tools/seg_ab.py [c1|c3] [rounds]. Prints the median it/s per layout and the largest
relative residual-history difference between them."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c1_problem, c3_problem  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 8
p = c1_problem() if cfg == "c1" else c3_problem()
p.d_obs = fw.simulate(p)
states = {}
for v in ("0", "1"):
    os.environ["FWI_EXACT_SEGMENTS"] = v
    states[v] = fw.GnState(p, exact=True)
o = fw.FsgnOptions(mode=fw.PrecondMode.exact, restart=30, tol=1e-3, maxit=60, ecg_stride=0)
res = {v: [] for v in states}
hist = {}
for r in range(rounds):
    for v in ("0", "1") if r % 2 == 0 else ("1", "0"):
        st = states[v]
        fw.fsgn_gmres_step(st, o)
        ts = []
        for _ in range(3):
            ds, log = fw.fsgn_gmres_step(st, o)
            ts.append(log.iterations() / log.entries[-1].wall_time)
            hist[v] = log.residuals()
        res[v].append(statistics.median(ts))
h0, h1 = hist["0"], hist["1"]
n = min(len(h0), len(h1))
dev = max(abs(a - b) / b for a, b in zip(h0[:n], h1[:n]))
print(json.dumps({"cfg": cfg, "segments=0": round(statistics.median(res["0"]), 1),
                  "segments=1": round(statistics.median(res["1"]), 1),
                  "iterations": [len(h0) - 1, len(h1) - 1], "max_rel_history_diff": dev,
                  "all": {v: [round(t) for t in x] for v, x in res.items()}}))
