"""Binary A/B of two builds of libfwi_b200.so on a GMRES solve, interleaved, one process per
measurement: python tools/ab_lib.py LIB_A LIB_B [c1|c3] [exact|ilu] [rounds] [ilu_level].
Prints the median it/s per library and every sample."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, statistics
sys.path.insert(0, %r)
from paper_2204_06489_b200 import api as fw
from paper_2204_06489_b200.problem import c1_problem, c3_problem
cfg, mode, lvl = sys.argv[1], sys.argv[2], int(sys.argv[3])
p = c1_problem() if cfg == "c1" else c3_problem()
p.d_obs = fw.simulate(p)
st = fw.GnState(p, exact=(mode == "exact"), ilu_level=lvl)
o = fw.FsgnOptions(mode=getattr(fw.PrecondMode, mode), restart=30, tol=1e-3, maxit=60, ecg_stride=0)
for _ in range(2):
    fw.fsgn_gmres_step(st, o)
ts = []
for _ in range(7):
    ds, log = fw.fsgn_gmres_step(st, o)
    ts.append(log.iterations() / log.entries[-1].wall_time)
print(statistics.median(ts), log.iterations(), repr(log.residuals()[-1]))
""" % ROOT

a, b = sys.argv[1:3]
cfg = sys.argv[3] if len(sys.argv) > 3 else "c1"
mode = sys.argv[4] if len(sys.argv) > 4 else "exact"
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 4
lvl = sys.argv[6] if len(sys.argv) > 6 else "4"
res = {a: [], b: []}
last = {}
for r in range(rounds):
    for lib in (a, b) if r % 2 == 0 else (b, a):
        env = dict(os.environ, FWI_B200_LIB=os.path.abspath(lib))
        out = subprocess.run([sys.executable, "-c", CHILD, cfg, mode, lvl], env=env, check=True,
                             capture_output=True, text=True).stdout.split()
        res[lib].append(float(out[0]))
        last[lib] = out[1:]
print(json.dumps({"cfg": cfg, "mode": mode, "level": lvl,
                  **{lib: round(statistics.median(x), 1) for lib, x in res.items()},
                  "all": {lib: [round(t) for t in x] for lib, x in res.items()}, "last": last}))
