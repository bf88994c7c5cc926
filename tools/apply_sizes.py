"""KKT apply time and HBM fraction at configs 1-3 for each K1 variant (env knobs are read per
plan, so each variant runs in its own process: python tools/apply_sizes.py [cfg])."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c1_problem, c2_problem, c3_problem, random_kkt  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
p = {"c1": c1_problem, "c2": c2_problem, "c3": c3_problem}[cfg]()
st = fw.GnState(p, exact=False)
n, K = p.n, p.K
alg = 80 * K * n + 24 * n
xs = [fw.KktVector.from_host(st, random_kkt(p, 11 + i)) for i in range(2)]
ys = [fw.KktVector(st) for _ in range(2)]
L = fw.lib()


def step(i):
    fw._check(L.fwi_dev_kkt_apply(st.h, xs[i & 1].h, ys[i & 1].h))


for i in range(20):
    step(i)
st.synchronize()
steps = 500
t = bench.timed_events(st.stream_ptr(), step, steps) / steps
peak = bench.peaks()[0]
env = {k: v for k, v in os.environ.items() if k.startswith("FWI_KKT")}
print(json.dumps({"cfg": cfg, "env": env, "us": round(t * 1e6, 2), "frac": round(alg / t / 1e9 / peak, 3)}))
