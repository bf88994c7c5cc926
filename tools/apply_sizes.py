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
c64 = len(sys.argv) > 2 and sys.argv[2] == "c64"  # complex64 mode
p = {"c1": c1_problem, "c2": c2_problem, "c3": c3_problem}[cfg]()
st = fw.GnState(p, exact=False, c64=c64)
n, K = p.n, p.K
alg = (40 * K * n + 12 * n) if c64 else (80 * K * n + 24 * n)
prec = fw._abi.FWI_C64 if c64 else fw._abi.FWI_C128
xs = [fw.KktVector.from_host(st, random_kkt(p, 11 + i).astype("float32" if c64 else "float64"), prec)
      for i in range(2)]
ys = [fw.KktVector(st, prec) for _ in range(2)]
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
print(json.dumps({"cfg": cfg + (" c64" if c64 else ""), "kernel": st.kkt_kernel(prec).split(" (")[0], "env": env, "us": round(t * 1e6, 2), "frac": round(alg / t / 1e9 / peak, 3)}))
