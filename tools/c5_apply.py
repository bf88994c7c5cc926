"""C5 (2048x1024, K=256, R=1024) batched KKT apply on one B200: throughput against the HBM
roofline plus size-independent self-consistency checks (the CPU reference cannot hold C5:
SURVEY §8(d)). Fields: u_k, r seeded CN(0,1); x: du, lambda ~ CN(0,1), ds ~ N(0,1).

  symmetry    <K x, y> = <x, K y> for the KKT inner product (the operator is symmetric)
  linearity   K(x + 2y) = K x + 2 K y
  determinism two applies of the same input are bitwise identical
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c5_problem, random_kkt  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
t0 = time.perf_counter()
p = c5_problem(with_u=True)
t_gen = time.perf_counter() - t0
t0 = time.perf_counter()
st = fw.GnState(p, exact=False)
t_state = time.perf_counter() - t0
p.u = None  # host copy no longer needed
K, n = st.K, st.n
print(f"C5 state: n={n} K={K} vec_len={st.vec_len} device_bytes={st.device_bytes / 1e9:.1f} GB "
      f"(gen {t_gen:.0f}s, ctx {t_state:.0f}s)", flush=True)
xh = random_kkt(p, 7)
x = fw.KktVector.from_host(st, xh)
del xh
kx = fw.kkt_apply(st, x)
y = kx.copy()
fw.scal(1.0 / fw.norm(kx), y)
ky = fw.kkt_apply(st, y)
a = fw.dot(kx, y)
b = fw.dot(x, ky)
sym = abs(a - b) / (fw.norm(kx) * fw.norm(y))
# linearity: t = x + 2y ; K t - (K x + 2 K y)
t = x.copy()
fw.axpy(2.0, y, t)
kt = fw.kkt_apply(st, t)
fw.axpy(-1.0, kx, kt)
fw.axpy(-2.0, ky, kt)
lin = fw.norm(kt) / (fw.norm(kx) + 2 * fw.norm(ky))
# determinism
kx2 = fw.kkt_apply(st, x)
fw.axpy(-1.0, kx, kx2)
det = fw.norm(kx2)
del t, kt, kx2
# timing: alternate two inputs (each 17.2 GB, far above L2) on the library stream
out = fw.KktVector(st)
ins = [x, y]
stream = st.stream_ptr()
for i in range(3):
    fw.kkt_apply(st, ins[i % 2], out)
sec = bench.timed_events(stream, lambda i: fw.kkt_apply(st, ins[i % 2], out), steps)
ms = sec / steps * 1e3
alg = 80 * K * n + 24 * n
peak = bench.peaks()[0]
res = {"config": "C5 2048x1024 K=256 R=1024 c128", "ms_per_apply": ms, "applies_per_s": 1e3 / ms,
       "algorithmic_bytes": alg, "achieved_gbs": alg / (ms * 1e-3) / 1e9,
       "frac_of_peak": alg / (ms * 1e-3) / 1e9 / peak, "peak_gbs": peak,
       "symmetry_rel": sym, "linearity_rel": lin, "determinism_abs": det, "steps": steps}
print(json.dumps(res), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/c5_apply.json", "w") as f:
    json.dump(res, f, indent=1)
