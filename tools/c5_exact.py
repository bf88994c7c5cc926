"""C5 exact block solver on one B200: factorisation time, batched 256-RHS solve time,
solve residual ||A x - b||/||b|| (A applied by the device stencil through the KKT
operator's lambda row with du = x, ds = 0: out.lambda = A x)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c5_problem  # noqa: E402

p = c5_problem()
p.d_obs = np.zeros(p.survey.num_data, np.complex128)
t0 = time.perf_counter()
st = fw.GnState(p, exact=True)
t_state = time.perf_counter() - t0
print(f"state (exact factor + {st.K} forward solves): {t_state:.1f} s, device {st.device_bytes / 1e9:.1f} GB",
      flush=True)
K, n = st.K, st.n
rng = np.random.default_rng(1)
nr = 8
b = rng.standard_normal((nr, n)) + 1j * rng.standard_normal((nr, n))
t0 = time.perf_counter()
x = st.solve(b)
t_solve8 = time.perf_counter() - t0
# residual through the KKT lambda row: out.lambda_k = A du_k - w^2 u_k ds, ds = 0
xi = np.zeros(st.vec_len)
xv = xi[:2 * K * n].view(np.complex128).reshape(K, n)
xv[:nr] = x
out = fw.kkt_apply_host(st, xi)
la = out[2 * K * n + n:].view(np.complex128).reshape(K, n)[:nr]
res = float(np.linalg.norm(la - b) / np.linalg.norm(b))
t0 = time.perf_counter()
sc = st.solve_count(fw.PrecondMode.exact)
xk = fw.KktVector.from_host(st, np.random.default_rng(2).standard_normal(st.vec_len))
yk = fw.KktVector(st)
times = []
for _ in range(3):  # the first apply also allocates the solve's work buffers
    t1 = time.perf_counter()
    fw.precond_apply(st, xk, out=yk)
    _ = fw.norm(yk)
    times.append(time.perf_counter() - t1)
t_prec = sorted(times[1:])[0]
r = {"config": "C5 exact", "state_s": t_state, "solve_8rhs_s": t_solve8, "precond_apply_s": t_prec,
     "precond_apply_first_s": times[0],
     "solve_residual_rel": res, "device_bytes": st.device_bytes}
print(json.dumps(r), flush=True)
with open("gpurun_out/c5_exact.json", "w") as f:
    json.dump(r, f, indent=1)
