"""A/B the exact block-solve sweep variants (FWI_EXACT_SWEEP=warp|cta|legacy) on C1 and C3."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c1_problem, c3_problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
p = c1_problem() if name == "c1" else c3_problem(freq_hz=3.0)
p.d_obs = fw.simulate(p)
st = fw.GnState(p, exact=True)
rng = np.random.default_rng(0)
b = (rng.standard_normal((8, p.grid.n)) + 1j * rng.standard_normal((8, p.grid.n)))
x = st.solve(b)
xa = st.solve(b, adjoint=True)
np.save(f"gpurun_out/sweep_{os.environ.get("FWI_EXACT_SWEEP", "warp")}_{name}.npy", np.stack([x, xa]))
for _ in range(3):
    fw.fsgn_gmres_step(st, fw.FsgnOptions(mode=fw.PrecondMode.exact, tol=1e-12, maxit=5, ecg_stride=0))
rates = []
for _ in range(5):
    t = time.perf_counter()
    ds, log = fw.fsgn_gmres_step(st, fw.FsgnOptions(mode=fw.PrecondMode.exact, tol=1e-3, maxit=30, ecg_stride=0))
    rates.append(log.iterations() / (time.perf_counter() - t))
print(os.environ.get("FWI_EXACT_SWEEP", "warp"), name, "its", log.iterations(), "res", log.final_residual(),
      "it/s", " ".join(f"{r:.1f}" for r in rates), "dsnorm", float(np.linalg.norm(ds)))
t = time.perf_counter()
for _ in range(20):
    st.solve(b)
print("  solve(8 rhs) ms", (time.perf_counter() - t) / 20 * 1e3)
