"""Per-step timeline of the warp-specialised exact sweep (CTA 0, warp 0) via FWI_SWEEP_TRACE."""
import os
import sys

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
for _ in range(3):
    st.solve(b)
path = f"gpurun_out/trace_{name}.bin"
if os.path.exists(path):
    os.remove(path)
os.environ["FWI_SWEEP_TRACE"] = path
st.solve(b)
del os.environ["FWI_SWEEP_TRACE"]
t = np.fromfile(path, dtype=np.uint64).astype(np.int64).reshape(-1, 8)
t -= t[0, 0]
gap = np.r_[t[1:, 0] - t[:-1, 5], 0]
t = (t / 1.965).astype(np.int64)  # SM cycles -> ns at 1965 MHz
print(f"{name}: steps {len(t)} total {t[-1, 5] / 1e3:.1f} us  per-step {t[-1, 5] / len(t):.0f} ns")
labs = ("full-wait", "rbar-wait", "w", "matvec", "push+store")
for k, lab in enumerate(labs):
    a = t[:, k + 1] - t[:, k]
    print(f"  {lab:13s} mean {a.mean():7.0f} ns  median {np.median(a):7.0f}  max {a.max():7.0f}")
for lab, a in (("gap", gap),):
    print(f"  {lab:13s} mean {a.mean():7.0f} ns  median {np.median(a):7.0f}  max {a.max():7.0f}")
