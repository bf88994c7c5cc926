"""Kernel launch list for exact solves under each sweep variant (run under ncu)."""
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
for v in ("warp", "cta"):
    os.environ["FWI_EXACT_SWEEP"] = v
    for _ in range(2):
        st.solve(b)
        st.solve(b, adjoint=True)
