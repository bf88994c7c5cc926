"""Block cyclic reduction vs the Schur sweeps (FWI_EXACT_BCR=1|0): solve agreement, residual
probe, and exact precond_apply / GMRES-iteration time on configs 1 and 3.

    python tools/bcr_probe.py
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c1_problem, c3_problem, random_kkt  # noqa: E402


def run(name, mk, mode):
    os.environ["FWI_EXACT_BCR"] = mode
    q = mk()
    rng = np.random.default_rng(3)
    q.u = rng.standard_normal(q.K * q.n) + 1j * rng.standard_normal(q.K * q.n)
    q.r = rng.standard_normal(q.survey.num_data) + 0j
    t0 = time.perf_counter()
    st = fw.GnState(q, exact=True)
    tf = time.perf_counter() - t0
    b = np.random.default_rng(5).standard_normal(q.n) + 1j * np.random.default_rng(6).standard_normal(q.n)
    x = st.solve(b, fw.PrecondMode.exact, False)
    xa = st.solve(b, fw.PrecondMode.exact, True)
    v = fw.KktVector.from_host(st, random_kkt(q, 1))
    y = fw.KktVector(st)
    for _ in range(3):
        fw.precond_apply(st, v, fw.PrecondMode.exact, out=y)
    st.synchronize()
    reps = 20
    t0 = time.perf_counter()
    for _ in range(reps):
        fw.precond_apply(st, v, fw.PrecondMode.exact, out=y)
    st.synchronize()
    tp = (time.perf_counter() - t0) / reps
    out = y.to_host()
    print(f"{name} bcr={mode}: factor {tf:.3f} s (probe {st.exact_probe_residual:.2e}), precond_apply "
          f"{tp * 1e3:.3f} ms", flush=True)
    st.close()
    return x, xa, out


for name, mk in (("C1", c1_problem), ("C3", lambda: c3_problem(freq_hz=3.0))):
    a = run(name, mk, "0")
    b = run(name, mk, "1")
    for lab, u, w in zip(("solve", "adjoint solve", "precond"), a, b):
        print(f"  {lab}: bcr vs sweeps rel {np.linalg.norm(u - w) / np.linalg.norm(u):.2e}")
