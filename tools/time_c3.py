"""Time the C3/C4 building blocks on the device (setup, exact/ILU Krylov)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c3_problem  # noqa: E402

p = c3_problem(freq_hz=float(sys.argv[1]) if len(sys.argv) > 1 else 3.0)
t = time.perf_counter()
p.d_obs = fw.simulate(p)
t_sim = time.perf_counter() - t
t = time.perf_counter()
st = fw.GnState(p, exact=True)
t_state = time.perf_counter() - t
t = time.perf_counter()
st.factor_ilu(4)
t_ilu = time.perf_counter() - t
print(f"simulate {t_sim:.2f}s  state(exact factor + {p.K} forward solves) {t_state:.2f}s  ilu(4) factor {t_ilu:.2f}s")
for mode in (fw.PrecondMode.exact, fw.PrecondMode.ilu):
    t = time.perf_counter()
    ds, log = fw.fsgn_gmres_step(st, fw.FsgnOptions(mode=mode, tol=1e-3, maxit=30, ecg_stride=0))
    print(mode.name, "its", log.iterations(), "conv", log.converged, "res", log.final_residual(),
          f"wall {time.perf_counter() - t:.2f}s  it/s {log.iterations() / log.entries[-1].wall_time:.1f}")
