"""One full-space Newton step at BASELINE config 5 (2048x1024, 10 Hz, K=256, R=1024) on one
B200: observed data by a device forward solve on the truth, then fwi::gn_step on the device
(exact factorisation, K forward solves, fsgn-gmres-exact to tol 1e-3, clamp, misfit re-solve).
GMRES restart 3 with the Krylov basis in pinned host memory (one KKT vector is 17.2 GB;
SURVEY §7 hard part 3)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c5_problem  # noqa: E402

restart = int(sys.argv[1]) if len(sys.argv) > 1 else 3
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 30
p = c5_problem()
t0 = time.perf_counter()
p.d_obs = fw.simulate(p)
t_sim = time.perf_counter() - t0
print(f"simulate (truth factor + {p.K} solves): {t_sim:.1f} s", flush=True)
cfg = fw.FwiConfig(solver="fsgn-gmres-exact", max_inner=maxit, inner_tol=1e-3, gmres_restart=restart)
t0 = time.perf_counter()
r = fw.gn_step(p, p.s, p.freq_hz, p.epsilon, cfg)
wall = time.perf_counter() - t0
log = r.log
its = log.iterations()
hist = [e.residual_norm for e in log.entries]
model_err0 = float(np.linalg.norm(p.s - p.s_true) / np.linalg.norm(p.s_true))
model_err1 = float(np.linalg.norm(r.s - p.s_true) / np.linalg.norm(p.s_true))
res = {"config": "C5 2048x1024 K=256 R=1024 10 Hz, fsgn-gmres-exact", "gmres_restart": restart,
       "max_inner": maxit, "inner_tol": 1e-3, "iterations": its, "converged": log.converged,
       "stagnated": log.stagnated, "final_residual": hist[-1], "residual_history": hist,
       "misfit_ini": r.misfit_ini, "misfit_fin": r.misfit_fin, "update_relnorm": r.update_relnorm,
       "model_error_start": model_err0, "model_error_after": model_err1,
       "gn_step_wall_s": wall, "gn_step_device_wall_s": r.wall_seconds, "simulate_s": t_sim,
       "krylov_wall_s": log.entries[-1].wall_time,
       "krylov_iters_per_s": its / log.entries[-1].wall_time if its else None}
print(json.dumps(res), flush=True)
with open("gpurun_out/c5_newton.json", "w") as f:
    json.dump(res, f, indent=1)
