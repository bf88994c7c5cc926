"""BASELINE configs 3/4: multi-frequency full-space Newton FWI on the Marmousi-like
section (384x128, 48 sources, 192 receivers), 3/5/7 Hz x N Newton steps each,
exact (C3) or ILU(p) (C4) block preconditioner. Observed data are device forward
solves on the truth. Writes a JSON report (one entry per Newton step)."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c3_problem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--solver", default="fsgn-gmres-exact")
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--freqs", default="3,5,7")
ap.add_argument("--ilu-level", type=int, default=4)
ap.add_argument("--max-inner", type=int, default=30)
ap.add_argument("--inner-tol", type=float, default=1e-3)
ap.add_argument("--out", default="")
ap.add_argument("--eps", default="auto", help="'auto' = 1e-2 ||J^H W^T W J|| per frequency at the start model "
                "(power iteration, the config-1 calibration rule), or a number")
a = ap.parse_args()
freqs = [float(f) for f in a.freqs.split(",")]
p = c3_problem()
t0 = time.perf_counter()
observed = {f: fw.simulate(p.__class__(**{**p.__dict__, "freq_hz": f})) for f in freqs}
t_data = time.perf_counter() - t0


def jhj_norm(f, its=10):
    q = p.__class__(**{**p.__dict__, "freq_hz": f, "epsilon": 1e-300, "d_obs": observed[f]})
    st = fw.GnState(q, exact=True)
    v = np.random.default_rng(0).standard_normal(q.n)
    v /= np.linalg.norm(v)
    lam = 0.0
    for _ in range(its):
        hv = fw.hessian_apply(st, v)
        lam = float(v @ hv)
        v = hv / np.linalg.norm(hv)
    st.close()
    return lam


eps = {f: (1e-2 * jhj_norm(f) if a.eps == "auto" else float(a.eps)) for f in freqs}
print("eps per frequency", eps, flush=True)
cfg = fw.FwiConfig(solver=a.solver, max_inner=a.max_inner, inner_tol=a.inner_tol, gmres_restart=30,
                   ilu_level=a.ilu_level, v_min=1400.0, v_max=5000.0)
t0 = time.perf_counter()
rep = fw.fwi_run(p, observed, p.s, eps, cfg, steps_per_frequency=a.steps)
wall = time.perf_counter() - t0
vt = p.meta["v_true"].ravel()
rows = []
for r in rep:
    v = 1.0 / np.sqrt(r.s)
    rows.append({"freq_hz": r.freq_hz, "outer_iterations": r.log.iterations(), "converged": r.log.converged,
                 "final_residual": r.log.final_residual(), "misfit_ini": r.misfit_ini, "misfit_fin": r.misfit_fin,
                 "update_relnorm": r.update_relnorm, "newton_step_s": r.wall_seconds,
                 "setup_s": r.setup_seconds, "host_ilu_factor_s": r.ilu_factor_seconds,
                 "krylov_s": r.krylov_seconds, "final_resolve_s": r.final_seconds,
                 "model_err_rel": float(np.linalg.norm(v - vt) / np.linalg.norm(vt)),
                 "inner_iterations": 0})
v0 = 1.0 / np.sqrt(p.s)
out = {"config": f"C3/C4 384x128 K=48 R=192, {a.solver}" + (f" ILU({a.ilu_level})" if "ilu" in a.solver else ""),
       "freqs": freqs, "epsilon": {str(k): v for k, v in eps.items()}, "steps_per_frequency": a.steps, "inner_tol": a.inner_tol, "max_inner": a.max_inner,
       "data_generation_s": t_data, "total_wall_s": wall,
       "mean_newton_step_s": float(np.mean([r["newton_step_s"] for r in rows])),
       "start_model_err_rel": float(np.linalg.norm(v0 - vt) / np.linalg.norm(vt)), "steps": rows}
s = json.dumps(out, indent=1)
print(s)
if a.out:
    open(a.out, "w").write(s)
