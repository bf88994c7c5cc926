"""Golden Newton steps on BASELINE config 3 (384x128, 48 sources, 3 Hz) from the UNMODIFIED
reference (oracle/_ref, the reference's own gn_step, src/driver.cpp:65-127), so the GPU test
run can check the device at config-3 scale in seconds (the reference takes ~10 min here):

    python tests/golden/make_golden_c3.py

Stored: the reference's observed data (its forward solve on the true model), the updated
model, both misfits and the GMRES residual history, for the exact (fsgn-gmres-exact) and the
ILU(4) (fsgn-gmres-ilu) solvers, with max_inner 30, inner_tol 1e-12, restart 30 (FwiConfig
defaults) and eps = 2.8e10 = 1e-2 ||J^H J|| with drop_reg_term.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import pyoracle as po  # noqa: E402
from paper_2204_06489_b200.problem import c3_problem  # noqa: E402

EPS = 2.8e10


def main():
    p = c3_problem(freq_hz=3.0)
    p.epsilon = EPS
    t0 = time.time()
    p.d_obs = po.ref_simulate(p)
    print(f"reference d_obs: {time.time() - t0:.0f} s", flush=True)
    out = {"d_obs": p.d_obs, "epsilon": EPS, "s0": p.s}
    for tag, solver, ilu in (("exact", 1, 4), ("ilu4", 2, 4)):
        t0 = time.time()
        s, mi, mf, log = po.ref_gn_step(p, solver=solver, max_inner=30, inner_tol=1e-12, restart=30, ilu_level=ilu)
        print(f"reference gn_step {tag}: {time.time() - t0:.0f} s, {log.iterations()} iterations, "
              f"misfit {mi:.6e} -> {mf:.6e}", flush=True)
        out[f"{tag}_s"] = s
        out[f"{tag}_misfit_ini"] = mi
        out[f"{tag}_misfit_fin"] = mf
        out[f"{tag}_history"] = np.array(log.residuals())
        out[f"{tag}_converged"] = int(log.converged)
    np.savez_compressed(os.path.join(HERE, "c3_gn_step.npz"), **out)


if __name__ == "__main__":
    main()
