"""Load a golden fixture (tests/golden/*.npz) back into a Problem."""
import os

import numpy as np

from paper_2204_06489_b200.problem import Grid, Problem, Survey

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    # operator-level fixtures of make_golden.py (c3_gn_step.npz, make_golden_c3.py, is a
    # Newton-step fixture read by tests/test_gpu_scale_parity.py)
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and f != "c3_gn_step.npz")


def load(name):
    z = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    g = Grid(int(z["nx"]), int(z["nz"]), float(z["h"]), int(z["n_pml"]), float(z["sigma_max"]), float(z["power"]))
    sv = Survey(src_ix=z["src_ix"], src_iz=z["src_iz"], recv_offset=z["recv_offset"], recv_ix=z["recv_ix"],
                recv_iz=z["recv_iz"], weight_mode=int(z["weight_mode"]))
    p = Problem(grid=g, survey=sv, freq_hz=float(z["freq_hz"]), epsilon=float(z["epsilon"]), s=z["s"],
                drop_reg_term=bool(z["drop"]), u=z["u"] if z["u"].size else None,
                r=z["r"] if z["r"].size else None, d_obs=z["d_obs"] if z["d_obs"].size else None, name=name)
    return p, z
