"""The north-star residual-history gate, exactly as stated: on config 1, GMRES with
tol = 0, maxit = 50, restart = 30 (the restart at j = 30 is crossed), every one of
the 51 ConvergenceLog entries of the device run within 1e-8 relative of the
reference's (oracle/_ref), with no floor — for the exact, ILU(4) and ILU(21)
(the paper's level) preconditioners.

Reference: gmres, include/fwi/krylov.hpp:179-253; fsgn_gmres_step, src/kkt.cpp:137-171.

The same test records the reference's own rounding-noise yardstick: its history
when b is perturbed by 1e-15 relative (the residual r, from which kkt_rhs builds
b, scaled elementwise by 1 + 1e-15 N(0,1)). Measured on the B200
(profiles/r02_history_gate.json): exact 1.6e-9 (reference drift 1.1e-9),
ILU(4) 7.0e-14 (2.0e-14), ILU(21) 1.2e-11 (8.3e-12).
"""
import numpy as np
import pytest

import pyoracle as po
from paper_2204_06489_b200 import api as fw
from paper_2204_06489_b200.problem import c1_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lin_point():
    p = c1_problem()
    p.d_obs = po.ref_simulate(p)
    base = po.Ref(p, full=True, exact=True, ilu_level=4)
    return base.u(), base.residual()


@pytest.mark.parametrize("name,mode,level", [("exact", fw.PrecondMode.exact, 4),
                                             ("ilu4", fw.PrecondMode.ilu, 4),
                                             ("ilu21", fw.PrecondMode.ilu, 21)])
def test_history_gate_50_iterations_no_floor(lin_point, name, mode, level):
    u, r = lin_point
    q = c1_problem()
    q.u, q.r = u, r
    ref = po.Ref(q, full=False, exact=True, ilu_level=level)
    qp = c1_problem()
    qp.u, qp.r = u, r * (1.0 + 1e-15 * np.random.default_rng(77).standard_normal(r.shape))
    refp = po.Ref(qp, full=False, exact=True, ilu_level=level)
    dev = fw.GnState(q, exact=True, ilu_level=level)
    _, lr = ref.fsgn(int(mode), 30, 0.0, 50, 0)
    _, lp = refp.fsgn(int(mode), 30, 0.0, 50, 0)
    _, ld = fw.fsgn_gmres_step(dev, fw.FsgnOptions(mode=mode, restart=30, tol=0.0, maxit=50, ecg_stride=0))
    hr, hp, hd = (np.array(x.residuals()) for x in (lr, lp, ld))
    assert len(hr) == len(hd) == 51
    dev_rel = np.abs(hd - hr) / hr
    drift = np.abs(hp - hr) / hr
    print(f"{name}: max deviation {dev_rel.max():.2e} at iteration {dev_rel.argmax()}; "
          f"reference drift under a 1e-15 perturbation of b: {drift.max():.2e}")
    assert dev_rel.max() <= 1e-8
    assert ld.converged == lr.converged and ld.stagnated == lr.stagnated
