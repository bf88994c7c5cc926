"""GPU parity at BASELINE scale, collected by default under -m gpu (marked slow: ~2 min).

* config 3 (384x128, 48 sources): the exact block solver — lines of nb = 128, factored by
  the block Gauss-Jordan whose pivot search is restricted to 64-wide diagonal blocks — against
  the reference sparse LU (src/lu.cpp:37-209), at 7 Hz (the highest config-3 frequency);
* config 3 Newton steps, exact and ILU(4), against the reference's own gn_step
  (src/driver.cpp:65-127) stored in tests/golden/c3_gn_step.npz (tests/golden/
  make_golden_c3.py ran the reference, ~10 min of CPU): model <= 1e-6 relative L2 (north
  star), misfits, and the GMRES residual history entry by entry;
* the config-5 geometry (2048x1024, 30-cell PML, K = 16 of the 256 sources, 1024
  receivers): the production source-major K1 kernel bit for bit against the reference
  kkt_apply (src/kkt.cpp:78-96). The full-K apply (FWI_C5=1, tests/test_gpu_c5.py) needs
  ~110 GB of host memory for the checker.
"""
import os

import numpy as np
import pytest

import pyoracle as po
from paper_2204_06489_b200 import _abi
from paper_2204_06489_b200 import api as fw
from paper_2204_06489_b200.problem import c3_problem, c5_problem, random_kkt

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c3_gn_step.npz")


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_c3_exact_block_solve_vs_reference_lu_7hz():
    p = c3_problem(freq_hz=7.0)
    rng = np.random.default_rng(71)
    p.u = rng.standard_normal(p.K * p.n) + 1j * rng.standard_normal(p.K * p.n)
    p.r = rng.standard_normal(p.survey.num_data) + 0j
    dev = fw.GnState(p, exact=True)
    print("device exact factor: residual probe", dev.exact_probe_residual)
    assert dev.exact_probe_residual <= 1e-10
    ref = po.Ref(p, full=False, exact=True)  # reference LU, ~1 min
    b = rng.standard_normal(p.n) + 1j * rng.standard_normal(p.n)
    for adj in (False, True):
        want = ref.solve(b, _abi.FWI_PRECOND_EXACT, adj)
        got = dev.solve(b, fw.PrecondMode.exact, adj)
        print("adjoint" if adj else "forward", "relative deviation", rel(got, want))
        assert rel(got, want) <= 1e-10


@pytest.mark.parametrize("tag,solver", [("exact", "fsgn-gmres-exact"), ("ilu4", "fsgn-gmres-ilu")])
def test_c3_gn_step_vs_reference_golden(tag, solver):
    g = np.load(GOLDEN)
    p = c3_problem(freq_hz=3.0)
    p.d_obs = g["d_obs"]
    eps = float(g["epsilon"])
    assert np.array_equal(p.s, g["s0"])
    cfg = fw.FwiConfig(solver=solver, max_inner=30, inner_tol=1e-12, gmres_restart=30, ilu_level=4)
    r = fw.gn_step(p, p.s, 3.0, eps, cfg)
    hist_ref = g[f"{tag}_history"]
    hist = np.array(r.log.residuals())
    dev_hist = np.abs(hist - hist_ref) / hist_ref
    print(f"{tag}: model {rel(r.s, g[f'{tag}_s']):.2e}, misfit_ini {r.misfit_ini:.6e} vs "
          f"{float(g[f'{tag}_misfit_ini']):.6e}, misfit_fin {r.misfit_fin:.6e} vs "
          f"{float(g[f'{tag}_misfit_fin']):.6e}, history max {dev_hist.max():.2e} over {len(hist)} entries")
    assert len(hist) == len(hist_ref)
    assert rel(r.s, g[f"{tag}_s"]) <= 1e-6
    assert abs(r.misfit_ini - float(g[f"{tag}_misfit_ini"])) <= 1e-9 * float(g[f"{tag}_misfit_ini"])
    assert abs(r.misfit_fin - float(g[f"{tag}_misfit_fin"])) <= 1e-6 * float(g[f"{tag}_misfit_fin"])
    assert dev_hist.max() <= 1e-8


def test_c5_geometry_apply_bitwise_vs_reference():
    p = c5_problem(K=16, with_u=True)
    xh = random_kkt(p, 5)
    os.environ["FWI_KKT_FORCE_TMA"] = "1"
    try:
        dev = fw.GnState(p, exact=False)
        out = fw.kkt_apply(dev, fw.KktVector.from_host(dev, xh)).to_host()
        kname = dev.kkt_kernel()
        dev.close()
    finally:
        del os.environ["FWI_KKT_FORCE_TMA"]
    print("K1 kernel:", kname)
    assert "km" in kname  # the source-major production kernel
    want = po.Ref(p, full=False, exact=False).kkt_apply(xh)
    assert np.array_equal(out, want), rel(out, want)
