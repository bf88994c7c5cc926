"""GPU: the remaining pins of the reference's own test suite on the device path —
F-block positivity (tests/test_kkt.cpp:92-108), ILU(level 1000) = exact preconditioner
(:142-151), the E_cg column starting at 1 (:161-177), and bitwise-identical repeated fwi_run
(tests/test_driver.cpp:123-148: deterministic reductions, no atomics in any sum)."""
from dataclasses import replace

import numpy as np
import pytest

import pyoracle as po
from paper_2204_06489_b200 import api as fw
from paper_2204_06489_b200.problem import c1_problem, random_kkt, small_problem

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.mark.parametrize("mk", [lambda: small_problem(), lambda: small_problem(nx=40, nz=30, n_pml=4, K=4, R=9,
                                                                              duplicate_receiver=True)])
def test_f_block_positive_semidefinite(mk):
    """With lambda = 0 and ds = 0 the du block of the apply is F du = Q^H W^T W Q du: Re<du, F du> >= 0,
    and the output equals the reference's bit for bit."""
    p = mk()
    dev = fw.GnState(p, exact=False)
    ref = po.Ref(p, full=False, exact=False)
    K, n = p.K, p.n
    for seed in range(5):
        x = random_kkt(p, 40 + seed)
        x[2 * K * n:] = 0.0  # ds and lambda blocks
        y = fw.kkt_apply(dev, fw.KktVector.from_host(dev, x)).to_host()
        assert np.array_equal(y, ref.kkt_apply(x))
        du = x[:2 * K * n].view(np.complex128)
        fdu = y[:2 * K * n].view(np.complex128)
        assert float(np.real(np.vdot(du, fdu))) >= 0.0
        assert np.count_nonzero(fdu) <= 2 * p.survey.num_data  # F touches receiver nodes only


def test_ilu_level_1000_preconditioner_equals_exact():
    """ILU with unlimited fill is the exact LU: precond_apply(ilu) = precond_apply(exact) to 1e-10."""
    p = small_problem()
    dev = fw.GnState(p, exact=True, ilu_level=1000)
    for seed in range(3):
        x = fw.KktVector.from_host(dev, random_kkt(p, 60 + seed))
        a = fw.precond_apply(dev, x, fw.PrecondMode.ilu).to_host()
        b = fw.precond_apply(dev, x, fw.PrecondMode.exact).to_host()
        assert rel(a, b) < 1e-10


def test_ecg_column_populated_and_starts_at_one():
    """fsgn_gmres_step with ecg_stride 1: every entry carries E_cg = ||H ds - g|| / ||g||, 1 at ds = 0."""
    p = c1_problem()
    p.d_obs = po.ref_simulate(p)
    dev = fw.GnState(p, exact=True)
    ds, log = fw.fsgn_gmres_step(dev, fw.FsgnOptions(tol=1e-3, maxit=30, ecg_stride=1))
    e = [x.normal_residual for x in log.entries]
    assert all(v is not None for v in e)
    assert e[0] == 1.0
    assert e[-1] < 0.1 and log.converged


@pytest.mark.parametrize("solver,ilu", [("fsgn-gmres-ilu", 2), ("fsgn-gmres-exact", 4)])
def test_repeated_fwi_run_bitwise_identical(solver, ilu):
    """Two fwi_run sweeps over two frequencies give identical models, misfits and residual
    histories bit for bit (the reference's determinism pin, ILU(2) there)."""
    p = c1_problem()
    observed = {f: fw.simulate(replace(p, freq_hz=f)) for f in (4.0, 5.0)}
    eps = {4.0: 1e10, 5.0: 1e10}
    cfg = fw.FwiConfig(solver=solver, max_inner=30, inner_tol=1e-3, gmres_restart=30, ilu_level=ilu)
    q = replace(p, drop_reg_term=True)
    runs = [fw.fwi_run(q, observed, p.s, eps, cfg) for _ in range(2)]
    for a, b in zip(*runs):
        assert np.array_equal(a.s, b.s)
        assert a.misfit_ini == b.misfit_ini and a.misfit_fin == b.misfit_fin
        assert a.log.residuals() == b.log.residuals()
        assert [e.precond_residual for e in a.log.entries] == [e.precond_residual for e in b.log.entries]
