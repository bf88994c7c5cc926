"""The pipelined GMRES loop (device Givens step, iteration j + 1 enqueued before iteration j's
residual reaches the host, the residual branch on a second stream; csrc/gmres.cu) against the
synchronous loop (host Givens, two host
round trips per iteration, FWI_GMRES_SYNC=1): bit-identical residual histories, preconditioned
residuals, flags and solutions — the Givens/y-solve arithmetic of include/fwi/krylov.hpp:190-230
restated on the device with explicit rounding, and speculative iterations after convergence
dropped without touching the result.
"""
import numpy as np
import pytest

from paper_2204_06489_b200 import api as fw
from paper_2204_06489_b200.problem import c1_problem, small_problem

pytestmark = pytest.mark.gpu


def run(state, opts, sync, monkeypatch, onestream=False):
    if sync:
        monkeypatch.setenv("FWI_GMRES_SYNC", "1")
    else:
        monkeypatch.delenv("FWI_GMRES_SYNC", raising=False)
    if onestream:
        monkeypatch.setenv("FWI_GMRES_ONESTREAM", "1")
    else:
        monkeypatch.delenv("FWI_GMRES_ONESTREAM", raising=False)
    return fw.fsgn_gmres_step(state, opts)


def same(a, b):
    (ds_a, log_a), (ds_b, log_b) = a, b
    assert np.array_equal(ds_a, ds_b)
    assert log_a.converged == log_b.converged and log_a.stagnated == log_b.stagnated
    assert [e.iteration for e in log_a.entries] == [e.iteration for e in log_b.entries]
    assert np.array_equal(np.array(log_a.residuals()), np.array(log_b.residuals()))
    pa = [e.precond_residual for e in log_a.entries]
    pb = [e.precond_residual for e in log_b.entries]
    assert pa == pb


@pytest.fixture(scope="module")
def c1_state():
    p = c1_problem()
    p.d_obs = fw.simulate(p)
    return fw.GnState(p, exact=True, ilu_level=4)


@pytest.mark.parametrize("mode", ["exact", "ilu"])
@pytest.mark.parametrize("tol,maxit,restart", [(1e-3, 60, 30), (0.0, 50, 30), (1e-6, 40, 7), (0.0, 9, 4)])
def test_pipelined_gmres_bit_identical_to_sync(c1_state, mode, tol, maxit, restart, monkeypatch):
    opts = fw.FsgnOptions(mode=getattr(fw.PrecondMode, mode), tol=tol, maxit=maxit, restart=restart,
                          ecg_stride=0)
    a = run(c1_state, opts, False, monkeypatch)
    b = run(c1_state, opts, True, monkeypatch)
    same(a, b)
    assert len(a[1].entries) > 1
    same(run(c1_state, opts, False, monkeypatch, onestream=True), b)  # residual branch on the main stream


def test_pipelined_gmres_converges_early_small(monkeypatch):
    """A problem GMRES solves in a few iterations (speculative iterations after convergence,
    happy-breakdown style short cycles)."""
    p = small_problem(nx=16, nz=12, n_pml=2, K=2, R=3, seed=5)
    st = fw.GnState(p, exact=True, ilu_level=1000)  # ILU(1000) = exact factors
    for mode in (fw.PrecondMode.exact, fw.PrecondMode.ilu):
        opts = fw.FsgnOptions(mode=mode, tol=1e-12, maxit=30, restart=30, ecg_stride=0)
        a = run(st, opts, False, monkeypatch)
        b = run(st, opts, True, monkeypatch)
        same(a, b)
