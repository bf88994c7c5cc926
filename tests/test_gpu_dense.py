"""The long-line exact solver (dense.cu: whole-GPU block Gauss-Jordan + GEMM sweeps, used
for nb > 512, i.e. BASELINE config 5) forced onto small grids with FWI_EXACT_DENSE=1 and
checked against the reference LU (oracle/_ref) on the same seeded inputs."""
import os

import numpy as np
import pytest

import pyoracle as po
from paper_2204_06489_b200 import _abi
from paper_2204_06489_b200 import api as fw
from paper_2204_06489_b200.problem import c1_problem, random_kkt, small_problem, standard_instance

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def dense_state(p, twisted=None, **kw):
    """Dense (GEMM-sweep) exact solver; twisted "0"/"1" forces the one-chain or the
    two-chain (twisted, the default for dense lines) factorisation."""
    os.environ["FWI_EXACT_DENSE"] = "1"
    if twisted is not None:
        os.environ["FWI_EXACT_TWISTED"] = twisted
    try:
        return fw.GnState(p, exact=True, **kw)
    finally:
        del os.environ["FWI_EXACT_DENSE"]
        os.environ.pop("FWI_EXACT_TWISTED", None)


@pytest.mark.parametrize("twisted", ["0", "1"])
@pytest.mark.parametrize("mk", [small_problem, standard_instance,
                                lambda: small_problem(nx=70, nz=90, n_pml=5, K=2, R=4)])
def test_dense_block_solve_matches_reference_lu(mk, twisted):
    p = mk()
    ref = po.Ref(p, full=False, exact=True)
    dev = dense_state(p, twisted)
    rng = np.random.default_rng(5)
    b = rng.standard_normal((3, p.n)) + 1j * rng.standard_normal((3, p.n))
    for adj in (False, True):
        for r in range(3):
            want = ref.solve(b[r], _abi.FWI_PRECOND_EXACT, adj)
            got = dev.solve(b[r], fw.PrecondMode.exact, adj)
            assert rel(got, want) <= 1e-10, (adj, rel(got, want))


def test_dense_solve_residual_c1():
    """||A x - b|| / ||b|| of the dense solve, with A the reference's assembled CSR."""
    import scipy.sparse as sp
    p = c1_problem()
    p.d_obs = po.ref_simulate(p)
    ref = po.Ref(p, full=True, exact=False)
    rp, ci, va = ref.csr()
    A = sp.csr_matrix((va, ci, rp), shape=(p.n, p.n))
    q = c1_problem()
    q.d_obs, q.u, q.r = p.d_obs, ref.u(), ref.residual()
    dev = dense_state(q)
    rng = np.random.default_rng(3)
    b = rng.standard_normal(p.n) + 1j * rng.standard_normal(p.n)
    x = dev.solve(b, fw.PrecondMode.exact, False)
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) < 1e-11
    xa = dev.solve(b, fw.PrecondMode.exact, True)
    assert np.linalg.norm(A.conj().T @ xa - b) / np.linalg.norm(b) < 1e-11


def test_dense_precond_and_gmres_history_c1():
    p = c1_problem()
    p.d_obs = po.ref_simulate(p)
    ref = po.Ref(p, full=True, exact=True)
    q = c1_problem()
    q.d_obs, q.u, q.r = p.d_obs, ref.u(), ref.residual()
    dev = dense_state(q)
    x = random_kkt(p, 9)
    want = ref.precond_apply(x, _abi.FWI_PRECOND_EXACT)
    got = fw.precond_apply(dev, fw.KktVector.from_host(dev, x), fw.PrecondMode.exact).to_host()
    assert rel(got, want) <= 1e-10
    _, log_r = ref.fsgn(_abi.FWI_PRECOND_EXACT, 30, 0.0, 50, 0)
    _, log_d = fw.fsgn_gmres_step(dev, fw.FsgnOptions(restart=30, tol=0.0, maxit=50, ecg_stride=0))
    rr, rd = np.array(log_r.residuals()), np.array(log_d.residuals())
    assert len(rr) == len(rd)
    assert (np.abs(rd - rr) / rr).max() <= 1e-8  # every entry, no floor


def test_host_basis_gmres_history_matches_reference_c1():
    """GMRES with the Krylov basis in pinned host memory (the config-5 storage plan,
    forced with FWI_GMRES_HOST_BASIS=1) keeps the reference's residual history."""
    p = c1_problem()
    p.d_obs = po.ref_simulate(p)
    ref = po.Ref(p, full=True, exact=True)
    q = c1_problem()
    q.d_obs, q.u, q.r = p.d_obs, ref.u(), ref.residual()
    dev = fw.GnState(q, exact=True)
    _, log_r = ref.fsgn(_abi.FWI_PRECOND_EXACT, 4, 0.0, 20, 0)
    os.environ["FWI_GMRES_HOST_BASIS"] = "1"
    try:
        ds_d, log_d = fw.fsgn_gmres_step(dev, fw.FsgnOptions(restart=4, tol=0.0, maxit=20, ecg_stride=0))
    finally:
        del os.environ["FWI_GMRES_HOST_BASIS"]
    rr, rd = np.array(log_r.residuals()), np.array(log_d.residuals())
    assert len(rr) == len(rd)
    assert (np.abs(rd - rr) / rr).max() <= 1e-8  # every entry, no floor
    assert log_d.stagnated == log_r.stagnated


def test_block_gauss_jordan_factor_with_cluster_sweep():
    """nb in (112, 512]: block Gauss-Jordan factor (dense.cu) + warp-specialised sweep."""
    p = small_problem(nx=150, nz=130, n_pml=8, K=3, R=6)
    ref = po.Ref(p, full=False, exact=True)
    dev = fw.GnState(p, exact=True)
    rng = np.random.default_rng(8)
    b = rng.standard_normal(p.n) + 1j * rng.standard_normal(p.n)
    for adj in (False, True):
        want = ref.solve(b, _abi.FWI_PRECOND_EXACT, adj)
        got = dev.solve(b, fw.PrecondMode.exact, adj)
        assert rel(got, want) <= 1e-10, (adj, rel(got, want))


@pytest.mark.parametrize("lines", ["short", "long"])
@pytest.mark.parametrize("mk", [lambda: small_problem(nx=40, nz=26, n_pml=4, K=3, R=5),
                                lambda: small_problem(nx=22, nz=37, n_pml=3, K=2, R=4, seed=5)])
def test_exact_solve_both_line_orientations(mk, lines):
    """The exact solver may cut the grid into short or long lines (chosen by its step
    model); both orientations match the reference LU."""
    p = mk()
    ref = po.Ref(p, full=False, exact=True)
    os.environ["FWI_EXACT_LINES"] = lines
    try:
        dev = fw.GnState(p, exact=True)
    finally:
        del os.environ["FWI_EXACT_LINES"]
    rng = np.random.default_rng(21)
    b = rng.standard_normal(p.n) + 1j * rng.standard_normal(p.n)
    for adj in (False, True):
        want = ref.solve(b, _abi.FWI_PRECOND_EXACT, adj)
        got = dev.solve(b, fw.PrecondMode.exact, adj)
        assert rel(got, want) <= 1e-10, (lines, adj, rel(got, want))


@pytest.mark.parametrize("restart", [1, 2])
def test_host_basis_small_restart_matches_reference(restart):
    """Host-resident basis at the restart lengths config 5 uses (1-4), incl. stagnation."""
    p = c1_problem()
    p.d_obs = po.ref_simulate(p)
    ref = po.Ref(p, full=True, exact=True)
    q = c1_problem()
    q.d_obs, q.u, q.r = p.d_obs, ref.u(), ref.residual()
    dev = fw.GnState(q, exact=True)
    _, log_r = ref.fsgn(_abi.FWI_PRECOND_EXACT, restart, 0.0, 12, 0)
    os.environ["FWI_GMRES_HOST_BASIS"] = "1"
    try:
        _, log_d = fw.fsgn_gmres_step(dev, fw.FsgnOptions(restart=restart, tol=0.0, maxit=12, ecg_stride=0))
    finally:
        del os.environ["FWI_GMRES_HOST_BASIS"]
    rr, rd = np.array(log_r.residuals()), np.array(log_d.residuals())
    assert len(rr) == len(rd) and log_d.stagnated == log_r.stagnated
    assert (np.abs(rd - rr) / rr).max() <= 1e-8  # every entry, no floor


@pytest.mark.parametrize("mk", [lambda: small_problem(nx=40, nz=26, n_pml=4, K=3, R=5),
                                lambda: small_problem(nx=22, nz=37, n_pml=3, K=2, R=4, seed=5),
                                lambda: small_problem(nx=31, nz=23, n_pml=4, K=9, R=7, seed=3)])
def test_twisted_factorisation_matches_reference(mk):
    """Factorisation from both ends meeting at the middle line; the solve runs the two
    half-sweeps concurrently. Forced with FWI_EXACT_TWISTED=1."""
    p = mk()
    ref = po.Ref(p, full=False, exact=True)
    os.environ["FWI_EXACT_TWISTED"] = "1"
    try:
        dev = fw.GnState(p, exact=True)
    finally:
        del os.environ["FWI_EXACT_TWISTED"]
    rng = np.random.default_rng(31)
    b = rng.standard_normal((2, p.n)) + 1j * rng.standard_normal((2, p.n))
    for adj in (False, True):
        for r in range(2):
            want = ref.solve(b[r], _abi.FWI_PRECOND_EXACT, adj)
            got = dev.solve(b[r], fw.PrecondMode.exact, adj)
            assert rel(got, want) <= 1e-10, (adj, rel(got, want))
    x = random_kkt(p, 4)
    want = ref.precond_apply(x, _abi.FWI_PRECOND_EXACT)
    got = fw.precond_apply(dev, fw.KktVector.from_host(dev, x), fw.PrecondMode.exact).to_host()
    assert rel(got, want) <= 1e-10


@pytest.mark.parametrize("mode,restart,maxit", [("exact", 1, 12), ("exact", 2, 12), ("exact", 4, 20),
                                                ("ilu", 3, 30)])
def test_host_basis_returns_the_device_mode_solution(mode, restart, maxit):
    """The host-resident basis keeps the best iterate recoverable (x + V y recomputed from
    the basis) instead of copying it out per improvement: the returned update equals the
    device-resident solver's bit for bit, including stagnation returns."""
    p = c1_problem()
    p.d_obs = po.ref_simulate(p)
    ref = po.Ref(p, full=True, exact=True, ilu_level=4) if mode == "ilu" else po.Ref(p, full=True, exact=True)
    q = c1_problem()
    q.d_obs, q.u, q.r = p.d_obs, ref.u(), ref.residual()
    dev = fw.GnState(q, exact=True, ilu_level=4 if mode == "ilu" else -1)
    pm = _abi.FWI_PRECOND_ILU if mode == "ilu" else _abi.FWI_PRECOND_EXACT
    ds_r, log_r = ref.fsgn(pm, restart, 0.0, maxit, 0)
    opts = fw.FsgnOptions(mode=fw.PrecondMode.ilu if mode == "ilu" else fw.PrecondMode.exact, restart=restart,
                          tol=0.0, maxit=maxit, ecg_stride=0)
    ds_dev, log_dev = fw.fsgn_gmres_step(dev, opts)
    os.environ["FWI_GMRES_HOST_BASIS"] = "1"
    try:
        ds_h, log_h = fw.fsgn_gmres_step(dev, opts)
    finally:
        del os.environ["FWI_GMRES_HOST_BASIS"]
    assert np.array_equal(np.asarray(ds_h), np.asarray(ds_dev))
    assert log_h.residuals() == log_dev.residuals() and log_h.stagnated == log_dev.stagnated
    assert log_h.stagnated == log_r.stagnated
    assert np.linalg.norm(np.asarray(ds_h) - np.asarray(ds_r)) <= 1e-6 * np.linalg.norm(np.asarray(ds_r))


@pytest.mark.parametrize("mk", [lambda: small_problem(nx=40, nz=26, n_pml=4, K=3, R=5),
                                lambda: small_problem(nx=22, nz=37, n_pml=3, K=2, R=4, seed=5),
                                lambda: small_problem(nx=31, nz=23, n_pml=4, K=9, R=7, seed=3),
                                lambda: small_problem(nx=150, nz=130, n_pml=8, K=3, R=6)])
@pytest.mark.parametrize("l0", ["tri", "gemm"])
def test_cyclic_reduction_matches_reference(mk, l0, monkeypatch):
    """Block cyclic reduction (csrc/bcr.cu; forced with FWI_EXACT_BCR=1: odd and even line
    counts, both orientations, nb > 112) against the reference LU (src/lu.cpp:168-209); level 0
    by the tridiagonal LU sweeps (default) and by the dense M_b products (FWI_BCR_L0=gemm)."""
    monkeypatch.setenv("FWI_EXACT_BCR", "1")
    if l0 == "gemm":
        monkeypatch.setenv("FWI_BCR_L0", "gemm")
    p = mk()
    ref = po.Ref(p, full=False, exact=True)
    dev = fw.GnState(p, exact=True)
    assert dev.exact_probe_residual <= 1e-11
    rng = np.random.default_rng(17)
    b = rng.standard_normal(p.n) + 1j * rng.standard_normal(p.n)
    for adj in (False, True):
        want = ref.solve(b, _abi.FWI_PRECOND_EXACT, adj)
        got = dev.solve(b, fw.PrecondMode.exact, adj)
        assert rel(got, want) <= 1e-10, (adj, rel(got, want))


def test_cyclic_reduction_gmres_history_c1(monkeypatch):
    """The history gate (50 iterations, restart crossed, every entry) with the exact
    preconditioner's block solves by cyclic reduction."""
    monkeypatch.setenv("FWI_EXACT_BCR", "1")
    p = c1_problem()
    p.d_obs = po.ref_simulate(p)
    ref = po.Ref(p, full=True, exact=True)
    q = c1_problem()
    q.d_obs, q.u, q.r = p.d_obs, ref.u(), ref.residual()
    dev = fw.GnState(q, exact=True)
    _, log_r = ref.fsgn(_abi.FWI_PRECOND_EXACT, 30, 0.0, 50, 0)
    _, log_d = fw.fsgn_gmres_step(dev, fw.FsgnOptions(restart=30, tol=0.0, maxit=50, ecg_stride=0))
    rr, rd = np.array(log_r.residuals()), np.array(log_d.residuals())
    assert len(rr) == len(rd) == 51
    print("cyclic reduction history deviation", (np.abs(rd - rr) / rr).max())
    assert (np.abs(rd - rr) / rr).max() <= 1e-8
