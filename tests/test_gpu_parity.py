"""GPU parity: the CUDA path (libfwi_b200.so through the C ABI) against the
reference CPU implementation run on the same seeded inputs.

The checker here is the unmodified reference core (oracle/_ref, built from
/root/reference/proj/src by oracle/Makefile) driven through its own API.
Tolerances are the north star's: complex128 operator applies bit-exact where
the arithmetic order is reproduced (kkt_apply, kkt_rhs, ILU preconditioner),
<= 1e-12 relative L2 otherwise; GMRES residual histories <= 1e-8 relative per
iteration.
"""
import numpy as np
import pytest

import pyoracle as po
from paper_2204_06489_b200 import _abi
from paper_2204_06489_b200 import api as fw
from paper_2204_06489_b200.problem import (c1_problem, c2_problem, no_receiver_instance, random_kkt,
                                           small_problem, standard_instance)

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def pair_direct(p, ilu_level=-1, exact=False):
    """Reference and device states built from identical inputs (u and r given)."""
    ref = po.Ref(p, full=False, exact=exact, ilu_level=ilu_level)
    dev = fw.GnState(p, exact=exact, ilu_level=ilu_level)
    return ref, dev


@pytest.fixture(scope="module")
def c1():
    p = c1_problem()
    p.d_obs = po.ref_simulate(p)
    ref = po.Ref(p, full=True, exact=True, ilu_level=4)
    # identical linearisation point on the device: upload the reference's u and r
    q = c1_problem()
    q.u, q.r = ref.u(), ref.residual()
    dev = fw.GnState(q, exact=True, ilu_level=4)
    return p, ref, dev


PROBLEMS = [
    lambda: small_problem(),
    lambda: small_problem(nx=31, nz=23, n_pml=4, K=4, R=7, duplicate_receiver=True,
                          weight_mode=_abi.FWI_WEIGHT_OFFSET, seed=3),
    lambda: small_problem(nx=17, nz=29, n_pml=2, K=2, R=3, seed=11),  # nz > nx: row lines
]


@pytest.mark.parametrize("mk", PROBLEMS)
def test_stencil_bitwise_equals_reference_csr(mk):
    p = mk()
    ref, dev = pair_direct(p)
    rp, ci, va = ref.csr()
    d, e, s = dev.stencil()
    nx = p.grid.nx
    for i in range(p.n):
        for q in range(rp[i], rp[i + 1]):
            j = ci[q]
            want = va[q]
            got = d[i] if j == i else e[i] if j == i + 1 else s[i] if j == i + nx else \
                e[j] if j == i - 1 else s[j]
            assert got == want, (i, j, got, want)


@pytest.mark.parametrize("mk", PROBLEMS)
def test_kkt_apply_bit_exact_small(mk):
    p = mk()
    ref, dev = pair_direct(p)
    for seed in range(3):
        x = random_kkt(p, 100 + seed)
        want = ref.kkt_apply(x)
        got = fw.kkt_apply(dev, fw.KktVector.from_host(dev, x)).to_host()
        assert np.array_equal(got, want), rel(got, want)


def test_kkt_apply_zero_and_unit_model_vector():
    """tests/test_kkt.cpp:48-69 restated: M 0 = 0; xi = (0, e_m, 0) -> (0, eps e_m, -P e_m)."""
    p = standard_instance()
    p.d_obs = po.ref_simulate(p)
    ref = po.Ref(p, full=True)
    q = standard_instance()
    q.u, q.r = ref.u(), ref.residual()
    dev = fw.GnState(q, exact=False)
    z = np.zeros(p.vec_len)
    assert np.all(fw.kkt_apply(dev, fw.KktVector.from_host(dev, z)).to_host() == 0.0)
    node = p.grid.index(5, 5)
    n, K = p.n, p.K
    x = z.copy()
    x[2 * K * n + node] = 1.0
    out = fw.kkt_apply(dev, fw.KktVector.from_host(dev, x)).to_host()
    assert np.all(out[: 2 * K * n] == 0.0)
    ds = out[2 * K * n: 2 * K * n + n]
    assert ds[node] == p.epsilon and np.count_nonzero(ds) == 1
    lam = out[2 * K * n + n:].view(np.complex128).reshape(K, n)
    u = ref.u().reshape(K, n)
    w2 = ref.omega ** 2
    for k in range(K):
        assert lam[k, node] == -(w2 * u[k, node])
        assert np.count_nonzero(lam[k]) == 1


def test_kkt_apply_c1_bit_exact(c1):
    p, ref, dev = c1
    x = random_kkt(p, 7)
    want = ref.kkt_apply(x)
    got = fw.kkt_apply(dev, fw.KktVector.from_host(dev, x)).to_host()
    assert np.array_equal(got, want), rel(got, want)


def test_kkt_apply_c2_parity():
    """BASELINE config 2 at full size: 1e-12 gate (bit-exact expected)."""
    p = c2_problem()
    ref, dev = pair_direct(p)
    x = random_kkt(p, 11)
    want = ref.kkt_apply(x)
    got = fw.kkt_apply(dev, fw.KktVector.from_host(dev, x)).to_host()
    assert rel(got, want) <= 1e-12
    assert np.array_equal(got, want)


@pytest.mark.parametrize("variant", ["plain", "plain_nodes", "tma", "tma_bands", "tma_balanced", "tile"])
@pytest.mark.parametrize("mk", PROBLEMS + [lambda: c2_problem(K=5, R=17),
                                           lambda: small_problem(nx=45, nz=20, n_pml=3, K=19, R=6,
                                                                 duplicate_receiver=True, seed=9),
                                           lambda: small_problem(nx=70, nz=42, n_pml=5, K=3, R=11,
                                                                 duplicate_receiver=True, seed=7)])
def test_kkt_apply_kernel_variants_bit_exact(mk, variant, monkeypatch):
    """Every K1 kernel (source-major TMA = "tma", the chunked tile-TMA kernel, plain with sources
    over threads or walked per node) reproduces
    the reference; the TMA kernels are forced on these small grids (partial strips and rectangles,
    duplicate receivers; odd widths fall back to the plain kernel)."""
    monkeypatch.setenv("FWI_KKT_KERNEL", variant)
    if variant == "plain_nodes":  # node-per-thread plain kernel (sources walked by each thread)
        monkeypatch.setenv("FWI_KKT_KERNEL", "plain")
        monkeypatch.setenv("FWI_KKT_KS", "0")
    elif variant != "plain":
        monkeypatch.setenv("FWI_KKT_FORCE_TMA", "1")
        monkeypatch.setenv("FWI_KKT_KM_FORCE", "1")  # source-major kernel even for 1-row rectangles
    if variant == "tma_balanced":  # area-balanced strips of two widths (the rectangle table)
        monkeypatch.setenv("FWI_KKT_KERNEL", "tma")
        monkeypatch.setenv("FWI_KKT_KM_BALANCED", "1")
    if variant == "tma_bands":  # several 3-row bands per CTA (the config-5 form)
        monkeypatch.setenv("FWI_KKT_KM_ROWS", "3")
        monkeypatch.setenv("FWI_KKT_KM_G", "2")
    p = mk()
    ref, dev = pair_direct(p)
    x = random_kkt(p, 5)
    want = ref.kkt_apply(x)
    got = fw.kkt_apply(dev, fw.KktVector.from_host(dev, x)).to_host()
    assert np.array_equal(got, want), rel(got, want)


def test_kkt_rhs_exact(c1):
    p, ref, dev = c1
    assert np.array_equal(fw.kkt_rhs(dev).to_host(), ref.kkt_rhs())
    dev.set_drop_reg_term(False)
    ref.set_drop(False)
    try:
        assert np.array_equal(fw.kkt_rhs(dev).to_host(), ref.kkt_rhs())
    finally:
        dev.set_drop_reg_term(True)
        ref.set_drop(True)


def test_operator_symmetric_in_real_inner_product(c1):
    """tests/test_kkt.cpp:81-90: <M xi, eta> = <M eta, xi>."""
    p, ref, dev = c1
    for s in range(3):
        xi = fw.KktVector.from_host(dev, random_kkt(p, 300 + s))
        eta = fw.KktVector.from_host(dev, random_kkt(p, 800 + s))
        lhs = fw.dot(fw.kkt_apply(dev, xi), eta)
        rhs = fw.dot(fw.kkt_apply(dev, eta), xi)
        assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))


def test_vector_ops_match_reference_formulas(c1):
    p, ref, dev = c1
    a, b = random_kkt(p, 1), random_kkt(p, 2)
    va, vb = fw.KktVector.from_host(dev, a), fw.KktVector.from_host(dev, b)
    assert abs(fw.dot(va, vb) - a @ b) <= 1e-12 * np.linalg.norm(a) * np.linalg.norm(b)
    assert abs(fw.norm(va) - np.linalg.norm(a)) <= 1e-13 * np.linalg.norm(a)
    fw.axpy(-0.37, va, vb)
    assert np.array_equal(vb.to_host(), b + (-0.37) * a)
    fw.scal(1.5, va)
    assert np.array_equal(va.to_host(), 1.5 * a)


def test_ilu_precond_bit_exact(c1):
    p, ref, dev = c1
    for s in range(2):
        x = random_kkt(p, 40 + s)
        want = ref.precond_apply(x, _abi.FWI_PRECOND_ILU)
        got = fw.precond_apply(dev, fw.KktVector.from_host(dev, x), fw.PrecondMode.ilu).to_host()
        assert np.array_equal(got, want), rel(got, want)


@pytest.mark.parametrize("level", [0, 1, 3])
@pytest.mark.parametrize("mk", PROBLEMS)
def test_ilu_solves_bit_exact_small(mk, level):
    p = mk()
    ref, dev = pair_direct(p, ilu_level=level)
    rng = np.random.default_rng(level)
    b = rng.standard_normal(p.n) + 1j * rng.standard_normal(p.n)
    for adj in (False, True):
        want = ref.solve(b, _abi.FWI_PRECOND_ILU, adj)
        got = dev.solve(b, fw.PrecondMode.ilu, adj)
        assert np.array_equal(got, want), (adj, rel(got, want))


@pytest.mark.parametrize("mk", PROBLEMS)
def test_exact_block_solve_matches_reference_lu(mk):
    p = mk()
    ref, dev = pair_direct(p, exact=True)
    rng = np.random.default_rng(5)
    b = rng.standard_normal(p.n) + 1j * rng.standard_normal(p.n)
    for adj in (False, True):
        want = ref.solve(b, _abi.FWI_PRECOND_EXACT, adj)
        got = dev.solve(b, fw.PrecondMode.exact, adj)
        assert rel(got, want) <= 1e-11, (adj, rel(got, want))


def test_exact_precond_c1(c1):
    p, ref, dev = c1
    x = random_kkt(p, 9)
    want = ref.precond_apply(x, _abi.FWI_PRECOND_EXACT)
    got = fw.precond_apply(dev, fw.KktVector.from_host(dev, x), fw.PrecondMode.exact).to_host()
    assert rel(got, want) <= 1e-10, rel(got, want)


def test_precond_cost_contract(c1):
    """tests/test_kkt.cpp:153-159: one exact precond_apply = 2K solve pairs."""
    p, ref, dev = c1
    dev.reset_solve_count(fw.PrecondMode.exact)
    fw.precond_apply(dev, fw.KktVector.from_host(dev, random_kkt(p, 1)), fw.PrecondMode.exact)
    assert dev.solve_count(fw.PrecondMode.exact) == 2 * p.K


def test_exact_precond_inverts_operator_without_receivers():
    """tests/test_kkt.cpp:132-140."""
    p = no_receiver_instance()
    dev = fw.GnState(p, exact=True)
    for s in range(3):
        x = random_kkt(p, 71 + s)
        xi = fw.KktVector.from_host(dev, x)
        back = fw.precond_apply(dev, fw.kkt_apply(dev, xi), fw.PrecondMode.exact).to_host()
        assert rel(back, x) < 1e-10


def test_forward_fields_match_reference(c1):
    p, ref, _ = c1
    dev = fw.GnState(p, exact=True)  # u by the device's own exact forward solves
    assert rel(dev.u(), ref.u()) < 1e-10
    assert rel(dev.residual(), ref.residual()) < 1e-8


@pytest.mark.parametrize("mode", [fw.PrecondMode.exact, fw.PrecondMode.ilu])
def test_fsgn_residual_history_c1(c1, mode):
    """Residual histories agree to 1e-8 per iteration (north-star gate)."""
    p, ref, dev = c1
    maxit = 50
    ds_r, log_r = ref.fsgn(int(mode), 30, 0.0, maxit, 0)
    ds_d, log_d = fw.fsgn_gmres_step(dev, fw.FsgnOptions(mode=mode, restart=30, tol=0.0, maxit=maxit,
                                                         ecg_stride=0))
    rr, rd = np.array(log_r.residuals()), np.array(log_d.residuals())
    assert len(rr) == len(rd)
    dev_rel = np.abs(rd - rr) / rr
    print("max history deviation", dev_rel.max(), "per-iter", dev_rel)
    assert dev_rel.max() <= 1e-8


def test_fsgn_converges_c1(c1):
    p, ref, dev = c1
    ds_r, log_r = ref.fsgn(_abi.FWI_PRECOND_EXACT, 30, 1e-3, 60, 0)
    ds_d, log_d = fw.fsgn_gmres_step(dev, fw.FsgnOptions(tol=1e-3, maxit=60, ecg_stride=0))
    assert log_d.converged and log_d.iterations() == log_r.iterations()
    assert rel(ds_d, ds_r) < 1e-6


def test_zero_receivers_converge_in_one_iteration():
    """tests/test_kkt.cpp:179-189."""
    p = no_receiver_instance()
    dev = fw.GnState(p, exact=True)
    ds, log = fw.fsgn_gmres_step(dev, fw.FsgnOptions(tol=1e-10, maxit=30))
    assert log.converged and log.iterations() == 1 and log.final_residual() < 1e-10


@pytest.mark.parametrize("variant", ["tma", "tile", "plain"])
def test_c64_apply_deviation(variant, monkeypatch):
    monkeypatch.setenv("FWI_KKT_KERNEL", variant)
    p = c2_problem()
    ref = po.Ref(p, full=False, exact=False)
    dev = fw.GnState(p, exact=False, c64=True)
    x = random_kkt(p, 11)
    want = ref.kkt_apply(x)
    got = fw.kkt_apply(dev, fw.KktVector.from_host(dev, x.astype(np.float32), _abi.FWI_C64)).to_host()
    err = rel(got.astype(np.float64), want)
    print("complex64 apply relative L2 deviation", err)
    assert err < 1e-5


@pytest.mark.parametrize("env", [{"FWI_KKT_KM_KS": "swap"}, {"FWI_KKT_KM_THR": "swap"},
                                 {"FWI_KKT_KM_WS": "2", "FWI_KKT_KM_STAGES": "3"},
                                 {"FWI_KKT_KM_WS": "2", "FWI_KKT_KM_KS": "2", "FWI_KKT_KM_STAGES": "4"}])
@pytest.mark.parametrize("c64", [False, True])
def test_km1_ring_variants_identical(env, c64, monkeypatch):
    """The one-band source-major K1's ring disciplines (block barrier / per-stage empty barriers)
    and sources per stage (complex64: two by default) give bit-identical applies on config 2."""
    p = c2_problem()
    x = random_kkt(p, 11)
    prec = _abi.FWI_C64 if c64 else _abi.FWI_C128
    xin = x.astype(np.float32) if c64 else x

    def run():
        dev = fw.GnState(p, exact=False, c64=c64)
        try:
            out = fw.kkt_apply(dev, fw.KktVector.from_host(dev, xin, prec)).to_host()
            return out, dev.kkt_kernel(prec)
        finally:
            dev.close()

    base, kbase = run()
    for k, v in env.items():
        swap = {"FWI_KKT_KM_KS": ("1", "2"), "FWI_KKT_KM_THR": ("1024", "1024")}[k] if v == "swap" else None
        monkeypatch.setenv(k, (swap[0] if c64 else swap[1]) if swap else v)
    got, kgot = run()
    assert "kkt_km1_kernel" in kbase and "kkt_km1_kernel" in kgot and kbase != kgot, (kbase, kgot)
    assert np.array_equal(got, base)


# ---- generic GMRES known answers (tests/test_krylov.cpp:63-125, real systems)

def test_gmres_identity_one_iteration():
    b = np.array([1.0, 2.0, 3.0, -1.0])
    x, log = fw.gmres(lambda v: v, lambda v: v, b, 5, 1e-12, 20)
    assert log.converged and log.iterations() == 1 and rel(x, b) < 1e-13


def test_gmres_exact_inverse_preconditioner():
    m = np.array([[2.0, 0.5], [-1.0, 3.0]])
    mi = np.linalg.inv(m)
    x, log = fw.gmres(lambda v: m @ v, lambda v: mi @ v, np.array([1.0, 0.5]), 5, 1e-10, 20)
    assert log.converged and log.iterations() == 1 and log.final_residual() < 1e-10


def test_gmres_4x4_by_iteration_4():
    m = np.array([[2, 1, 0, 1], [0, 3, 1, 0], [1, 0, 4, 1], [0, -1, 0, 5.0]])
    x0 = np.array([1.0, -2.0, 3.0, 2.0])
    x, log = fw.gmres(lambda v: m @ v, lambda v: v, m @ x0, 4, 1e-12, 4)
    assert log.converged and log.iterations() <= 4 and rel(x, x0) < 1e-10


def test_gmres_stagnation_on_nilpotent():
    m = np.array([[0.0, 1.0], [0.0, 0.0]])
    x, log = fw.gmres(lambda v: m @ v, lambda v: v, np.array([1.0, 0.0]), 2, 1e-12, 8)
    assert not log.converged and log.stagnated


def test_gmres_observer_stops():
    m = np.array([[4, 1, 0, 0], [1, 3, 1, 0], [0, 1, 5, 0], [0, 0, 0, 2.0]])
    calls = []
    x, log = fw.gmres(lambda v: m @ v, lambda v: v, np.array([1.0, 2, 3, 1]), 3, 1e-14, 50,
                      observer=lambda it, x: calls.append(it) or len(calls) >= 2)
    assert len(calls) == 2 and log.iterations() == 2 and not log.converged


def test_gmres_zero_rhs():
    x, log = fw.gmres(lambda v: v, lambda v: v, np.zeros(4), 3, 1e-12, 9)
    assert log.converged and log.iterations() == 0 and np.all(x == 0)


def test_invalid_arguments_raise():
    with pytest.raises(fw.InvalidArgument):
        fw.gmres(lambda v: v, lambda v: v, np.ones(2), 0, 1e-12, 9)
    p = small_problem()
    dev = fw.GnState(p, exact=False)
    with pytest.raises(fw.InvalidArgument):
        fw.precond_apply(dev, fw.KktVector(dev), fw.PrecondMode.ilu)
    bad = small_problem()
    bad.epsilon = 0.0
    with pytest.raises(fw.InvalidArgument):
        fw.GnState(bad)


@pytest.mark.parametrize("mk", [lambda: small_problem(), lambda: c2_problem(K=11, R=9)])
def test_kkt_apply_host_pipelined_bit_exact(mk):
    """fwi_dev_kkt_apply_host (chunked H2D/compute/D2H) equals the reference."""
    p = mk()
    ref, dev = pair_direct(p)
    for seed in (3, 4):
        x = random_kkt(p, seed)
        assert np.array_equal(fw.kkt_apply_host(dev, x), ref.kkt_apply(x))


@pytest.mark.parametrize("solver,ilu", [(1, 4), (2, 4)])
def test_gn_step_matches_reference_c1(solver, ilu):
    """gn_step (src/driver.cpp:65-127): the Newton-updated model within 1e-6 relative L2
    (north-star gate) and the misfits of the reference."""
    p = c1_problem()
    p.d_obs = po.ref_simulate(p)
    s_ref, mi_ref, mf_ref, log_ref = po.ref_gn_step(p, solver=solver, max_inner=30, inner_tol=1e-12,
                                                    restart=30, ilu_level=ilu)
    cfg = fw.FwiConfig(solver="fsgn-gmres-exact" if solver == 1 else "fsgn-gmres-ilu", max_inner=30,
                       inner_tol=1e-12, gmres_restart=30, ilu_level=ilu)
    r = fw.gn_step(p, p.s, p.freq_hz, p.epsilon, cfg)
    print("model rel dev", rel(r.s, s_ref), "misfits", r.misfit_ini, mi_ref, r.misfit_fin, mf_ref)
    assert rel(r.s, s_ref) <= 1e-6
    assert abs(r.misfit_ini - mi_ref) <= 1e-9 * mi_ref
    assert abs(r.misfit_fin - mf_ref) <= 1e-6 * mf_ref
    assert r.log.iterations() == log_ref.iterations()


def test_rsgn_cg_matches_reference_and_agrees_with_fsgn(c1):
    """rsgn_cg_step on the device vs the reference (C1: the early CG iterations,
    before CG's rounding sensitivity on this ill-conditioned system takes over),
    and RSGN vs FSGN at tight tolerance on the standard instance
    (tests/test_kkt.cpp:206-215)."""
    p, ref, dev = c1
    ds_r, log_r = ref.rsgn(1e-6, 8)
    ds_d, log_d = fw.rsgn_cg_step(dev, 1e-6, 8)
    rr, rd = np.array(log_r.residuals()), np.array(log_d.residuals())
    assert len(rr) == len(rd) == 9
    assert np.max(np.abs(rd - rr) / rr) <= 1e-8
    assert rel(ds_d, ds_r) <= 1e-6
    q = standard_instance()
    q.d_obs = po.ref_simulate(q)
    r0 = po.Ref(q, full=True)
    q.u, q.r = r0.u(), r0.residual()
    dv = fw.GnState(q, exact=True)
    ds_cg, _ = fw.rsgn_cg_step(dv, 1e-12, 400)
    ds_gm, _ = fw.fsgn_gmres_step(dv, fw.FsgnOptions(tol=1e-12, maxit=400, ecg_stride=0))
    assert rel(ds_gm, ds_cg) < 1e-5


def test_gradient_matches_reference(c1):
    """gradient (src/reduced_space.cpp:141-152): K adjoint exact solves."""
    p, ref, dev = c1
    assert rel(fw.gradient(dev), ref.gradient()) <= 1e-10


def test_hessian_apply_matches_reference(c1):
    """hessian_apply (src/reduced_space.cpp:120-139): 2K exact solves."""
    p, ref, dev = c1
    v = np.random.default_rng(17).standard_normal(p.n)
    assert rel(fw.hessian_apply(dev, v), ref.hessian_apply(v)) <= 1e-10


@pytest.mark.parametrize("level", [0, 4])
def test_ilu_solves_bit_exact_beyond_shared_memory(level):
    """n * 16 B above shared memory (the config-4 regime): the sweep keeps the vector in L2 and
    stages only the level metadata; still bit-identical to the reference IluFactors::solve."""
    p = small_problem(nx=170, nz=120, n_pml=8, K=3, R=6)
    assert p.n * 16 > 220 * 1024
    ref, dev = pair_direct(p, ilu_level=level)
    rng = np.random.default_rng(level + 11)
    b = rng.standard_normal((3, p.n)) + 1j * rng.standard_normal((3, p.n))
    for adj in (False, True):
        for r in range(3):
            want = ref.solve(b[r], _abi.FWI_PRECOND_ILU, adj)
            got = dev.solve(b[r], fw.PrecondMode.ilu, adj)
            assert np.array_equal(got, want), (adj, rel(got, want))


def test_fused_mgs_bitwise_equals_stepwise(c1):
    """The one-launch MGS sweep (grid barrier between steps) reproduces the per-step
    launches bit for bit: same grid-stride passes, same ordered partial sums."""
    import os
    p, ref, dev = c1
    opts = fw.FsgnOptions(restart=30, tol=0.0, maxit=20, ecg_stride=0)
    ds_f, log_f = fw.fsgn_gmres_step(dev, opts)
    os.environ["FWI_GMRES_MGS_STEPS"] = "1"
    try:
        ds_s, log_s = fw.fsgn_gmres_step(dev, opts)
    finally:
        del os.environ["FWI_GMRES_MGS_STEPS"]
    assert log_f.residuals() == log_s.residuals()
    assert np.array_equal(ds_f, ds_s)


@pytest.mark.parametrize("level", [4, 21])
def test_ilu_solves_bit_exact_config3_size(level):
    """ILU(p) sweeps on the 384x128 config-3 grid (vector beyond shared memory: the
    level-ordered ring sweep) are bit-identical to the reference's IluFactors::solve
    (src/ilu.cpp:131-174), forward and adjoint, at the default level and the paper's."""
    from paper_2204_06489_b200.problem import c3_problem
    p = c3_problem(freq_hz=3.0)
    rng = np.random.default_rng(31)
    p.u = rng.standard_normal(p.K * p.n) + 1j * rng.standard_normal(p.K * p.n)
    p.r = rng.standard_normal(p.survey.num_data) + 0j
    ref = po.Ref(p, full=False, exact=False, ilu_level=level)
    dev = fw.GnState(p, exact=False, ilu_level=level)
    b = rng.standard_normal(p.n) + 1j * rng.standard_normal(p.n)
    for adj in (False, True):
        assert np.array_equal(dev.solve(b, fw.PrecondMode.ilu, adj), ref.solve(b, _abi.FWI_PRECOND_ILU, adj)), adj
