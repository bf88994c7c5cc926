"""CPU: the plain-C oracle restatement (oracle/fwi_oracle.c) pinned against the
committed golden vectors (tests/golden/, produced by the unmodified reference
via tests/golden/make_golden.py) and against the reference library itself
(oracle/_ref) on fresh seeded inputs. Bit-exact everywhere: both sides run the
same IEEE operations in the same order."""
import numpy as np
import pytest

import golden_io
import pyoracle as po
from paper_2204_06489_b200 import _abi
from paper_2204_06489_b200.problem import (no_receiver_instance, random_kkt, singular_instance, small_problem,
                                           standard_instance, zero_pivot_instance)


def eq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a, b, equal_nan=True)


@pytest.mark.parametrize("name", golden_io.names())
def test_oracle_reproduces_golden_vectors(name):
    p, z = golden_io.load(name)
    o = po.Orc(p, exact=True, ilu_level=int(z["ilu_level"]))
    rp, ci, va = o.csr()
    assert eq(rp, z["csr_rp"]) and eq(ci, z["csr_ci"]) and eq(va, z["csr_va"])
    assert eq(o.u(), z["u_ref"])
    assert eq(o.residual(), z["r_ref"])
    assert eq(o.kkt_apply(z["x1"]), z["kkt_apply_x1"])
    assert eq(o.kkt_apply(z["x2"]), z["kkt_apply_x2"])
    assert eq(o.kkt_rhs(), z["kkt_rhs"])
    assert eq(o.precond_apply(z["x1"], _abi.FWI_PRECOND_EXACT), z["precond_exact_x1"])
    if "precond_ilu_x1" in z:
        assert eq(o.precond_apply(z["x1"], _abi.FWI_PRECOND_ILU), z["precond_ilu_x1"])
    if "gradient" in z:
        assert eq(o.gradient(), z["gradient"])
    for tag, mode in (("exact", _abi.FWI_PRECOND_EXACT), ("ilu", _abi.FWI_PRECOND_ILU)):
        if f"fsgn_{tag}_ds" not in z:
            continue
        ds, log = o.fsgn(mode, 30, 0.0, 12, 2 if int(z["full"]) else 0)
        assert eq(ds, z[f"fsgn_{tag}_ds"])
        assert eq(np.array(log.residuals()), z[f"fsgn_{tag}_res"])
        assert eq(np.array([e.precond_residual or 0.0 for e in log.entries]), z[f"fsgn_{tag}_prec"])
        assert eq(np.array([np.nan if e.normal_residual is None else e.normal_residual for e in log.entries]),
                  z[f"fsgn_{tag}_normal"])


@pytest.mark.parametrize("name", golden_io.names())
def test_reference_library_reproduces_golden_vectors(name):
    """The shipped oracle/_ref build still matches what made the fixtures."""
    p, z = golden_io.load(name)
    r = po.Ref(p, full=bool(z["full"]), exact=True, ilu_level=int(z["ilu_level"]))
    assert eq(r.kkt_apply(z["x1"]), z["kkt_apply_x1"])
    assert eq(r.precond_apply(z["x1"], _abi.FWI_PRECOND_EXACT), z["precond_exact_x1"])


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_oracle_matches_reference_on_seeded_problems(seed):
    p = small_problem(nx=20 + seed, nz=16 + 2 * seed, n_pml=2 + seed % 2, K=2 + seed, R=3 + seed,
                      seed=seed, duplicate_receiver=seed == 2,
                      weight_mode=_abi.FWI_WEIGHT_OFFSET if seed == 3 else _abi.FWI_WEIGHT_IDENTITY)
    r = po.Ref(p, full=False, exact=True, ilu_level=seed)
    o = po.Orc(p, exact=True, ilu_level=seed)
    for s in range(2):
        x = random_kkt(p, 50 + s)
        assert eq(o.kkt_apply(x), r.kkt_apply(x))
        assert eq(o.precond_apply(x, _abi.FWI_PRECOND_EXACT), r.precond_apply(x, _abi.FWI_PRECOND_EXACT))
        assert eq(o.precond_apply(x, _abi.FWI_PRECOND_ILU), r.precond_apply(x, _abi.FWI_PRECOND_ILU))
    b = np.random.default_rng(seed).standard_normal(p.n) * (1 + 1j)
    for mode in (_abi.FWI_PRECOND_EXACT, _abi.FWI_PRECOND_ILU):
        for adj in (False, True):
            assert eq(o.solve(b, mode, adj), r.solve(b, mode, adj))
    for mode in (_abi.FWI_PRECOND_EXACT, _abi.FWI_PRECOND_ILU):
        ds_r, lr = r.fsgn(mode, 5, 0.0, 9, 0)
        ds_o, lo = o.fsgn(mode, 5, 0.0, 9, 0)
        assert eq(ds_o, ds_r) and lr.residuals() == lo.residuals()
        assert lr.converged == lo.converged and lr.stagnated == lo.stagnated


# ---- the reference's own KKT unit tests (tests/test_kkt.cpp), restated on the oracle


@pytest.fixture(scope="module")
def std_orc():
    p = standard_instance()
    p.d_obs = po.ref_simulate(p)
    return p, po.Orc(p, exact=True, ilu_level=1000)


def test_zero_maps_to_zero_and_unit_model_vector(std_orc):
    """tests/test_kkt.cpp:48-69"""
    p, o = std_orc
    n, K = p.n, p.K
    assert np.all(o.kkt_apply(np.zeros(p.vec_len)) == 0.0)
    node = p.grid.index(5, 5)
    x = np.zeros(p.vec_len)
    x[2 * K * n + node] = 1.0
    out = o.kkt_apply(x)
    assert np.all(out[: 2 * K * n] == 0.0)
    ds = out[2 * K * n: 2 * K * n + n]
    assert ds[node] == p.epsilon and np.count_nonzero(ds) == 1
    lam = out[2 * K * n + n:].view(np.complex128).reshape(K, n)
    u = o.u().reshape(K, n)
    for k in range(K):
        assert lam[k, node] == -(o.omega ** 2 * u[k, node]) and np.count_nonzero(lam[k]) == 1


def test_symmetric_in_real_inner_product(std_orc):
    """tests/test_kkt.cpp:81-90"""
    p, o = std_orc
    for s in range(4):
        xi, eta = random_kkt(p, 300 + s), random_kkt(p, 800 + s)
        lhs, rhs = o.kkt_apply(xi) @ eta, o.kkt_apply(eta) @ xi
        assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))


def test_f_block_is_psd(std_orc):
    """tests/test_kkt.cpp:92-108"""
    p, o = std_orc
    n, K = p.n, p.K
    for s in range(10):
        x = np.zeros(p.vec_len)
        x[: 2 * K * n] = random_kkt(p, 5000 + s)[: 2 * K * n]
        assert o.kkt_apply(x)[: 2 * K * n] @ x[: 2 * K * n] >= 0.0


def test_ilu_full_fill_equals_exact(std_orc):
    """tests/test_kkt.cpp:142-151"""
    p, o = std_orc
    v = random_kkt(p, 55)
    a, b = o.precond_apply(v, _abi.FWI_PRECOND_ILU), o.precond_apply(v, _abi.FWI_PRECOND_EXACT)
    assert np.linalg.norm(a - b) < 1e-10 * np.linalg.norm(b)


def test_exact_precond_costs_2k_solves(std_orc):
    """tests/test_kkt.cpp:153-159"""
    p, o = std_orc
    before = o.solve_count(_abi.FWI_PRECOND_EXACT)
    o.precond_apply(random_kkt(p, 7), _abi.FWI_PRECOND_EXACT)
    assert o.solve_count(_abi.FWI_PRECOND_EXACT) - before == 2 * p.K


def test_no_receivers_exact_precond_inverts_and_converges_in_one():
    """tests/test_kkt.cpp:132-140 and :179-189"""
    p = no_receiver_instance()
    o = po.Orc(p, exact=True)
    x = random_kkt(p, 71)
    back = o.precond_apply(o.kkt_apply(x), _abi.FWI_PRECOND_EXACT)
    assert np.linalg.norm(back - x) < 1e-10 * np.linalg.norm(x)
    ds, log = o.fsgn(_abi.FWI_PRECOND_EXACT, 30, 1e-10, 30, 1)
    assert log.converged and log.iterations() == 1 and log.final_residual() < 1e-10


def test_zero_rhs_returns_zero_in_zero_iterations():
    """tests/test_kkt.cpp:191-204"""
    p = standard_instance()
    p.drop_reg_term = True
    p.d_obs = po.ref_simulate(p, p.s)  # data of the linearisation point itself: r = 0
    o = po.Orc(p, exact=True)
    ds, log = o.fsgn(_abi.FWI_PRECOND_EXACT, 30, 1e-10, 30, 1)
    assert np.linalg.norm(ds) == 0.0 and log.iterations() == 0


def test_zero_pivot_reported_like_reference():
    """ZeroPivotError index (include/fwi/ilu.hpp:11-17; tests/test_ilu.cpp:107-120) agrees with
    the reference on a Helmholtz operator whose pivot cancels exactly, and a shift rescues it."""
    p = zero_pivot_instance()
    o = po.Orc(p, exact=True)
    r = po.Ref(p, full=False, exact=True)
    for level in (0, 2, 5):
        assert o.ilu_factor_status(level, 0.0) == r.ilu_factor_status(level, 0.0) == \
            (_abi.FWI_ERR_ZERO_PIVOT, p.grid.index(1, 1))
    assert o.ilu_factor_status(2, 0.5) == r.ilu_factor_status(2, 0.5) == (0, -1)
    q = small_problem()
    assert po.Orc(q, exact=False).ilu_factor_status(2, 0.0) == \
        po.Ref(q, full=False, exact=False).ilu_factor_status(2, 0.0) == (0, -1)


def test_singular_pivot_reported_like_reference():
    """SingularPivotError index (include/fwi/lu.hpp:11-16; tests/test_lu.cpp:44-47): a zero row."""
    p = singular_instance()
    got = []
    for mk in (lambda: po.Orc(p, exact=True), lambda: po.Ref(p, full=False, exact=True)):
        with pytest.raises(po.CheckerError) as e:
            mk()
        got.append((e.value.code, e.value.index))
    assert got[0] == got[1] == (_abi.FWI_ERR_SINGULAR_PIVOT, p.grid.index(1, 1))
