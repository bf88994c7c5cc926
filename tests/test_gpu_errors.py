"""GPU: the reference's error conventions on the device path, against the reference.

ZeroPivotError{index} (include/fwi/ilu.hpp:11-17; pinned by tests/test_ilu.cpp:107-120)
and SingularPivotError{index} (include/fwi/lu.hpp:11-16; tests/test_lu.cpp:44-47) are
triggered on real Helmholtz operators crafted so that a stencil diagonal cancels
exactly (problem.zero_pivot_instance / singular_instance), and the index the device
reports is compared with the one the reference (oracle/_ref) reports.
"""
import numpy as np
import pytest

import pyoracle as po
from paper_2204_06489_b200 import _abi
from paper_2204_06489_b200 import api as fw
from paper_2204_06489_b200.problem import singular_instance, small_problem, zero_pivot_instance

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("level", [0, 2, 5])
def test_device_ilu_zero_pivot_index_matches_reference(level):
    p = zero_pivot_instance()
    code, ref_index = po.Ref(p, full=False, exact=True).ilu_factor_status(level, 0.0)
    assert code == _abi.FWI_ERR_ZERO_PIVOT
    with pytest.raises(fw.ZeroPivotError) as e:
        fw.GnState(p, exact=True, ilu_level=level)
    assert e.value.index == ref_index == p.grid.index(1, 1)
    # the same through an existing context (IluFactors::factor on demand)
    dev = fw.GnState(p, exact=True)
    with pytest.raises(fw.ZeroPivotError) as e:
        fw._check(fw.lib().fwi_dev_factor_ilu(dev.h, level, 0.0))
    assert e.value.index == ref_index


def test_device_ilu_shift_rescues_the_zero_pivot_like_reference():
    p = zero_pivot_instance()
    ref = po.Ref(p, full=False, exact=True, ilu_level=2, ilu_shift=0.5)
    dev = fw.GnState(p, exact=True, ilu_level=2, ilu_diag_shift=0.5)
    rng = np.random.default_rng(4)
    b = rng.standard_normal(p.n) + 1j * rng.standard_normal(p.n)
    for adj in (False, True):
        assert np.array_equal(dev.solve(b, fw.PrecondMode.ilu, adj), ref.solve(b, _abi.FWI_PRECOND_ILU, adj))


def test_device_exact_factor_passes_a_zero_diagonal_like_reference():
    """The exact factorisation pivots past the cancelled diagonal (the operator is nonsingular)."""
    p = zero_pivot_instance()
    ref = po.Ref(p, full=False, exact=True)
    dev = fw.GnState(p, exact=True)
    rng = np.random.default_rng(5)
    b = rng.standard_normal(p.n) + 1j * rng.standard_normal(p.n)
    for adj in (False, True):
        want = ref.solve(b, _abi.FWI_PRECOND_EXACT, adj)
        got = dev.solve(b, fw.PrecondMode.exact, adj)
        assert np.linalg.norm(got - want) <= 1e-10 * np.linalg.norm(want)


def test_device_singular_pivot_index_matches_reference():
    p = singular_instance()
    with pytest.raises(po.CheckerError) as e:
        po.Ref(p, full=False, exact=True)
    assert e.value.code == _abi.FWI_ERR_SINGULAR_PIVOT
    with pytest.raises(fw.SingularPivotError) as d:
        fw.GnState(p, exact=True)
    assert d.value.index == e.value.index == p.grid.index(1, 1)


def test_residual_probe_accepts_regular_factorisations():
    """The post-factorisation residual probe (exact.cu exact_factor) passes on a regular
    instance and leaves the solve count untouched."""
    p = small_problem()
    dev = fw.GnState(p, exact=True)
    assert dev.solve_count(fw.PrecondMode.exact) == 0
