"""Generate the golden vectors in tests/golden/*.npz from the UNMODIFIED reference.

The reference core is compiled from /root/reference/proj/src by oracle/Makefile
into oracle/_ref/libfwiref.so and driven through its own public API
(oracle/ref_harness.cpp). Inputs come from the seeded generators in
paper_2204_06489_b200/problem.py, so the fixtures are small and reproducible:

    python tests/golden/make_golden.py

Each .npz stores the inputs it was made from (problem arrays and the KKT
vectors fed to the operators) and the reference outputs.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle as po  # noqa: E402
from paper_2204_06489_b200 import _abi  # noqa: E402
from paper_2204_06489_b200.problem import (no_receiver_instance, random_kkt, small_problem,  # noqa: E402
                                           standard_instance)


def problem_arrays(p):
    sv = p.survey
    return dict(nx=p.grid.nx, nz=p.grid.nz, h=p.grid.h, n_pml=p.grid.n_pml, sigma_max=p.grid.sigma_max,
                power=p.grid.power, freq_hz=p.freq_hz, epsilon=p.epsilon, drop=int(p.drop_reg_term),
                s=p.s, src_ix=sv.src_ix, src_iz=sv.src_iz, recv_offset=sv.recv_offset, recv_ix=sv.recv_ix,
                recv_iz=sv.recv_iz, weight_mode=sv.weight_mode,
                u=p.u if p.u is not None else np.zeros(0, np.complex128),
                r=p.r if p.r is not None else np.zeros(0, np.complex128),
                d_obs=p.d_obs if p.d_obs is not None else np.zeros(0, np.complex128))


def make(name, p, full, ilu_level, fsgn_modes):
    ref = po.Ref(p, full=full, exact=True, ilu_level=ilu_level)
    out = problem_arrays(p)
    out["full"] = int(full)
    out["ilu_level"] = ilu_level
    x1, x2 = random_kkt(p, 101), random_kkt(p, 202)
    out["x1"], out["x2"] = x1, x2
    out["u_ref"] = ref.u()
    out["r_ref"] = ref.residual()
    rp, ci, va = ref.csr()
    out["csr_rp"], out["csr_ci"], out["csr_va"] = rp, ci, va
    out["kkt_apply_x1"] = ref.kkt_apply(x1)
    out["kkt_apply_x2"] = ref.kkt_apply(x2)
    out["kkt_rhs"] = ref.kkt_rhs()
    out["precond_exact_x1"] = ref.precond_apply(x1, _abi.FWI_PRECOND_EXACT)
    if ilu_level >= 0:
        out["precond_ilu_x1"] = ref.precond_apply(x1, _abi.FWI_PRECOND_ILU)
    if full:
        out["gradient"] = ref.gradient()
    for mode in fsgn_modes:
        ds, log = ref.fsgn(mode, 30, 0.0, 12, 2 if full else 0)
        tag = "exact" if mode == _abi.FWI_PRECOND_EXACT else "ilu"
        out[f"fsgn_{tag}_ds"] = ds
        out[f"fsgn_{tag}_res"] = np.array(log.residuals())
        out[f"fsgn_{tag}_prec"] = np.array([e.precond_residual or 0.0 for e in log.entries])
        out[f"fsgn_{tag}_normal"] = np.array([np.nan if e.normal_residual is None else e.normal_residual
                                             for e in log.entries])
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print("wrote", name, {k: np.asarray(v).shape for k, v in out.items() if np.asarray(v).size > 1})


def main():
    p = standard_instance()
    p.d_obs = po.ref_simulate(p)
    make("standard_instance", p, True, 2, [_abi.FWI_PRECOND_EXACT, _abi.FWI_PRECOND_ILU])
    p = no_receiver_instance()
    make("no_receiver_instance", p, True, -1, [_abi.FWI_PRECOND_EXACT])
    p = small_problem(nx=31, nz=23, n_pml=4, K=4, R=7, duplicate_receiver=True,
                      weight_mode=_abi.FWI_WEIGHT_OFFSET, seed=3)
    make("small_offset_dupreceivers", p, False, 3, [_abi.FWI_PRECOND_ILU])
    p = small_problem(nx=17, nz=29, n_pml=2, K=2, R=3, seed=11)
    make("small_tall", p, False, 1, [_abi.FWI_PRECOND_ILU])


if __name__ == "__main__":
    main()
