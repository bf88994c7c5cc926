"""GPU: `fwi invert` from the reference's own files (tools/fwi.cpp:283-338) on the device —
model / survey / data / config written by the reference's writers (oracle/_ref), loaded by
paper_2204_06489_b200.model_io, inverted with the device gn_step, and checked step by step
against the reference's gn_step chain on the same inputs (north-star gate: 1e-6 relative L2)."""
import ctypes as C
import os

import numpy as np
import pytest

import pyoracle as po
from paper_2204_06489_b200 import model_io as mio
from paper_2204_06489_b200.problem import Problem, c1_problem, pml_sigma_max

pytestmark = pytest.mark.gpu
_dp, _ip = C.POINTER(C.c_double), C.POINTER(C.c_int)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def test_invert_from_reference_files_matches_reference_chain(tmp_path):
    L = po.ref_lib()
    L.ref_write_model.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, _dp]
    L.ref_write_survey.argtypes = [C.c_char_p, C.c_int, _dp, C.c_int, C.c_int, _ip, _ip, _dp, _ip, _ip, _ip]
    L.ref_write_data.argtypes = [C.c_char_p, C.c_char_p, _dp]
    p = c1_problem()
    g, sv = p.grid, p.survey
    freqs = [4.0, 5.0]
    mp, sp, dpth, cp = (str(tmp_path / n) for n in ("start.mod", "survey.txt", "data.csv", "fwi.cfg"))
    v0 = 1.0 / np.sqrt(p.s)
    assert L.ref_write_model(mp.encode(), g.nx, g.nz, g.h, g.n_pml, 0, v0.ctypes.data_as(_dp)) == 0
    fr = np.array(freqs)
    amp = np.ones(sv.num_sources)
    off = np.ascontiguousarray(sv.recv_offset, np.int32)
    arrs = [np.ascontiguousarray(a, np.int32) for a in (sv.src_ix, sv.src_iz, sv.recv_ix, sv.recv_iz)]
    ip = lambda a: a.ctypes.data_as(_ip)  # noqa: E731
    assert L.ref_write_survey(sp.encode(), 2, fr.ctypes.data_as(_dp), sv.weight_mode, sv.num_sources, ip(arrs[0]),
                              ip(arrs[1]), amp.ctypes.data_as(_dp), ip(off), ip(arrs[2]), ip(arrs[3])) == 0
    # observed data: the reference forward solve on the truth, with the PML the CLI derives
    # from the starting model file (mean velocity)
    mf = mio.read_model(mp)
    g2 = type(g)(g.nx, g.nz, g.h, g.n_pml, pml_sigma_max(mf.grid, mf.mean_velocity()), 2.0)
    blocks = []
    for f in freqs:
        q = Problem(grid=g2, survey=sv, freq_hz=f, epsilon=1.0, s=p.s, s_true=p.s_true)
        blocks.append(po.ref_simulate(q))
    flat = np.ascontiguousarray(np.concatenate(blocks)).view(np.float64)
    assert L.ref_write_data(dpth.encode(), sp.encode(), flat.ctypes.data_as(_dp)) == 0
    with open(cp, "w") as fcfg:
        fcfg.write("# two frequencies, paper setting (drop_reg_term)\nsolver = fsgn-gmres-exact\n"
                   "epsilon_list = 1e10 1.5e10\ndrop_reg_term = true\ninner_tol = 1e-3\nmax_inner = 30\n")

    inv = mio.load_inversion(mp, sp, dpth, cp)
    assert inv.problem.grid.sigma_max == g2.sigma_max
    out = str(tmp_path / "out")
    steps = mio.invert(inv, out)

    s = inv.s0
    for st, f in zip(steps, freqs):
        q = Problem(grid=inv.problem.grid, survey=inv.problem.survey, freq_hz=f, epsilon=inv.epsilons[f], s=s,
                    drop_reg_term=True, d_obs=inv.observed[f])
        s_ref, mi_ref, mf_ref, log_ref = po.ref_gn_step(q, solver=1, max_inner=30, inner_tol=1e-3, restart=30)
        print(f"f={f}: model rel dev {rel(st.s, s_ref):.2e}, its {st.log.iterations()} vs {log_ref.iterations()}")
        assert rel(st.s, s_ref) <= 1e-6
        assert abs(st.misfit_ini - mi_ref) <= 1e-8 * mi_ref
        assert st.log.iterations() == log_ref.iterations()
        s = st.s  # per-step parity: the reference step starts from the device model
    for name in ("misfit.csv", "steps.csv", "timing.csv", "model_00.mod", "model_01.mod", "convergence_01.csv"):
        assert os.path.exists(os.path.join(out, name)), name
    snap = mio.read_model(os.path.join(out, "model_01.mod"))
    assert np.array_equal(snap.values, 1.0 / np.sqrt(steps[-1].s))
    rows = open(os.path.join(out, "steps.csv")).read().splitlines()
    assert rows[0] == "frequency_hz,epsilon,iterations,update_relnorm,final_inner_residual" and len(rows) == 3
    assert rows[1].startswith("4,1e+10,")
