"""GPU: the `fwi` command line's device subcommands (paper_2204_06489_b200/cli.py, the reference's
tools/fwi.cpp) end to end from files: simulate -> compare-solvers -> invert on a small lens
problem; the written data equal the reference's forward solve to 1e-10, the invert steps match
the reference gn_step, and an aborted inversion exits 4 after writing its completed steps."""
import os

import numpy as np
import pytest

import pyoracle as po
from paper_2204_06489_b200 import cli
from paper_2204_06489_b200 import model_io as mio
from paper_2204_06489_b200.problem import Problem

pytestmark = pytest.mark.gpu


def _files(tmp_path):
    d = tmp_path
    assert cli.main(["make-model", "--kind", "lens", "--nx", "48", "--nz", "36", "--spacing", "20", "--n-pml", "6",
                     "--out", str(d / "true.mod"), "--background", "2000", "--amplitude", "250"]) == 0
    assert cli.main(["make-model", "--kind", "lens", "--nx", "48", "--nz", "36", "--spacing", "20", "--n-pml", "6",
                     "--out", str(d / "init.mod"), "--background", "2000", "--amplitude", "0"]) == 0
    src = [mio.SurveySource(ix, 8, 1.0, [(x, 8) for x in range(8, 40, 2)]) for ix in (10, 24, 37)]
    mio.write_survey(str(d / "s.svy"), mio.SurveyFile([2.0, 3.0], 0, src))
    (d / "c.cfg").write_text("epsilon_list = 1e-3 1e-3\nmax_inner = 20\ninner_tol = 1e-6\n")
    return d


def test_simulate_compare_invert_from_files(tmp_path):
    d = _files(tmp_path)
    assert cli.main(["simulate", "--model", str(d / "true.mod"), "--survey", str(d / "s.svy"),
                     "--out", str(d / "obs.csv")]) == 0
    sf = mio.read_survey(str(d / "s.svy"))
    blocks = mio.read_data(str(d / "obs.csv"), sf)
    # the reference's forward solve on the same model/survey/PML (cmd_simulate)
    mf = mio.read_model(str(d / "true.mod"))
    from paper_2204_06489_b200.cli import _grid_with_pml
    import argparse
    g = _grid_with_pml(mf, mio.FileConfig(), argparse.Namespace(pml_power=0.0, pml_c_ref=0.0, pml_sigma_max=0.0))
    for f, b in zip(sf.frequencies_hz, blocks):
        p = Problem(grid=g, survey=sf.to_survey(), freq_hz=f, epsilon=1.0, s=mf.to_slowness())
        want = po.ref_simulate(p, p.s)
        assert np.linalg.norm(b - want) <= 1e-10 * np.linalg.norm(want)
    out = d / "cmp"
    # compare-solvers takes epsilon_for(0, 1): an epsilon_list must hold one value (as the
    # reference's cmd_compare, which rejects the two-value list with exit code 3)
    assert cli.main(["compare-solvers", "--initial", str(d / "init.mod"), "--survey", str(d / "s.svy"),
                     "--data", str(d / "obs.csv"), "--freq", "2", "--out", str(out), "--ilu-levels", "0,3",
                     "--config", str(d / "c.cfg")]) == 3
    (d / "c1.cfg").write_text("epsilon_start = 1e-3\nepsilon_end = 1e-3\nmax_inner = 20\ninner_tol = 1e-6\n")
    assert cli.main(["compare-solvers", "--initial", str(d / "init.mod"), "--survey", str(d / "s.svy"),
                     "--data", str(d / "obs.csv"), "--freq", "2", "--out", str(out), "--ilu-levels", "0,3",
                     "--config", str(d / "c1.cfg")]) == 0
    for tag in ("cg", "gmres_full", "gmres_ilu_p0", "gmres_ilu_p3"):
        assert (out / f"convergence_{tag}.csv").exists() and (out / f"update_{tag}.f64").exists()
    assert (out / "summary.csv").read_text().startswith('metric,"CG","GMRes-full"')
    inv = d / "inv"
    assert cli.main(["invert", "--initial", str(d / "init.mod"), "--survey", str(d / "s.svy"),
                     "--data", str(d / "obs.csv"), "--config", str(d / "c.cfg"), "--out", str(inv)]) == 0
    for name in ("misfit.csv", "steps.csv", "timing.csv", "model_00.mod", "model_01.mod", "heatmap_01.ppm",
                 "heatmap_01.txt", "convergence_00.csv"):
        assert (inv / name).exists(), name
    # step 0 against the reference gn_step from the same files
    invp = mio.load_inversion(str(d / "init.mod"), str(d / "s.svy"), str(d / "obs.csv"), str(d / "c.cfg"))
    q = invp.problem
    q.d_obs = invp.observed[2.0]
    q.epsilon = 1e-3
    s_ref, _, _, _ = po.ref_gn_step(q, solver=1, max_inner=20, inner_tol=1e-6, restart=30)
    v0 = mio.read_model(str(inv / "model_00.mod")).values
    assert np.linalg.norm(1.0 / v0 ** 2 - s_ref) <= 1e-6 * np.linalg.norm(s_ref)


def test_invert_abort_exits_4_after_writing_completed_steps(tmp_path):
    d = _files(tmp_path)
    assert cli.main(["simulate", "--model", str(d / "true.mod"), "--survey", str(d / "s.svy"),
                     "--out", str(d / "obs.csv")]) == 0
    # an ILU solver at an invalid fill level: the first gn_step fails (std::invalid_argument
    # from IluFactors::factor), fwi_run keeps the empty report, fwi invert exits 4
    (d / "bad.cfg").write_text("epsilon_list = 1e-3 1e-3\nsolver = fsgn-gmres-ilu\nilu_level = -1\n")
    inv = d / "inv"
    rc = cli.main(["invert", "--initial", str(d / "init.mod"), "--survey", str(d / "s.svy"),
                   "--data", str(d / "obs.csv"), "--config", str(d / "bad.cfg"), "--out", str(inv)])
    assert rc == 4
    assert (inv / "misfit.csv").read_text() == "frequency_hz,resid_norm_ini,resid_norm_fin\n"
