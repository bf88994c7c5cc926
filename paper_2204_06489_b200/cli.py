"""`fwi` command line on the device path — the reference CLI (tools/fwi.cpp:342-435) with the
same subcommands, flags, outputs and exit codes:

    python -m paper_2204_06489_b200.cli make-model      --kind layered|lens|import-raw ...
    python -m paper_2204_06489_b200.cli simulate        --model M --survey S --out D [--config C]
    python -m paper_2204_06489_b200.cli compare-solvers --initial M --survey S (--data D | --true-model T)
                                                        --out DIR [--freq F] [--ilu-levels 0,4,21]
    python -m paper_2204_06489_b200.cli invert          --initial M --survey S --data D --out DIR [--config C]

PML flags --pml-power / --pml-c-ref / --pml-sigma-max on simulate, compare-solvers and invert
(PmlFlags, tools/fwi.cpp:16-39). Exit codes (tools/fwi.cpp:415-433): 0 ok; 2 io error
(IoError); 3 parse error or invalid input (ParseError, std::invalid_argument); 4 any other
failure, and an inversion that aborted after writing its completed steps. Command-line usage
errors take CLI11's codes: 106 a required option or the subcommand missing, 109 an unknown
argument, 104 a value that does not convert.

Forward solves, the reduced-space CG, both GMRES variants and the Newton steps run on the B200
through the C ABI (libfwi_b200.so); the file formats are model_io.py's, byte-identical to the
reference's writers.
"""
from __future__ import annotations

import argparse
import os
import sys
import time
from dataclasses import replace

import numpy as np

from . import model_io as mio
from .problem import Grid, Problem


class _Usage(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # CLI11's exit codes instead of argparse's 2
        code = 106
        if "unrecognized arguments" in message:
            code = 109
        elif "invalid" in message and "value" in message:
            code = 104
        raise _Usage(code, f"{self.prog}: {message}")


def _csv(kind):
    def conv(text):
        return [kind(t) for t in text.split(",") if t != ""]
    return conv


def _pml(p):
    p.add_argument("--pml-power", type=float, default=0.0, help="PML ramp exponent (default 2)")
    p.add_argument("--pml-c-ref", type=float, default=0.0,
                   help="reference speed for the PML amplitude (default: model mean)")
    p.add_argument("--pml-sigma-max", type=float, default=0.0, help="explicit PML damping amplitude, 1/s")


def _grid_with_pml(mf: mio.ModelFile, cfg: mio.FileConfig, a) -> Grid:
    """PmlFlags::resolve (tools/fwi.cpp:28-38)."""
    from .problem import pml_sigma_max
    power = a.pml_power if a.pml_power > 0.0 else cfg.pml_power
    c_ref = a.pml_c_ref if a.pml_c_ref > 0.0 else (cfg.pml_c_ref if cfg.pml_c_ref is not None
                                                    else mf.mean_velocity())
    if not c_ref > 0.0:
        raise ValueError("make_pml_profile: c_ref must be positive")
    if not power > 0.0:
        raise ValueError("make_pml_profile: power must be positive")
    g = Grid(mf.grid.nx, mf.grid.nz, mf.grid.h, mf.grid.n_pml, pml_sigma_max(mf.grid, c_ref), power)
    if a.pml_sigma_max > 0.0:
        g.sigma_max = a.pml_sigma_max
    elif cfg.pml_sigma_max is not None:
        g.sigma_max = cfg.pml_sigma_max
    return g


def cmd_make_model(a) -> int:
    """cmd_make_model (tools/fwi.cpp:82-113)."""
    g = Grid(a.nx, a.nz, a.spacing, a.n_pml)
    g.validate()
    mk = mio.SLOWNESS_SQ if a.out_kind == "slowness_sq" else mio.VELOCITY_MPS
    if a.kind == "layered":
        m = mio.make_layered_model(g, a.velocities, a.interfaces)
    elif a.kind == "lens":
        cx = a.center_x if a.center_x >= 0.0 else (a.nx - 1) / 2.0
        cz = a.center_z if a.center_z >= 0.0 else (a.nz - 1) / 2.0
        rad = a.radius if a.radius > 0.0 else a.nx / 8.0
        m = mio.make_lens_model(g, a.background, a.amplitude, cx, cz, rad)
    elif a.kind == "import-raw":
        if not a.raw:
            raise mio.ParseError("import-raw requires --raw")
        m = mio.import_raw_model(g, a.raw, mk)
    else:
        raise mio.ParseError(f"unknown model kind '{a.kind}'")
    if mk == mio.SLOWNESS_SQ and m.kind == mio.VELOCITY_MPS:
        m = mio.ModelFile(m.grid, mio.SLOWNESS_SQ, 1.0 / (m.values * m.values))
    mio.write_model(a.out, m)
    print(f"wrote {a.out} ({a.nx}x{a.nz}, h={a.spacing:g})")
    return 0


def _simulate_blocks(grid: Grid, sf: mio.SurveyFile, s: np.ndarray, freqs) -> list:
    """Observed data per frequency with the device's exact block solver (cmd_simulate's loop,
    tools/fwi.cpp:124-130)."""
    from . import api
    out = []
    for f in freqs:
        p = Problem(grid=grid, survey=sf.to_survey(), freq_hz=float(f), epsilon=1.0, s=s)
        out.append(api.simulate(p, s))
    return out


def cmd_simulate(a) -> int:
    """cmd_simulate (tools/fwi.cpp:115-135)."""
    mf = mio.read_model(a.model)
    sf = mio.read_survey(a.survey)
    sf.validate(mf.grid)
    cfg = mio.read_config(a.config) if a.config else mio.FileConfig()
    g = _grid_with_pml(mf, cfg, a)
    blocks = _simulate_blocks(g, sf, mf.to_slowness(), sf.frequencies_hz)
    mio.write_data(a.out, sf, blocks)
    print(f"wrote {a.out} ({len(sf.frequencies_hz)} frequencies, {sf.num_data} receivers each)")
    return 0


def cmd_compare(a) -> int:
    """cmd_compare (tools/fwi.cpp:145-281): one linearisation, then CG (reduced space),
    GMRes-full (exact block preconditioner) and GMRes-approx(p) per ILU level, E_cg every
    iteration; per-solver CSVs / updates and the summary table."""
    from . import api
    mf = mio.read_model(a.initial)
    sf = mio.read_survey(a.survey)
    sf.validate(mf.grid)
    cfg = mio.read_config(a.config) if a.config else mio.FileConfig()
    g = _grid_with_pml(mf, cfg, a)
    s0 = mf.to_slowness()
    if a.data:
        blocks = mio.read_data(a.data, sf)
    else:
        if not a.true_model:
            raise mio.ParseError("compare-solvers needs --data or --true-model")
        tm = mio.read_model(a.true_model)
        blocks = _simulate_blocks(g, sf, tm.to_slowness(), sf.frequencies_hz)
    freq = a.freq
    if freq <= 0.0:
        if len(sf.frequencies_hz) != 1:
            raise mio.ParseError("compare-solvers: select one frequency with --freq")
        freq = sf.frequencies_hz[0]
    fi = -1
    for i, f in enumerate(sf.frequencies_hz):
        if abs(f - freq) <= 1e-9 * freq:
            fi = i
    if fi < 0:
        raise mio.ParseError("compare-solvers: no data at the requested frequency")
    levels = a.ilu_levels or [cfg.ilu_level]
    eps = cfg.epsilon_for(0, 1)
    p = Problem(grid=g, survey=sf.to_survey(cfg.weight_mode), freq_hz=float(freq), epsilon=eps, s=s0,
                drop_reg_term=cfg.drop_reg_term, d_obs=blocks[fi])
    st = api.GnState(p, exact=True)
    os.makedirs(a.out, exist_ok=True)
    runs = []
    tol = cfg.ecg_stop_tol if cfg.ecg_stop_tol > 0.0 else cfg.inner_tol
    ds, log = api.rsgn_cg_step(st, tol, cfg.max_inner)
    runs.append(("CG", "cg", log, ds, 0.0))
    o = api.FsgnOptions(mode=api.PrecondMode.exact, restart=cfg.gmres_restart, tol=cfg.inner_tol,
                        maxit=cfg.max_inner, ecg_stride=1, ecg_stop_tol=cfg.ecg_stop_tol)
    ds, log = api.fsgn_gmres_step(st, o)
    runs.append(("GMRes-full", "gmres_full", log, ds, 0.0))
    for lev in levels:
        t0 = time.perf_counter()
        st.factor_ilu(lev, cfg.ilu_diag_shift)
        setup = time.perf_counter() - t0
        ds, log = api.fsgn_gmres_step(st, replace(o, mode=api.PrecondMode.ilu))
        runs.append((f"GMRes-approx(p={lev})", f"gmres_ilu_p{lev}", log, ds, setup))
    st.close()
    for label, tag, log, ds, setup in runs:
        mio.write_convergence_csv(os.path.join(a.out, f"convergence_{tag}.csv"), log)
        mio.write_timing_csv(os.path.join(a.out, f"timing_{tag}.csv"), log)
        mio.atomic_write(os.path.join(a.out, f"update_{tag}.f64"), np.asarray(ds, "<f8").tobytes())
    header, r_iter = "metric", "Iterations"
    r_tpi, r_ilu, r_tot = '"Time per iteration, s"', '"ILU initialization, s"', '"Total time, s"'
    print(f"{'solver':<28s} {'iterations':>12s} {'time/iteration [s]':>18s} {'ILU initialization [s]':>20s} "
          f"{'total [s]':>14s}")
    for label, tag, log, ds, setup in runs:
        it = log.iterations()
        wall = log.entries[-1].wall_time if log.entries else 0.0
        tpi = wall / it if it > 0 else 0.0
        total = wall + setup
        header += f',"{label}"'
        r_iter += f",{it}"
        r_tpi += f",{tpi:.3f}"
        r_ilu += f",{setup:.3f}"
        r_tot += f",{total:.3f}"
        print(f"{label:<28s} {it:12d} {tpi:18.3f} {setup:20.3f} {total:14.3f}")
    mio.atomic_write(os.path.join(a.out, "summary.csv"),
                     (header + "\n" + r_iter + "\n" + r_tpi + "\n" + r_ilu + "\n" + r_tot + "\n").encode())
    return 0


def cmd_invert(a) -> int:
    """cmd_invert (tools/fwi.cpp:283-338): fwi_run on the device, outputs per completed step."""
    inv = mio.load_inversion(a.initial, a.survey, a.data, a.config or None, a.pml_power, a.pml_c_ref,
                             a.pml_sigma_max)
    try:
        steps = mio.invert(inv, a.out)
        aborted = None
    except mio.InversionAborted as e:
        steps, aborted = e.steps, str(e)
    for st in steps:
        print(f"f = {st.freq_hz:<8g} Hz   misfit {st.misfit_ini:.6f} -> {st.misfit_fin:.6f}   "
              f"({st.log.iterations()} inner iterations)")
    if aborted is not None:
        print(f"inversion aborted: {aborted}", file=sys.stderr)
        return 4
    return 0


def parser() -> argparse.ArgumentParser:
    ap = _Parser(prog="fwi", description="2D frequency-domain acoustic full-waveform inversion (B200)")
    sub = ap.add_subparsers(dest="cmd", parser_class=_Parser)
    mm = sub.add_parser("make-model", help="generate or import a model file")
    mm.add_argument("--kind", required=True, help="layered | lens | import-raw")
    mm.add_argument("--nx", type=int, required=True)
    mm.add_argument("--nz", type=int, required=True)
    mm.add_argument("--spacing", type=float, required=True, help="grid spacing h, m")
    mm.add_argument("--n-pml", type=int, required=True)
    mm.add_argument("--out", required=True)
    mm.add_argument("--out-kind", default="velocity_mps", help="velocity_mps | slowness_sq")
    mm.add_argument("--velocities", type=_csv(float), default=[], help="layer velocities, m/s")
    mm.add_argument("--interfaces", type=_csv(int), default=[], help="layer interface depths, z nodes")
    mm.add_argument("--background", type=float, default=1500.0, help="lens background velocity, m/s")
    mm.add_argument("--amplitude", type=float, default=0.0, help="lens velocity anomaly, m/s")
    mm.add_argument("--center-x", type=float, default=-1.0, help="lens center, x node")
    mm.add_argument("--center-z", type=float, default=-1.0, help="lens center, z node")
    mm.add_argument("--radius", type=float, default=0.0, help="lens radius, nodes")
    mm.add_argument("--raw", default="", help="headerless float32 velocity grid")
    sim = sub.add_parser("simulate", help="forward-simulate data for a survey")
    sim.add_argument("--model", required=True)
    sim.add_argument("--survey", required=True)
    sim.add_argument("--out", required=True)
    sim.add_argument("--config", default="")
    _pml(sim)
    cs = sub.add_parser("compare-solvers", help="run all inner solvers on one linearization")
    cs.add_argument("--initial", required=True)
    cs.add_argument("--survey", required=True)
    cs.add_argument("--data", default="")
    cs.add_argument("--true-model", default="", help="simulate data in-memory when --data is absent")
    cs.add_argument("--config", default="")
    cs.add_argument("--freq", type=float, default=0.0, help="frequency to compare at, Hz")
    cs.add_argument("--out", required=True)
    cs.add_argument("--ilu-levels", type=_csv(int), default=[], help="fill levels for the approximate preconditioner")
    _pml(cs)
    inv = sub.add_parser("invert", help="multi-frequency inversion")
    inv.add_argument("--initial", required=True)
    inv.add_argument("--survey", required=True)
    inv.add_argument("--data", required=True)
    inv.add_argument("--config", default="")
    inv.add_argument("--out", required=True)
    _pml(inv)
    return ap


def main(argv=None) -> int:
    try:
        a = parser().parse_args(argv)
        if a.cmd is None:
            raise _Usage(106, "fwi: a subcommand is required")
    except _Usage as e:
        print(str(e), file=sys.stderr)
        return e.code
    cmds = {"make-model": cmd_make_model, "simulate": cmd_simulate, "compare-solvers": cmd_compare,
            "invert": cmd_invert}
    try:
        return cmds[a.cmd](a)
    except mio.IoError as e:
        print(f"io error: {e}", file=sys.stderr)
        return 2
    except mio.ParseError as e:
        print(f"parse error: {e}", file=sys.stderr)
        return 3
    except ValueError as e:  # std::invalid_argument (api.InvalidArgument is one too)
        print(f"invalid input: {e}", file=sys.stderr)
        return 3
    except Exception as e:  # noqa: BLE001
        print(f"error: {e}", file=sys.stderr)
        return 4


if __name__ == "__main__":
    sys.exit(main())
