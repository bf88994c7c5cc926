"""The reference's on-disk formats on the device path.

Readers and writers for the four files the reference CLI consumes
(src/model_io.cpp, include/fwi/model_io.hpp:18-52) — model, survey, data CSV
and key = value config — with the same syntax, canonical orders, error
classes and shortest round-trip number formatting, so files written by the
reference load here and files written here are byte-identical to the
reference's. ``load_inversion`` assembles them the way ``fwi invert`` does
(tools/fwi.cpp:283-297: grid from the model header, PML amplitude from the
model's mean velocity unless the config overrides it) and ``invert`` runs the
frequency sweep on the device (``api.fwi_run``) and writes the reference's
output set (model snapshots, convergence / misfit / steps / timing CSVs).
"""
from __future__ import annotations

import math
import os
import re
from dataclasses import dataclass, field
from decimal import Decimal

import numpy as np

from . import _abi
from .problem import Grid, Problem, Survey
from .problem import pml_sigma_max as _sigma_max_of


class ParseError(ValueError):
    """fwi::ParseError (include/fwi/model_io.hpp:10-12)."""


class IoError(OSError):
    """fwi::IoError (include/fwi/model_io.hpp:13-15)."""


# --------------------------------------------------------------------------
# numbers: std::to_chars / std::from_chars semantics (src/model_io.cpp:18-41)
# --------------------------------------------------------------------------

def format_double(v: float) -> str:
    """Shortest round-trip decimal as std::to_chars(double) prints it: the shorter of the fixed
    and scientific forms of the shortest digit string, fixed on a tie (model_io.cpp:18-22)."""
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    if v == 0.0:
        return sign + "0"
    t = Decimal(repr(abs(v))).as_tuple()  # repr = shortest round-trip digits
    digits = "".join(map(str, t.digits)).lstrip("0")
    exp = t.exponent
    # normalise: value = int(digits) * 10**exp with no trailing zeros in digits
    stripped = digits.rstrip("0")
    exp += len(digits) - len(stripped)
    digits = stripped
    if exp >= 0:  # an integer: fixed notation prints its exact digits (closest of equal length)
        fixed = str(int(abs(v)))
    else:
        pos = len(digits) + exp
        fixed = digits[:pos] + "." + digits[pos:] if pos > 0 else "0." + "0" * (-pos) + digits
    e10 = exp + len(digits) - 1
    sci = digits[0] + ("." + digits[1:] if len(digits) > 1 else "") + "e" + ("-" if e10 < 0 else "+") + \
        f"{abs(e10):02d}"
    return sign + (fixed if len(fixed) <= len(sci) else sci)


_FLOAT_RE = re.compile(r"-?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|(?i:inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?))")
_INT_RE = re.compile(r"-?\d+")


def parse_double(tok: str, what: str) -> float:
    """std::from_chars(double) over the whole token (model_io.cpp:26-32); a finite literal
    that overflows ('1e400') is result_out_of_range there, a parse error here too."""
    if not _FLOAT_RE.fullmatch(tok):
        raise ParseError(f"bad numeric value for {what}: '{tok}'")
    v = float(tok)
    if math.isinf(v) and "inf" not in tok.lower():
        raise ParseError(f"bad numeric value for {what}: '{tok}'")
    return v


def parse_int(tok: str, what: str) -> int:
    """std::from_chars(int) over the whole token (model_io.cpp:34-40)."""
    if not _INT_RE.fullmatch(tok) or not -2 ** 31 <= int(tok) < 2 ** 31:
        raise ParseError(f"bad integer value for {what}: '{tok}'")
    return int(tok)


def atomic_write(path: str, content: bytes) -> None:
    """Write-temp-then-rename (model_io.cpp:60-71)."""
    tmp = str(path) + ".tmp"
    try:
        with open(tmp, "wb") as f:
            f.write(content)
    except OSError as e:
        raise IoError(f"cannot open {tmp} for writing") from e
    try:
        os.replace(tmp, path)
    except OSError as e:
        raise IoError(f"failed renaming {tmp} to {path}") from e


# --------------------------------------------------------------------------
# model file (model_io.cpp:93-144)
# --------------------------------------------------------------------------

VELOCITY_MPS, SLOWNESS_SQ = 0, 1


@dataclass
class ModelFile:
    """fwi::ModelFile (model_io.hpp:21-30): grid, value kind, nx*nz values (x fastest)."""
    grid: Grid
    kind: int
    values: np.ndarray

    def to_slowness(self) -> np.ndarray:
        """ModelFile::to_slowness (model_io.cpp:73-84): squared slowness 1/v^2."""
        v = np.asarray(self.values, np.float64)
        s = v.copy() if self.kind == SLOWNESS_SQ else 1.0 / (v * v)
        if s.size != self.grid.n or not np.all(np.isfinite(s)) or not np.all(s > 0):
            raise ValueError("SlownessModel: values must be finite, positive and match the grid")
        return s

    def mean_velocity(self) -> float:
        """ModelFile::mean_velocity (model_io.cpp:86-91): sequential sum, as the reference."""
        acc = 0.0
        for x in np.asarray(self.values, np.float64).tolist():
            acc += x if self.kind == VELOCITY_MPS else 1.0 / math.sqrt(x)
        return acc / float(self.values.size)


def _header_field(toks: list[str], key: str) -> str:
    prefix = key + "="
    for t in toks:
        if t.startswith(prefix):
            return t[len(prefix):]
    raise ParseError(f"model header: missing field '{key}'")


def read_model(path: str) -> ModelFile:
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError as e:
        raise IoError(f"cannot open model file {path}") from e
    if not raw:
        raise ParseError("model header: empty file")
    nl = raw.find(b"\n")
    header, payload = (raw, b"") if nl < 0 else (raw[:nl], raw[nl + 1:])
    toks = header.decode("latin-1").split()
    if not toks or toks[0] != "fwi-model":
        raise ParseError("model header: missing 'fwi-model' magic")
    nx = parse_int(_header_field(toks, "nx"), "nx")
    nz = parse_int(_header_field(toks, "nz"), "nz")
    h = parse_double(_header_field(toks, "h"), "h")
    n_pml = parse_int(_header_field(toks, "n_pml"), "n_pml")
    kind_s = _header_field(toks, "kind")
    if kind_s == "velocity_mps":
        kind = VELOCITY_MPS
    elif kind_s == "slowness_sq":
        kind = SLOWNESS_SQ
    else:
        raise ParseError(f"model header: bad field 'kind': '{kind_s}'")
    grid = Grid(nx, nz, h, n_pml)
    grid.validate()  # build_grid's std::invalid_argument
    need = nx * nz * 8
    if len(payload) < need:
        raise ParseError(f"model payload: expected {need} bytes, found {len(payload)}")
    if len(payload) > need:
        raise ParseError("model payload: trailing bytes beyond declared length")
    values = np.frombuffer(payload, dtype="<f8").astype(np.float64)
    if not np.all(np.isfinite(values)) or not np.all(values > 0.0):
        raise ParseError("model payload: values must be finite and positive")
    return ModelFile(grid, kind, values)


def write_model(path: str, m: ModelFile) -> None:
    g = m.grid
    vals = np.ascontiguousarray(m.values, dtype="<f8")
    if vals.size != g.n:
        raise ValueError("write_model: value count does not match grid")
    head = (f"fwi-model nx={g.nx} nz={g.nz} h={format_double(g.h)} n_pml={g.n_pml} kind="
            f"{'velocity_mps' if m.kind == VELOCITY_MPS else 'slowness_sq'}\n")
    atomic_write(path, head.encode() + vals.tobytes())


# --------------------------------------------------------------------------
# survey file (model_io.cpp:146-217)
# --------------------------------------------------------------------------

@dataclass
class SurveySource:
    ix: int
    iz: int
    amplitude: float = 1.0
    receivers: list = field(default_factory=list)  # [(ix, iz), ...]


@dataclass
class SurveyFile:
    """fwi::Survey as the file holds it (include/fwi/forward.hpp:16-33)."""
    frequencies_hz: list = field(default_factory=list)
    weight_mode: int = _abi.FWI_WEIGHT_IDENTITY
    sources: list = field(default_factory=list)

    @property
    def num_sources(self) -> int:
        return len(self.sources)

    @property
    def num_data(self) -> int:
        return sum(len(s.receivers) for s in self.sources)

    def to_survey(self, weight_mode: int | None = None) -> Survey:
        sv = Survey.per_source([(s.ix, s.iz) for s in self.sources], [list(s.receivers) for s in self.sources],
                               weight_mode=self.weight_mode if weight_mode is None else weight_mode)
        sv.src_amp = np.array([s.amplitude for s in self.sources], np.float64)
        return sv

    def validate(self, grid: Grid, require_data: bool = True) -> None:
        """Survey::validate (src/forward.cpp:23-41)."""
        if not self.sources:
            raise ValueError("Survey: no sources")
        for k, s in enumerate(self.sources):
            if not grid.usable_node(s.ix, s.iz):
                raise ValueError(f"Survey: source {k} is outside the core region")
            for rx, rz in s.receivers:
                if not grid.usable_node(rx, rz):
                    raise ValueError(f"Survey: receiver of source {k} is outside the core region")
        if require_data and self.num_data == 0:
            raise ValueError("Survey: no receivers configured")
        for f in self.frequencies_hz:
            if not f > 0.0:
                raise ValueError("Survey: frequencies must be positive")


def _text_lines(path: str, what: str) -> list[str]:
    try:
        with open(path, "rb") as f:
            raw = f.read().decode("latin-1")
    except OSError as e:
        raise IoError(f"cannot open {what} file {path}") from e
    lines = raw.split("\n")
    if lines and lines[-1] == "":
        lines.pop()  # std::getline: a final newline does not start another line
    return lines


def read_survey(path: str) -> SurveyFile:
    s = SurveyFile()
    have_magic = False
    for lineno, line in enumerate(_text_lines(path, "survey"), 1):
        def fail(msg):
            raise ParseError(f"survey line {lineno}: {msg}")
        toks = line.split("#", 1)[0].split()
        if not toks:
            continue
        if not have_magic:
            if toks[0] != "fwi-survey":
                fail("missing 'fwi-survey' magic")
            have_magic = True
            continue
        d = toks[0]
        if d == "frequencies_hz":
            s.frequencies_hz += [parse_double(t, "frequency") for t in toks[1:]]
        elif d == "weight_mode":
            if len(toks) != 2:
                fail("weight_mode takes one value")
            if toks[1] == "identity":
                s.weight_mode = _abi.FWI_WEIGHT_IDENTITY
            elif toks[1] == "offset":
                s.weight_mode = _abi.FWI_WEIGHT_OFFSET
            else:
                fail(f"unknown weight_mode '{toks[1]}'")
        elif d == "source":
            if len(toks) not in (3, 4):
                fail("source takes ix iz [amplitude]")
            src = SurveySource(parse_int(toks[1], "source ix"), parse_int(toks[2], "source iz"))
            if len(toks) == 4:
                src.amplitude = parse_double(toks[3], "source amplitude")
            s.sources.append(src)
        elif d == "receivers":
            if not s.sources:
                fail("receivers before any source")
            if len(toks) % 2 == 0:
                fail("receivers takes ix iz pairs")
            for i in range(1, len(toks) - 1, 2):
                s.sources[-1].receivers.append((parse_int(toks[i], "receiver ix"),
                                                parse_int(toks[i + 1], "receiver iz")))
        else:
            fail(f"unknown directive '{d}'")
    if not have_magic:
        raise ParseError("survey file: missing 'fwi-survey' magic")
    if not s.frequencies_hz:
        raise ParseError("survey file: no frequencies configured")
    return s


def write_survey(path: str, s: SurveyFile) -> None:
    out = ["fwi-survey\n", "frequencies_hz"]
    out += [" " + format_double(f) for f in s.frequencies_hz]
    out.append(f"\nweight_mode {'identity' if s.weight_mode == _abi.FWI_WEIGHT_IDENTITY else 'offset'}\n")
    for src in s.sources:
        out.append(f"source {src.ix} {src.iz} {format_double(src.amplitude)}\n")
        out.append("receivers" + "".join(f" {rx} {rz}" for rx, rz in src.receivers) + "\n")
    atomic_write(path, "".join(out).encode())


# --------------------------------------------------------------------------
# data CSV (model_io.cpp:219-295)
# --------------------------------------------------------------------------

DATA_HEADER = "frequency_hz,source_index,receiver_index,node_x,node_z,real,imag"


def read_data(path: str, survey: SurveyFile) -> list[np.ndarray]:
    """One complex128 block of num_data values per survey frequency, canonical order."""
    lines = _text_lines(path, "data")
    if not lines:
        raise ParseError("data file: empty")
    lineno = 1

    def fail(msg):
        raise ParseError(f"data line {lineno}: {msg}")
    if lines[0] != DATA_HEADER:
        fail("unexpected CSV header")
    nd = survey.num_data
    blocks = [np.zeros(nd, np.complex128) for _ in survey.frequencies_hz]
    pos = 1
    for fi, fsv in enumerate(survey.frequencies_hz):
        off = 0
        for k, src in enumerate(survey.sources):
            for j, (rx, rz) in enumerate(src.receivers):
                lineno += 1
                if pos >= len(lines):
                    fail("unexpected end of file; data must cover every configured frequency")
                cells = lines[pos].split(",")
                pos += 1
                if lines[pos - 1].endswith(","):
                    cells = cells[:-1]  # std::getline(ss, cell, ',') drops an empty last cell
                if len(cells) != 7:
                    fail("expected 7 columns")
                f = parse_double(cells[0], "frequency_hz")
                if abs(f - fsv) > 1e-9 * max(1.0, abs(f)):
                    fail("rows out of canonical frequency order")
                if parse_int(cells[1], "source_index") != k:
                    fail("rows out of source order")
                if parse_int(cells[2], "receiver_index") != j:
                    fail("rows out of receiver order")
                if parse_int(cells[3], "node_x") != rx or parse_int(cells[4], "node_z") != rz:
                    fail("receiver node does not match survey")
                blocks[fi][off + j] = complex(parse_double(cells[5], "real"), parse_double(cells[6], "imag"))
            off += len(src.receivers)
    if pos < len(lines):
        lineno += 1
        if lines[pos].split():
            fail("trailing rows beyond the configured survey")
    return blocks


def write_data(path: str, survey: SurveyFile, blocks: list) -> None:
    if len(blocks) != len(survey.frequencies_hz):
        raise ValueError("write_data: one block per frequency required")
    out = [DATA_HEADER + "\n"]
    for fi, b in enumerate(blocks):
        b = np.asarray(b, np.complex128)
        if b.size != survey.num_data:
            raise ValueError("write_data: block length mismatch")
        fs = format_double(survey.frequencies_hz[fi])
        off = 0
        for k, src in enumerate(survey.sources):
            for j, (rx, rz) in enumerate(src.receivers):
                v = b[off + j]
                out.append(f"{fs},{k},{j},{rx},{rz},{format_double(v.real)},{format_double(v.imag)}\n")
            off += len(src.receivers)
    atomic_write(path, "".join(out).encode())


# --------------------------------------------------------------------------
# config (model_io.cpp:297-381; fields include/fwi/driver.hpp:17-42)
# --------------------------------------------------------------------------

SOLVERS = ("rsgn-cg", "fsgn-gmres-exact", "fsgn-gmres-ilu")  # InnerSolver order (driver.cpp:10-24)


@dataclass
class FileConfig:
    """fwi::FwiConfig with every key read_config accepts."""
    frequencies_hz: list = field(default_factory=list)
    epsilon_list: list = field(default_factory=list)
    epsilon_start: float = 1.0
    epsilon_end: float = 1.0
    solver: str = "fsgn-gmres-exact"
    max_inner: int = 30
    inner_tol: float = 1e-12
    gmres_restart: int = 30
    ilu_level: int = 4
    ilu_diag_shift: float = 0.0
    drop_reg_term: bool = False
    weight_mode: int | None = None
    v_min: float = 300.0
    v_max: float = 8000.0
    ecg_stride: int = 0
    ecg_stop_tol: float = 0.0
    pml_power: float = 2.0
    pml_c_ref: float | None = None
    pml_sigma_max: float | None = None

    def epsilon_for(self, step_index: int, num_steps: int) -> float:
        """FwiConfig::epsilon_for (src/driver.cpp:26-35)."""
        if self.epsilon_list:
            if len(self.epsilon_list) != num_steps:
                raise ValueError("epsilon_list length does not match frequency count")
            return self.epsilon_list[step_index]
        if num_steps <= 1:
            return self.epsilon_start
        return self.epsilon_start + (self.epsilon_end - self.epsilon_start) * step_index / (num_steps - 1)

    def validate(self) -> None:
        """FwiConfig::validate (src/driver.cpp:37-50)."""
        f = self.frequencies_hz
        if any(not f[i] > f[i - 1] for i in range(1, len(f))):
            raise ValueError("FwiConfig: frequencies must be strictly ascending")
        if any(not x > 0.0 for x in f):
            raise ValueError("FwiConfig: frequencies must be positive")
        if not self.epsilon_list and (not self.epsilon_start > 0.0 or not self.epsilon_end > 0.0):
            raise ValueError("FwiConfig: epsilon ramp endpoints must be positive")
        if any(not e > 0.0 for e in self.epsilon_list):
            raise ValueError("FwiConfig: epsilon values must be positive")
        if self.max_inner < 1:
            raise ValueError("FwiConfig: max_inner must be >= 1")
        if not self.v_min > 0.0 or not self.v_max > self.v_min:
            raise ValueError("FwiConfig: need 0 < v_min < v_max")


def read_config(path: str) -> FileConfig:
    c = FileConfig()
    dbl = {"epsilon_start", "epsilon_end", "inner_tol", "ilu_diag_shift", "v_min", "v_max", "ecg_stop_tol",
           "pml_power", "pml_c_ref", "pml_sigma_max"}
    ints = {"max_inner", "gmres_restart", "ilu_level", "ecg_stride"}
    for lineno, line in enumerate(_text_lines(path, "config"), 1):
        def fail(msg):
            raise ParseError(f"config line {lineno}: {msg}")
        line = line.split("#", 1)[0]
        if "=" not in line:
            if line.split():
                fail("expected 'key = value'")
            continue
        eq = line.index("=")
        keys, vals = line[:eq].split(), line[eq + 1:].split()
        if len(keys) != 1:
            fail("expected a single key before '='")
        if not vals:
            fail("missing value")
        key = keys[0]

        def one():
            if len(vals) != 1:
                fail(f"key '{key}' takes a single value")
            return vals[0]
        if key == "frequencies_hz":
            c.frequencies_hz = [parse_double(v, key) for v in vals]
        elif key == "epsilon_list":
            c.epsilon_list = [parse_double(v, key) for v in vals]
        elif key == "solver":
            v = one()
            if v not in SOLVERS:
                raise ValueError(f"unknown inner solver '{v}'")  # std::invalid_argument
            c.solver = v
        elif key == "drop_reg_term":
            v = one()
            if v not in ("true", "false"):
                fail("drop_reg_term must be true or false")
            c.drop_reg_term = v == "true"
        elif key == "weight_mode":
            v = one()
            if v == "identity":
                c.weight_mode = _abi.FWI_WEIGHT_IDENTITY
            elif v == "offset":
                c.weight_mode = _abi.FWI_WEIGHT_OFFSET
            else:
                fail(f"unknown weight_mode '{v}'")
        elif key in dbl:
            setattr(c, key, parse_double(one(), key))
        elif key in ints:
            setattr(c, key, parse_int(one(), key))
        else:
            fail(f"unknown key '{key}'")
    return c


# --------------------------------------------------------------------------
# fwi invert from files (tools/fwi.cpp:283-338) on the device
# --------------------------------------------------------------------------

@dataclass
class Inversion:
    """What cmd_invert assembles: the problem (grid, PML profile, survey), observed data per
    frequency, the starting model, the config and the frequency / epsilon schedule."""
    problem: Problem
    observed: dict
    s0: np.ndarray
    config: FileConfig
    frequencies: list
    epsilons: dict


def load_inversion(model_path: str, survey_path: str, data_path: str, config_path: str | None = None,
                   pml_power: float = 0.0, pml_c_ref: float = 0.0, pml_sigma_max: float = 0.0) -> Inversion:
    mf = read_model(model_path)
    sf = read_survey(survey_path)
    sf.validate(mf.grid)
    cfg = read_config(config_path) if config_path else FileConfig()
    # PmlFlags::resolve (tools/fwi.cpp:28-38)
    power = pml_power if pml_power > 0.0 else cfg.pml_power
    c_ref = pml_c_ref if pml_c_ref > 0.0 else (cfg.pml_c_ref if cfg.pml_c_ref is not None else mf.mean_velocity())
    if not c_ref > 0.0:  # make_pml_profile (src/grid.cpp:21-27)
        raise ValueError("make_pml_profile: c_ref must be positive")
    if not power > 0.0:
        raise ValueError("make_pml_profile: power must be positive")
    grid = Grid(mf.grid.nx, mf.grid.nz, mf.grid.h, mf.grid.n_pml, _sigma_max_of(mf.grid, c_ref), power)
    if pml_sigma_max > 0.0:
        grid.sigma_max = pml_sigma_max
    elif cfg.pml_sigma_max is not None:
        grid.sigma_max = cfg.pml_sigma_max
    blocks = read_data(data_path, sf)
    observed = {float(f): b for f, b in zip(sf.frequencies_hz, blocks)}
    cfg.validate()
    freqs = sorted(cfg.frequencies_hz or sf.frequencies_hz)
    epsilons = {f: cfg.epsilon_for(i, len(freqs)) for i, f in enumerate(freqs)}
    s0 = mf.to_slowness()
    survey = sf.to_survey(cfg.weight_mode)
    prob = Problem(grid=grid, survey=survey, freq_hz=freqs[0], epsilon=epsilons[freqs[0]], s=s0,
                   drop_reg_term=cfg.drop_reg_term, name=os.path.basename(model_path))
    return Inversion(prob, observed, s0, cfg, freqs, epsilons)


def _observed_at(inv: Inversion, f: float) -> np.ndarray:
    for fo, b in inv.observed.items():  # frequency_index (src/driver.cpp:54-62)
        if abs(fo - f) <= 1e-9 * max(1.0, abs(fo)):
            return b
    raise ValueError(f"no observed data at frequency {f}")


class InversionAborted(RuntimeError):
    """fwi_run's incomplete report (FwiReport::completed == false, src/driver.cpp:142-152):
    raised by invert after the outputs of the completed steps are written (fwi invert exits 4)."""

    def __init__(self, msg: str, steps: list):
        super().__init__(msg)
        self.steps = steps


def invert(inv: Inversion, out_dir: str) -> list:
    """fwi_run over the schedule on the device (src/driver.cpp:129-155: a failing step ends the
    sweep, keeping the completed steps), then cmd_invert's outputs (tools/fwi.cpp:299-337) for
    the completed steps: model_XX.mod (velocity), heatmap_XX.ppm + .txt, convergence_XX.csv,
    misfit.csv, steps.csv, timing.csv. Raises InversionAborted after writing them if a step
    failed."""
    from dataclasses import replace

    from . import api
    c = inv.config
    gcfg = api.FwiConfig(solver=c.solver, max_inner=c.max_inner, inner_tol=c.inner_tol,
                         gmres_restart=c.gmres_restart, ilu_level=c.ilu_level, ilu_diag_shift=c.ilu_diag_shift,
                         v_min=c.v_min, v_max=c.v_max, ecg_stride=c.ecg_stride, ecg_stop_tol=c.ecg_stop_tol)
    os.makedirs(out_dir, exist_ok=True)
    steps, s, error = [], inv.s0, None
    for f in inv.frequencies:
        try:
            q = replace(inv.problem, d_obs=_observed_at(inv, f))
            r = api.gn_step(q, s, f, inv.epsilons[f], gcfg)
        except Exception as e:  # noqa: BLE001 — fwi_run catches std::exception
            error = f"step at {f:.6f} Hz failed: {e}"
            break
        steps.append(r)
        s = r.s
    misfit = ["frequency_hz,resid_norm_ini,resid_norm_fin\n"]
    rows = ["frequency_hz,epsilon,iterations,update_relnorm,final_inner_residual\n"]
    timing = ["frequency_hz,wall_seconds\n"]
    for i, st in enumerate(steps):
        misfit.append(f"{format_double(st.freq_hz)},{format_double(st.misfit_ini)},{format_double(st.misfit_fin)}\n")
        rows.append(f"{format_double(st.freq_hz)},{format_double(st.epsilon)},{st.log.iterations()},"
                    f"{format_double(st.update_relnorm)},{format_double(st.log.final_residual())}\n")
        timing.append(f"{format_double(st.freq_hz)},{st.wall_seconds:.3f}\n")
        tag = f"{i:02d}"
        vel = 1.0 / np.sqrt(st.s)
        write_model(os.path.join(out_dir, f"model_{tag}.mod"), ModelFile(inv.problem.grid, VELOCITY_MPS, vel))
        write_heatmap(os.path.join(out_dir, f"heatmap_{tag}.ppm"), inv.problem.grid, vel)
        write_convergence_csv(os.path.join(out_dir, f"convergence_{tag}.csv"), st.log)
    atomic_write(os.path.join(out_dir, "misfit.csv"), "".join(misfit).encode())
    atomic_write(os.path.join(out_dir, "steps.csv"), "".join(rows).encode())
    atomic_write(os.path.join(out_dir, "timing.csv"), "".join(timing).encode())
    if error is not None:
        raise InversionAborted(error, steps)
    return steps


def write_convergence_csv(path: str, log) -> None:
    """write_convergence_csv (tools/fwi.cpp:45-53)."""
    conv = ["iteration,normal_resid,solver_resid,precond_resid\n"]
    for e in log.entries:
        nr = format_double(e.normal_residual) if e.normal_residual is not None else ""
        pr = format_double(e.precond_residual) if e.precond_residual is not None else ""
        conv.append(f"{e.iteration},{nr},{format_double(e.residual_norm)},{pr}\n")
    atomic_write(path, "".join(conv).encode())


def write_timing_csv(path: str, log) -> None:
    """write_timing_csv (tools/fwi.cpp:55-63)."""
    out = ["iteration,wall_seconds\n"] + [f"{e.iteration},{e.wall_time:.3f}\n" for e in log.entries]
    atomic_write(path, "".join(out).encode())


# --------------------------------------------------------------------------
# heatmap and model generators (src/model_io.cpp:383-513)
# --------------------------------------------------------------------------

_STOPS = ((0, 0, 96), (32, 96, 255), (245, 245, 245), (255, 128, 32), (128, 16, 16))


def _colormap(t: float):
    """The fixed diverging colormap (model_io.cpp:389-401)."""
    t = min(max(t, 0.0), 1.0)
    pos = t * 4.0
    i = min(3, int(pos))
    f = pos - i
    a, b = _STOPS[i], _STOPS[i + 1]
    return tuple(a[c] + f * (b[c] - a[c]) for c in range(3))


def write_heatmap(path: str, grid: Grid, node_values) -> None:
    """write_heatmap (model_io.cpp:405-435): binary PPM of the core, min/max .txt sidecar."""
    v = np.asarray(node_values, np.float64)
    if v.size != grid.n:
        raise ValueError("write_heatmap: value count does not match grid")
    p = grid.n_pml
    core = v.reshape(grid.nz, grid.nx)[p:grid.nz - p, p:grid.nx - p]
    lo, hi = float(core.min()), float(core.max())
    span = hi - lo if hi > lo else 1.0
    px = bytearray()
    for val in core.ravel().tolist():
        r, g, b = _colormap((val - lo) / span)
        px += bytes((int(r + 0.5) & 255, int(g + 0.5) & 255, int(b + 0.5) & 255))
    atomic_write(path, f"P6\n{core.shape[1]} {core.shape[0]}\n255\n".encode() + bytes(px))
    atomic_write(os.path.splitext(path)[0] + ".txt", f"min {format_double(lo)}\nmax {format_double(hi)}\n".encode())


def make_layered_model(grid: Grid, velocities: list, interfaces: list) -> ModelFile:
    """make_layered_model (model_io.cpp:437-463)."""
    if not velocities:
        raise ValueError("make_layered_model: need at least one layer")
    if len(interfaces) + 1 != len(velocities):
        raise ValueError("make_layered_model: need one interface fewer than layers")
    for i, z in enumerate(interfaces):
        if z <= 0 or z >= grid.nz:
            raise ValueError("make_layered_model: interface outside the grid")
        if i > 0 and z <= interfaces[i - 1]:
            raise ValueError("make_layered_model: interfaces must ascend")
    if any(not v > 0.0 for v in velocities):
        raise ValueError("make_layered_model: velocities must be positive")
    vals = np.empty(grid.n)
    for iz in range(grid.nz):
        layer = 0
        while layer < len(interfaces) and iz >= interfaces[layer]:
            layer += 1
        vals[iz * grid.nx:(iz + 1) * grid.nx] = velocities[layer]
    return ModelFile(grid, VELOCITY_MPS, vals)


def make_lens_model(grid: Grid, background: float, amplitude: float, cx: float, cz: float,
                    radius: float) -> ModelFile:
    """make_lens_model (model_io.cpp:465-487), the same operations per node."""
    if not background > 0.0:
        raise ValueError("make_lens_model: background must be positive")
    if not radius > 0.0:
        raise ValueError("make_lens_model: radius must be positive")
    two_r2 = 2.0 * radius * radius
    vals = np.empty(grid.n)
    for iz in range(grid.nz):
        for ix in range(grid.nx):
            dx, dz = ix - cx, iz - cz
            v = background + amplitude * math.exp(-(dx * dx + dz * dz) / two_r2)
            if not v > 0.0:
                raise ValueError("make_lens_model: non-positive velocity produced")
            vals[iz * grid.nx + ix] = v
    return ModelFile(grid, VELOCITY_MPS, vals)


def import_raw_model(grid: Grid, raw_path: str, out_kind: int) -> ModelFile:
    """import_raw_model (model_io.cpp:489-513): headerless float32 velocities."""
    try:
        with open(raw_path, "rb") as f:
            raw = f.read()
    except OSError as e:
        raise IoError(f"cannot open raw model {raw_path}") from e
    expected = grid.n * 4
    if len(raw) != expected:
        raise ParseError(f"raw model: expected {expected} bytes ({grid.n} float32 values), found {len(raw)}")
    v = np.frombuffer(raw, dtype="<f4").astype(np.float64)
    if not np.all(np.isfinite(v)) or not np.all(v > 0.0):
        raise ParseError("raw model: velocities must be finite and positive")
    return ModelFile(grid, out_kind, v if out_kind == VELOCITY_MPS else 1.0 / (v * v))
