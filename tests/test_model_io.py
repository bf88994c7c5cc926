"""CPU: the reference's on-disk formats (src/model_io.cpp) — paper_2204_06489_b200.model_io
against the reference's own writers and readers (oracle/_ref, via ref_harness.cpp):
byte-identical output, identical parsed values, and the same inputs rejected."""
import ctypes as C
import math
import os
import struct

import numpy as np
import pytest

import pyoracle as po
from paper_2204_06489_b200 import _abi
from paper_2204_06489_b200 import model_io as mio
from paper_2204_06489_b200.problem import Grid, pml_sigma_max

_dp, _ip = C.POINTER(C.c_double), C.POINTER(C.c_int)


@pytest.fixture(scope="module")
def ref():
    L = po.ref_lib()
    L.ref_format_double.argtypes = [C.c_double, C.c_char_p, C.c_int]
    L.ref_write_model.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, _dp]
    L.ref_read_model.argtypes = [C.c_char_p, _ip, _dp, _dp, C.c_long]
    L.ref_write_survey.argtypes = [C.c_char_p, C.c_int, _dp, C.c_int, C.c_int, _ip, _ip, _dp, _ip, _ip, _ip]
    L.ref_read_survey.argtypes = [C.c_char_p, _ip, _dp, _ip, _ip, _dp, _ip, _ip, _ip]
    L.ref_write_data.argtypes = [C.c_char_p, C.c_char_p, _dp]
    L.ref_read_data.argtypes = [C.c_char_p, C.c_char_p, _dp]
    L.ref_read_config.argtypes = [C.c_char_p, _dp, _ip, _dp, _dp]
    return L


def dp(a):
    return a.ctypes.data_as(_dp)


def ip(a):
    return a.ctypes.data_as(_ip)


def ref_fmt(L, v):
    buf = C.create_string_buffer(64)
    n = L.ref_format_double(v, buf, 64)
    return buf.value[:n].decode()


def test_format_double_matches_to_chars(ref):
    rng = np.random.default_rng(5)
    vals = [0.0, -0.0, 1.0, -1.0, 5.0, 10.0, 100.0, 0.1, 0.5, 1e-5, 1e-4, 1e15, 1e16, 1e17, 123456.0,
            1234567.0, 1e21, 1e22, 1.5e-7, 2.5e300, 5e-324, 1.7976931348623157e308, 2.2250738585072014e-308,
            math.pi, -math.e, 1500.0, 3500.0, 0.004, 0.0004, 12345678901234567890.0, 1e100, 3.0e-10,
            float("inf"), float("-inf")]
    vals += list(rng.standard_normal(300) * 10.0 ** rng.integers(-30, 30, 300))
    vals += list(np.round(rng.uniform(0, 1e6, 100)))
    vals += list(rng.integers(-10 ** 9, 10 ** 9, 100).astype(float) / 10.0 ** rng.integers(0, 12, 100))
    for v in vals:
        assert mio.format_double(v) == ref_fmt(ref, float(v)), v


def test_parse_numbers_follow_from_chars():
    assert mio.parse_double("1e5", "x") == 1e5 and mio.parse_double("-.5", "x") == -0.5
    assert mio.parse_double("inf", "x") == math.inf
    for bad in ("+1", " 1", "1 ", "1_0", "0x10", "", "1e", "e5", "--1", "1.0f"):
        with pytest.raises(mio.ParseError):
            mio.parse_double(bad, "x")
    assert mio.parse_int("-12", "x") == -12
    for bad in ("+1", "1.0", "2147483648", "", "1e3"):
        with pytest.raises(mio.ParseError):
            mio.parse_int(bad, "x")


@pytest.mark.parametrize("kind", [mio.VELOCITY_MPS, mio.SLOWNESS_SQ])
def test_model_file_bytes_and_values_match_reference(tmp_path, ref, kind):
    rng = np.random.default_rng(kind + 3)
    nx, nz, h, npml = 17, 11, 12.5, 2
    v = rng.uniform(1500, 4500, nx * nz)
    vals = v if kind == mio.VELOCITY_MPS else 1.0 / (v * v)
    a, b = str(tmp_path / "ref.mod"), str(tmp_path / "ours.mod")
    assert ref.ref_write_model(a.encode(), nx, nz, h, npml, kind, dp(vals)) == 0
    mio.write_model(b, mio.ModelFile(Grid(nx, nz, h, npml), kind, vals))
    assert open(a, "rb").read() == open(b, "rb").read()
    m = mio.read_model(a)
    assert (m.grid.nx, m.grid.nz, m.grid.h, m.grid.n_pml, m.kind) == (nx, nz, h, npml, kind)
    assert np.array_equal(m.values, vals)
    if kind == mio.VELOCITY_MPS:
        assert np.array_equal(m.to_slowness(), 1.0 / (vals * vals))


def _ref_model_status(ref, path):
    hdr = np.zeros(4, np.int32)
    h = np.zeros(1)
    return ref.ref_read_model(path.encode(), ip(hdr), dp(h), None, 0)


@pytest.mark.parametrize("case", ["magic", "field", "kind", "int", "short", "trailing", "nonpositive",
                                  "nan", "empty"])
def test_model_file_rejections_match_reference(tmp_path, ref, case):
    body = struct.pack("<6d", *([2000.0] * 6))
    head = b"fwi-model nx=3 nz=2 h=10 n_pml=0 kind=velocity_mps\n"
    data = {
        "magic": b"fwi-mod nx=3 nz=2 h=10 n_pml=0 kind=velocity_mps\n" + body,
        "field": b"fwi-model nx=3 h=10 n_pml=0 kind=velocity_mps\n" + body,
        "kind": b"fwi-model nx=3 nz=2 h=10 n_pml=0 kind=speed\n" + body,
        "int": b"fwi-model nx=3.0 nz=2 h=10 n_pml=0 kind=velocity_mps\n" + body,
        "short": head + body[:-8],
        "trailing": head + body + b"\0",
        "nonpositive": head + struct.pack("<6d", 2000.0, 0.0, 1, 1, 1, 1),
        "nan": head + struct.pack("<6d", 2000.0, float("nan"), 1, 1, 1, 1),
        "empty": b"",
    }[case]
    # nx=3, nz=2 fails build_grid (nz < 3) after the header parses: use a 3 x 3 grid for payload cases
    if case in ("short", "trailing", "nonpositive", "nan"):
        data = data.replace(b"nz=2", b"nz=3") + struct.pack("<3d", 1.0, 1.0, 1.0)
        if case == "short":
            data = data[:-16]
    p = str(tmp_path / "m.mod")
    open(p, "wb").write(data)
    assert _ref_model_status(ref, p) == 1, case  # ParseError in the reference
    with pytest.raises(mio.ParseError):
        mio.read_model(p)


def _survey(seed=1, K=3, offset=True):
    rng = np.random.default_rng(seed)
    s = mio.SurveyFile(frequencies_hz=[2.5, 5.0, 7.25], weight_mode=_abi.FWI_WEIGHT_OFFSET if offset else 0)
    for k in range(K):
        rec = [(int(rng.integers(3, 20)), int(rng.integers(3, 9))) for _ in range(int(rng.integers(1, 6)))]
        s.sources.append(mio.SurveySource(int(4 + 3 * k), 4, float(rng.uniform(0.5, 2.0)), rec))
    return s


def _ref_write_survey(ref, path, s):
    K = s.num_sources
    fr = np.array(s.frequencies_hz)
    sx = np.array([x.ix for x in s.sources], np.int32)
    sz = np.array([x.iz for x in s.sources], np.int32)
    amp = np.array([x.amplitude for x in s.sources])
    off = np.zeros(K + 1, np.int32)
    off[1:] = np.cumsum([len(x.receivers) for x in s.sources])
    rx = np.array([r[0] for x in s.sources for r in x.receivers] + [0], np.int32)
    rz = np.array([r[1] for x in s.sources for r in x.receivers] + [0], np.int32)
    return ref.ref_write_survey(path.encode(), len(fr), dp(fr), s.weight_mode, K, ip(sx), ip(sz), dp(amp), ip(off),
                                ip(rx), ip(rz))


def test_survey_file_bytes_and_values_match_reference(tmp_path, ref):
    s = _survey()
    a, b = str(tmp_path / "ref.txt"), str(tmp_path / "ours.txt")
    assert _ref_write_survey(ref, a, s) == 0
    mio.write_survey(b, s)
    assert open(a, "rb").read() == open(b, "rb").read()
    got = mio.read_survey(a)
    assert got == s
    sv = got.to_survey()
    assert sv.num_sources == 3 and sv.num_data == s.num_data and sv.weight_mode == _abi.FWI_WEIGHT_OFFSET


def test_survey_syntax_comments_and_rejections(tmp_path, ref):
    ok = ("# leading comment\n\n fwi-survey  # magic\nfrequencies_hz 3 4\nfrequencies_hz 5\n"
          "weight_mode identity\nsource 5 5 # default amplitude\nreceivers 6 5 7 5\nreceivers 8 5\n"
          "source 6 5 2.5\n")
    p = str(tmp_path / "s.txt")
    open(p, "w").write(ok)
    s = mio.read_survey(p)
    counts = np.zeros(4, np.int32)
    assert ref.ref_read_survey(p.encode(), ip(counts), None, None, None, None, None, None, None) == 0
    assert (len(s.frequencies_hz), s.weight_mode, s.num_sources, s.num_data) == tuple(counts)
    assert s.frequencies_hz == [3.0, 4.0, 5.0] and s.sources[0].receivers == [(6, 5), (7, 5), (8, 5)]
    assert s.sources[0].amplitude == 1.0 and s.sources[1].amplitude == 2.5
    bad = ["frequencies_hz 3\n", "fwi-survey\n", "fwi-survey\nfrequencies_hz 3\nreceivers 1 2\n",
           "fwi-survey\nfrequencies_hz 3\nsource 1\n", "fwi-survey\nfrequencies_hz 3\nsource 1 2\nreceivers 1\n",
           "fwi-survey\nfrequencies_hz 3\nweight_mode flat\n", "fwi-survey\nfrequencies_hz 3\nshot 1 2\n",
           "fwi-survey\nfrequencies_hz x\n", "fwi-survey\nweight_mode offset identity\nfrequencies_hz 3\n"]
    for text in bad:
        open(p, "w").write(text)
        assert ref.ref_read_survey(p.encode(), ip(counts), None, None, None, None, None, None, None) == 1, text
        with pytest.raises(mio.ParseError):
            mio.read_survey(p)


def test_data_csv_bytes_and_values_match_reference(tmp_path, ref):
    s = _survey(seed=4)
    sp = str(tmp_path / "s.txt")
    mio.write_survey(sp, s)
    rng = np.random.default_rng(9)
    blocks = [rng.standard_normal(s.num_data) * 1e-3 + 1j * rng.standard_normal(s.num_data) for _ in range(3)]
    flat = np.ascontiguousarray(np.concatenate(blocks)).view(np.float64)
    a, b = str(tmp_path / "ref.csv"), str(tmp_path / "ours.csv")
    assert ref.ref_write_data(a.encode(), sp.encode(), dp(flat)) == 0
    mio.write_data(b, s, blocks)
    assert open(a, "rb").read() == open(b, "rb").read()
    got = mio.read_data(a, s)
    assert all(np.array_equal(x, y) for x, y in zip(got, blocks))
    # rejections: header, order, node mismatch, truncation, trailing rows, column count
    lines = open(a).read().splitlines(keepends=True)
    variants = {
        "header": [lines[0].replace("frequency_hz", "freq_hz")] + lines[1:],
        "order": [lines[0], lines[2], lines[1]] + lines[3:],
        "node": [lines[0], lines[1].replace(",", ",9", 4)] + lines[2:],
        "truncated": lines[:-1],
        "trailing": lines + [lines[-1]],
        "columns": [lines[0], lines[1].rstrip("\n") + ",0\n"] + lines[2:],
    }
    out = np.zeros_like(flat)
    for name, ls in variants.items():
        p = str(tmp_path / f"bad_{name}.csv")
        open(p, "w").write("".join(ls))
        assert ref.ref_read_data(p.encode(), sp.encode(), dp(out)) == 1, name
        with pytest.raises(mio.ParseError):
            mio.read_data(p, s)
    # blank trailing lines are accepted by both
    p = str(tmp_path / "blank.csv")
    open(p, "w").write("".join(lines) + "\n")
    assert ref.ref_read_data(p.encode(), sp.encode(), dp(out)) == 0
    assert all(np.array_equal(x, y) for x, y in zip(mio.read_data(p, s), blocks))


def _ref_config(ref, path):
    d, i = np.zeros(11), np.zeros(9, np.int32)
    fr, ep = np.zeros(64), np.zeros(64)
    st = ref.ref_read_config(path.encode(), dp(d), ip(i), dp(fr), dp(ep))
    return st, d, i, fr[:i[7]], ep[:i[8]]


def test_config_matches_reference(tmp_path, ref):
    text = ("# full-space GN configuration\nfrequencies_hz = 3 5 7\n  epsilon_list=1e10 2e10 3.5e10 # per f\n"
            "epsilon_start = 2\nepsilon_end = 4\nsolver = fsgn-gmres-ilu\nmax_inner = 25\ninner_tol = 1e-3\n"
            "gmres_restart = 12\nilu_level = 21\nilu_diag_shift = 0.5\ndrop_reg_term = true\n"
            "weight_mode = offset\nv_min = 1400\nv_max = 4800\necg_stride = 2\necg_stop_tol = 1e-4\n"
            "pml_power = 3\npml_c_ref = 2100.5\npml_sigma_max = 44\n\n")
    p = str(tmp_path / "c.cfg")
    open(p, "w").write(text)
    st, d, i, fr, ep = _ref_config(ref, p)
    assert st == 0
    c = mio.read_config(p)
    assert [c.epsilon_start, c.epsilon_end, c.inner_tol, c.ilu_diag_shift, c.v_min, c.v_max, c.ecg_stop_tol,
            c.pml_power, c.pml_c_ref, c.pml_sigma_max] == list(d[:10])
    assert [mio.SOLVERS.index(c.solver), c.max_inner, c.gmres_restart, c.ilu_level, int(c.drop_reg_term),
            c.weight_mode, c.ecg_stride, len(c.frequencies_hz), len(c.epsilon_list)] == list(i)
    assert c.frequencies_hz == list(fr) and c.epsilon_list == list(ep)
    assert [c.epsilon_for(k, 3) for k in range(3)] == [1e10, 2e10, 3.5e10]
    # defaults when a key is absent (include/fwi/driver.hpp:18-38)
    open(p, "w").write("solver = rsgn-cg\n")
    st, d, i, _, _ = _ref_config(ref, p)
    c = mio.read_config(p)
    assert st == 0 and c.pml_c_ref is None and math.isnan(d[8]) and c.weight_mode is None and i[5] == -1
    assert c.max_inner == i[1] == 30 and c.inner_tol == d[2] == 1e-12
    for text in ["max_inner = 3 4\n", "frequencies_hz =\n", "a b = 1\n", "solver_x = 1\n", "just words\n",
                 "drop_reg_term = yes\n", "max_inner = 2.5\n", "weight_mode = flat\n"]:
        open(p, "w").write(text)
        assert _ref_config(ref, p)[0] == 1, text
        with pytest.raises(mio.ParseError):
            mio.read_config(p)
    open(p, "w").write("solver = lu\n")  # inner_solver_from_string: std::invalid_argument
    assert _ref_config(ref, p)[0] == 3
    with pytest.raises(ValueError):
        mio.read_config(p)


def test_load_inversion_assembles_the_cli_problem(tmp_path):
    nx, nz, npml = 30, 20, 4
    v = np.linspace(1500, 2500, nx * nz)
    mp, sp, dpth, cp = (str(tmp_path / n) for n in ("m.mod", "s.txt", "d.csv", "c.cfg"))
    mio.write_model(mp, mio.ModelFile(Grid(nx, nz, 10.0, npml), mio.VELOCITY_MPS, v))
    s = mio.SurveyFile(frequencies_hz=[6.0, 4.0], sources=[mio.SurveySource(10, 6, 1.0, [(8, 6), (12, 6)]),
                                                          mio.SurveySource(18, 6, 2.0, [(20, 6)])])
    mio.write_survey(sp, s)
    mio.write_data(dpth, s, [np.full(3, 1 + 2j), np.full(3, 3 - 1j)])
    open(cp, "w").write("epsilon_start = 1\nepsilon_end = 3\ndrop_reg_term = true\n")
    inv = mio.load_inversion(mp, sp, dpth, cp)
    mf = mio.read_model(mp)
    assert inv.problem.grid.sigma_max == pml_sigma_max(mf.grid, mf.mean_velocity())
    assert inv.frequencies == [4.0, 6.0] and inv.epsilons == {4.0: 1.0, 6.0: 3.0}
    assert np.array_equal(inv.observed[4.0], np.full(3, 3 - 1j)) and inv.problem.drop_reg_term
    assert np.array_equal(inv.s0, 1.0 / (v * v)) and list(inv.problem.survey.src_amp) == [1.0, 2.0]
    open(cp, "w").write("pml_c_ref = 1800\npml_power = 3\n")
    inv = mio.load_inversion(mp, sp, dpth, cp)
    assert inv.problem.grid.sigma_max == pml_sigma_max(mf.grid, 1800.0) and inv.problem.grid.power == 3.0
    open(cp, "w").write("pml_sigma_max = 77\n")
    assert mio.load_inversion(mp, sp, dpth, cp).problem.grid.sigma_max == 77.0
    bad = mio.SurveyFile(frequencies_hz=[4.0], sources=[mio.SurveySource(1, 1, 1.0, [(8, 6)])])
    mio.write_survey(sp, bad)
    with pytest.raises(ValueError, match="outside the core"):
        mio.load_inversion(mp, sp, dpth)
    assert not os.path.exists(mp + ".tmp")
