"""CPU: the `fwi` command line (paper_2204_06489_b200/cli.py, the reference's tools/fwi.cpp:342-435)
— flags, exit codes and the file-only subcommand (make-model) against the reference's own
generators and writers (oracle/_ref via ref_harness.cpp); the device subcommands are covered by
tests/test_gpu_cli.py."""
import ctypes as C
import os

import numpy as np
import pytest

import pyoracle as po
from paper_2204_06489_b200 import cli
from paper_2204_06489_b200 import model_io as mio
from paper_2204_06489_b200.problem import Grid

_dp, _ip = C.POINTER(C.c_double), C.POINTER(C.c_int)


@pytest.fixture(scope="module")
def ref():
    L = po.ref_lib()
    L.ref_make_model.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, _dp, C.c_int, _ip, C.c_int,
                                 C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, _dp]
    L.ref_write_model.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, _dp]
    L.ref_write_heatmap.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_double, C.c_int, _dp]
    return L


def _ref_model(L, kind, nx, nz, h, npml, vel=(), ifc=(), bg=0.0, amp=0.0, cx=0.0, cz=0.0, rad=0.0):
    v = np.ascontiguousarray(vel, np.float64)
    i = np.ascontiguousarray(ifc, np.int32)
    out = np.empty(nx * nz)
    assert L.ref_make_model(kind, nx, nz, h, npml, v.ctypes.data_as(_dp), v.size, i.ctypes.data_as(_ip), i.size, bg,
                            amp, cx, cz, rad, out.ctypes.data_as(_dp)) == 0
    return out


def test_make_model_layered_byte_identical(tmp_path, ref):
    out = str(tmp_path / "lay.mod")
    rc = cli.main(["make-model", "--kind", "layered", "--nx", "40", "--nz", "30", "--spacing", "12.5", "--n-pml", "5",
                   "--out", out, "--velocities", "1500,2200,3100", "--interfaces", "8,19"])
    assert rc == 0
    want = _ref_model(ref, 0, 40, 30, 12.5, 5, vel=[1500, 2200, 3100], ifc=[8, 19])
    wpath = str(tmp_path / "ref.mod")
    assert ref.ref_write_model(wpath.encode(), 40, 30, 12.5, 5, 0, want.ctypes.data_as(_dp)) == 0
    assert open(out, "rb").read() == open(wpath, "rb").read()


@pytest.mark.parametrize("out_kind", ["velocity_mps", "slowness_sq"])
def test_make_model_lens_byte_identical(tmp_path, ref, out_kind):
    out = str(tmp_path / "lens.mod")
    rc = cli.main(["make-model", "--kind", "lens", "--nx", "33", "--nz", "21", "--spacing", "10", "--n-pml", "4",
                   "--out", out, "--background", "2000", "--amplitude", "-300", "--out-kind", out_kind])
    assert rc == 0
    want = _ref_model(ref, 1, 33, 21, 10.0, 4, bg=2000.0, amp=-300.0, cx=16.0, cz=10.0, rad=33 / 8.0)
    if out_kind == "slowness_sq":
        want = 1.0 / (want * want)
    wpath = str(tmp_path / "ref.mod")
    assert ref.ref_write_model(wpath.encode(), 33, 21, 10.0, 4, int(out_kind == "slowness_sq"),
                               want.ctypes.data_as(_dp)) == 0
    assert open(out, "rb").read() == open(wpath, "rb").read()


def test_make_model_import_raw(tmp_path):
    raw = tmp_path / "v.f32"
    v = np.linspace(1500, 3000, 12 * 9).astype("<f4")
    raw.write_bytes(v.tobytes())
    out = str(tmp_path / "imp.mod")
    assert cli.main(["make-model", "--kind", "import-raw", "--nx", "12", "--nz", "9", "--spacing", "5",
                     "--n-pml", "2", "--raw", str(raw), "--out", out]) == 0
    m = mio.read_model(out)
    assert np.array_equal(m.values, v.astype(np.float64))
    raw.write_bytes(v.tobytes()[:-4])  # wrong size: ParseError -> 3
    assert cli.main(["make-model", "--kind", "import-raw", "--nx", "12", "--nz", "9", "--spacing", "5",
                     "--n-pml", "2", "--raw", str(raw), "--out", out]) == 3


def test_heatmap_byte_identical(tmp_path, ref):
    g = Grid(30, 20, 10.0, 3)
    vals = 1500.0 + 30.0 * np.sin(np.arange(g.n) * 0.37)
    mio.write_heatmap(str(tmp_path / "a.ppm"), g, vals)
    assert ref.ref_write_heatmap(str(tmp_path / "b.ppm").encode(), 30, 20, 10.0, 3, vals.ctypes.data_as(_dp)) == 0
    assert (tmp_path / "a.ppm").read_bytes() == (tmp_path / "b.ppm").read_bytes()
    assert (tmp_path / "a.txt").read_bytes() == (tmp_path / "b.txt").read_bytes()


def test_exit_codes(tmp_path):
    # usage errors: CLI11's codes
    assert cli.main([]) == 106
    assert cli.main(["invert", "--initial", "x"]) == 106
    assert cli.main(["simulate", "--model", "a", "--survey", "b", "--out", "c", "--bogus"]) == 109
    assert cli.main(["make-model", "--kind", "lens", "--nx", "ten", "--nz", "3", "--spacing", "1", "--n-pml", "0",
                     "--out", "x"]) == 104
    # io error -> 2
    assert cli.main(["simulate", "--model", str(tmp_path / "missing.mod"), "--survey", "s", "--out", "o"]) == 2
    # invalid input (std::invalid_argument) -> 3
    assert cli.main(["make-model", "--kind", "layered", "--nx", "10", "--nz", "10", "--spacing", "1",
                     "--n-pml", "1", "--out", str(tmp_path / "m.mod"), "--velocities", "1500,2000",
                     "--interfaces", "12"]) == 3
    # parse error -> 3
    assert cli.main(["make-model", "--kind", "cube", "--nx", "10", "--nz", "10", "--spacing", "1", "--n-pml", "1",
                     "--out", str(tmp_path / "m.mod")]) == 3
    cfg = tmp_path / "bad.cfg"
    cfg.write_text("max_inner = 1e400\n")
    with pytest.raises(mio.ParseError):
        mio.read_config(str(cfg))
