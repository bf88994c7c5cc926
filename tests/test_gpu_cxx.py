"""GPU: the C++ drop-in header (include/fwi_b200/kkt.hpp) against the reference
library, as a compiled program (tests/cpp/test_cxx_parity.cpp, built by
__graft_entry__.build() where the reference sources exist)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "test_cxx_parity")

pytestmark = pytest.mark.gpu


def test_cxx_header_parity_program():
    if not os.path.exists(EXE):
        pytest.skip("build/test_cxx_parity was not built (needs the reference sources at build time)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-3000:]
