"""CPU: the C-ABI library loads and exports every entry point include/fwi_b200.h
declares (no compute calls: there is no GPU here). Also checks that the
plain-C structs mirrored in Python (_abi.py) have the C layout."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2204_06489_b200 import _abi, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fwi_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b((?:fwi_dev|fwi_host)_\w+)\s*\(", src)))


def test_header_declares_the_reference_interface():
    names = declared()
    for must in ["fwi_dev_ctx_create", "fwi_dev_kkt_apply", "fwi_dev_kkt_apply_host", "fwi_dev_kkt_rhs",
                 "fwi_dev_precond_apply", "fwi_dev_fsgn_gmres_step", "fwi_dev_gmres_generic",
                 "fwi_dev_vec_dot", "fwi_dev_vec_axpy", "fwi_dev_solve", "fwi_dev_factor_ilu"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(api.build_library())
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a_only():
    so = api.build_library()
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_struct_layouts_match_the_header():
    # compile a tiny C program printing sizeof/offsetof of the header structs
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "fwi_b200.h"
int main(void){
 printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(fwi_grid_desc), sizeof(fwi_survey_desc), sizeof(fwi_state_desc),
        sizeof(fwi_state_info), sizeof(fwi_fsgn_options), sizeof(fwi_log_entry), sizeof(fwi_convergence_log));
 printf("%zu %zu %zu\n", offsetof(fwi_state_desc, s), offsetof(fwi_state_desc, precision_mask),
        offsetof(fwi_log_entry, wall_time));
 return 0;}
'''
    tmp = os.path.join(ROOT, "build")
    os.makedirs(tmp, exist_ok=True)
    src, exe = os.path.join(tmp, "layout.c"), os.path.join(tmp, "layout")
    open(src, "w").write(prog)
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
    sizes, offs = subprocess.run([exe], capture_output=True, text=True).stdout.split("\n")[:2]
    got = [C.sizeof(t) for t in (_abi.GridDesc, _abi.SurveyDesc, _abi.StateDesc, _abi.StateInfo,
                                 _abi.FsgnOptions, _abi.LogEntry, _abi.ConvergenceLogC)]
    assert got == [int(v) for v in sizes.split()]
    assert [_abi.StateDesc.s.offset, _abi.StateDesc.precision_mask.offset,
            _abi.LogEntry.wall_time.offset] == [int(v) for v in offs.split()]


def test_no_cpu_fallback_without_gpu():
    """With no CUDA device, creating a device state must fail loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2204_06489_b200.problem import small_problem
    with pytest.raises(api.FwiError):
        api.GnState(small_problem())
