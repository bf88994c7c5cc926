"""ctypes mirror of the plain-C descriptor structs in include/fwi_b200.h.

Shared by the product binding (paper_2204_06489_b200.api) and by the test-only
oracle bindings (oracle/pyoracle.py); it holds types only, no behaviour.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

FWI_OK = 0
FWI_ERR_INVALID_ARGUMENT = 1
FWI_ERR_SINGULAR_PIVOT = 2
FWI_ERR_ZERO_PIVOT = 3
FWI_ERR_CUDA = 4
FWI_ERR_NOT_SUPPORTED = 5
FWI_ERR_OUT_OF_MEMORY = 6

FWI_PRECOND_EXACT = 0
FWI_PRECOND_ILU = 1
FWI_WEIGHT_IDENTITY = 0
FWI_WEIGHT_OFFSET = 1
FWI_C128 = 0
FWI_C64 = 1

_ip = C.POINTER(C.c_int)
_dp = C.POINTER(C.c_double)


class GridDesc(C.Structure):
    _fields_ = [("nx", C.c_int), ("nz", C.c_int), ("h", C.c_double), ("n_pml", C.c_int),
                ("pml_sigma_max", C.c_double), ("pml_power", C.c_double)]


class SurveyDesc(C.Structure):
    _fields_ = [("num_sources", C.c_int), ("src_ix", _ip), ("src_iz", _ip), ("src_amp", _dp),
                ("recv_offset", _ip), ("recv_ix", _ip), ("recv_iz", _ip),
                ("weight_mode", C.c_int)]


class StateDesc(C.Structure):
    _fields_ = [("grid", GridDesc), ("survey", SurveyDesc), ("freq_hz", C.c_double),
                ("epsilon", C.c_double), ("drop_reg_term", C.c_int), ("s", _dp), ("u", _dp),
                ("r", _dp), ("d_obs", _dp), ("exact_factor", C.c_int), ("ilu_level", C.c_int),
                ("ilu_diag_shift", C.c_double), ("precision_mask", C.c_int)]


class StateInfo(C.Structure):
    _fields_ = [("nx", C.c_int), ("nz", C.c_int), ("n", C.c_int), ("num_sources", C.c_int),
                ("num_data", C.c_int), ("omega", C.c_double), ("epsilon", C.c_double),
                ("drop_reg_term", C.c_int), ("has_exact", C.c_int), ("has_ilu", C.c_int),
                ("vec_doubles", C.c_int64), ("device_bytes", C.c_int64),
                ("exact_factor_bytes", C.c_int64), ("ilu_factor_bytes", C.c_int64),
                ("exact_probe_residual", C.c_double)]


class FsgnOptions(C.Structure):
    _fields_ = [("mode", C.c_int), ("restart", C.c_int), ("tol", C.c_double),
                ("maxit", C.c_int), ("ecg_stride", C.c_int), ("ecg_stop_tol", C.c_double)]


FWI_SOLVER_FSGN_EXACT = 1
FWI_SOLVER_FSGN_ILU = 2


class GnOptions(C.Structure):
    _fields_ = [("solver", C.c_int), ("max_inner", C.c_int), ("inner_tol", C.c_double),
                ("gmres_restart", C.c_int), ("ilu_level", C.c_int), ("ilu_diag_shift", C.c_double),
                ("v_min", C.c_double), ("v_max", C.c_double), ("ecg_stride", C.c_int),
                ("ecg_stop_tol", C.c_double)]


class GnResult(C.Structure):
    _fields_ = [("misfit_ini", C.c_double), ("misfit_fin", C.c_double), ("update_relnorm", C.c_double),
                ("wall_seconds", C.c_double), ("setup_seconds", C.c_double), ("ilu_factor_seconds", C.c_double),
                ("krylov_seconds", C.c_double), ("final_seconds", C.c_double)]


class LogEntry(C.Structure):
    _fields_ = [("iteration", C.c_int), ("has_precond_residual", C.c_int),
                ("has_normal_residual", C.c_int), ("pad_", C.c_int),
                ("residual_norm", C.c_double), ("precond_residual", C.c_double),
                ("normal_residual", C.c_double), ("wall_time", C.c_double)]


class ConvergenceLogC(C.Structure):
    _fields_ = [("entries", C.POINTER(LogEntry)), ("capacity", C.c_int), ("count", C.c_int),
                ("converged", C.c_int), ("stagnated", C.c_int)]


def iptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_ip)


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype in (np.float64, np.complex128) and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


class LogBuffer:
    """Caller-owned storage for fwi_convergence_log."""

    def __init__(self, capacity: int):
        self.entries = (LogEntry * max(capacity, 1))()
        self.c = ConvergenceLogC(C.cast(self.entries, C.POINTER(LogEntry)), max(capacity, 1), 0, 0, 0)

    def to_log(self):
        from .krylov import ConvergenceLog, LogEntryPy
        out = ConvergenceLog(converged=bool(self.c.converged), stagnated=bool(self.c.stagnated))
        for i in range(self.c.count):
            e = self.entries[i]
            out.entries.append(LogEntryPy(
                iteration=e.iteration, residual_norm=e.residual_norm,
                normal_residual=e.normal_residual if e.has_normal_residual else None,
                precond_residual=e.precond_residual if e.has_precond_residual else None,
                wall_time=e.wall_time))
        return out
